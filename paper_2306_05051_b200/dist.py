"""Frame sharding across ranks.

Every (pixel, light) evaluation is a pure function of its G-buffer entry, the
scene and the seed, so frames are independent: rank r shades frames
f = r, r + world, r + 2 world, ... with no data-path collective. The only
collectives are control-plane ones: a barrier around the timed region and a
max-reduction of the per-rank device time. Result assembly on rank 0 is
optional and outside the timed region.
"""
from __future__ import annotations

import os
from typing import List, Sequence

import torch
import torch.distributed as dist


def env_rank_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init(backend: str = "nccl"):
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def shard(frame_ids: Sequence[int], rank: int, world: int) -> List[int]:
    """Round-robin frame assignment (f mod world == rank)."""
    return [f for f in frame_ids if f % world == rank]


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def gather_frames(images: dict, frame_ids: Sequence[int], shape, dtype=torch.float32, device=None, dst: int = 0):
    """Assemble {frame_id: image} from every rank on rank ``dst`` (point-to-point
    sends over the process group; NCCL over NVLink on GPUs, gloo on CPU). Each
    rank passes the frames it shaded; returns the full dict on ``dst``."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(images)
    rank, world = dist.get_rank(), dist.get_world_size()
    out = dict(images) if rank == dst else None
    for src in range(world):
        if src == dst:
            continue
        for f in shard(frame_ids, src, world):
            if rank == src:
                dist.send(images[f].contiguous(), dst=dst)
            elif rank == dst:
                buf = torch.empty(shape, dtype=dtype, device=device)
                dist.recv(buf, src=src)
                out[f] = buf
    return out


def peer_buffer(shape, dtype=torch.float32, device=None, src: int = 0):
    """One device buffer owned by rank ``src`` and mapped into every rank's
    address space (CUDA IPC: cudaIpcGetMemHandle / cudaIpcOpenMemHandle with
    lazy peer access, through torch's tensor-sharing reductions). A rank that
    passes a slice of it as ``out`` to glint_eval has its kernel store the
    radiance straight into rank ``src``'s HBM over NVLink: the gather to rank 0
    becomes part of the shading kernel, overlapping it tile by tile, with no
    separate collective. Returns the buffer (``src``) or its
    mapping (others); the control plane only moves the IPC handle."""
    from torch.multiprocessing.reductions import rebuild_cuda_tensor, reduce_tensor
    rank = dist.get_rank() if dist.is_initialized() else 0
    world = dist.get_world_size() if dist.is_initialized() else 1
    if rank == src:
        buf = torch.empty(shape, dtype=dtype, device=device)
        if world == 1:
            return buf
        _, args = reduce_tensor(buf)
        obj = [args]
    else:
        buf, obj = None, [None]
    if world > 1:
        dist.broadcast_object_list(obj, src=src)
        if rank != src:
            buf = rebuild_cuda_tensor(*obj[0])
    return buf
