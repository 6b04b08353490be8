"""Work partitioning across ranks and the gather to rank 0 (DESIGN.md §8,
SURVEY §8e).

Every (pixel, light) evaluation is a pure function of its G-buffer entry, the
scene and the seed, so any split of the pixels is exact: the unit of work is a
*tile* (frame, y0, y1), a band of full-width rows of one frame. Multi-frame
configs (C4, C5) use whole frames; single-frame ones (C2's elevations, C3) at
more than one rank use 64-row bands dealt round-robin, so the sky / plane /
sphere mix (and the per-pixel cost) balances across ranks. Each
rank generates its own tiles' G-buffers (no input scatter).

The one data-path collective is the gather of radiance to rank 0, in either of
two forms:

* fused (``peer_buffer``): rank 0's full-frame outputs are mapped into every
  rank through CUDA IPC; a rank passes them, with each tile's origin (glint.h
  x0, y0), as its kernels' outputs, so the radiance streams straight into
  rank 0's HBM over NVLink tile by tile, with no separate pass;
* NCCL (``TileGather``): each rank shades into local buffers and sends each
  tile to rank 0 on a dedicated communication stream as soon as that tile's
  kernel is done (a CUDA event), so the transfer overlaps the next tiles'
  shading; rank 0 receives in place into its full frames.

Control plane: a barrier on both sides of the timed region and max / sum
reductions of per-rank numbers.
"""
from __future__ import annotations

import datetime
import os
from typing import Dict, List, Sequence, Tuple

import torch
import torch.distributed as dist

Tile = Tuple[int, int, int]          # (frame, y0, y1): rows [y0, y1) of a frame, full width

# a hung peer must not hang the job (and the GPU box) forever
TIMEOUT = datetime.timedelta(seconds=int(os.environ.get("GLINT_DIST_TIMEOUT_S", "600")))


def env_rank_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init(backend: str = "nccl"):
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=TIMEOUT)
        else:
            dist.init_process_group(backend, timeout=TIMEOUT)
    return rank, world, local


def shard(items: Sequence, rank: int, world: int) -> List:
    """Round-robin assignment by position: item i goes to rank i mod world."""
    return [x for i, x in enumerate(items) if i % world == rank]


def row_bands(height: int, rows: int = 64) -> List[Tuple[int, int]]:
    """Full-width bands of ``rows`` rows (the last one ragged)."""
    return [(y, min(height, y + rows)) for y in range(0, height, rows)]


def plan_tiles(n_frames: int, height: int, world: int, band_rows: int = 64) -> List[Tile]:
    """The global tile list of a step: whole frames when there are at least
    as many frames as ranks (C4, C5) or a single rank; otherwise 64-row bands
    of every frame (C2, C3), listed frame by frame."""
    if world == 1 or n_frames >= world:
        return [(f, 0, height) for f in range(n_frames)]
    return [(f, y0, y1) for f in range(n_frames) for (y0, y1) in row_bands(height, band_rows)]


def _reduce_device(device):
    """gloo reduces host tensors; NCCL device tensors."""
    return "cpu" if dist.get_backend() == "gloo" else device


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_reduce_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_reduce_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def gather_frames(images: dict, frame_ids: Sequence[int], shape, dtype=torch.float32, device=None, dst: int = 0):
    """Assemble {frame_id: image} from every rank on rank ``dst`` (point-to-point
    sends over the process group; NCCL over NVLink on GPUs, gloo on CPU). Each
    rank passes the frames it shaded (frame f on rank f mod world); returns the
    full dict on ``dst``."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(images)
    rank, world = dist.get_rank(), dist.get_world_size()
    out = dict(images) if rank == dst else None
    for src in range(world):
        if src == dst:
            continue
        for f in shard(list(frame_ids), src, world):
            if rank == src:
                dist.send(images[f].contiguous(), dst=dst)
            elif rank == dst:
                buf = torch.empty(shape, dtype=dtype, device=device)
                dist.recv(buf, src=src)
                out[f] = buf
    return out


class TileGather:
    """Per-tile gather of radiance to rank 0 over the process group, overlapped
    with shading. ``tiles`` is the global tile list and ``full`` (rank 0 only)
    the full-frame outputs; tile i is shaded by rank i mod world.

    Round k moves the k-th tile of every rank r >= 1 to rank 0 as one batched
    send/recv group (NCCL grouped p2p: all peers stream into rank 0 at once).
    On a GPU the rounds run on ``comm_stream``; a rank's send of its k-th tile
    first waits for that tile's CUDA event (recorded after its kernel on the
    compute stream), so the transfer overlaps the shading of its next tiles.
    Rank 0 receives straight into ``full[frame][y0:y1]`` (contiguous rows).
    On CPU (gloo) the same rounds run synchronously."""

    def __init__(self, tiles: Sequence[Tile], rank: int, world: int, full=None, comm_stream=None):
        self.tiles, self.rank, self.world = list(tiles), rank, world
        self.full, self.stream = full, comm_stream
        self.mine = [i for i in range(len(self.tiles)) if i % world == rank]
        self.rounds = (len(self.tiles) + world - 1) // world

    def _round_ops(self, k: int, local_outs: Dict[int, torch.Tensor]):
        ops = []
        if self.rank == 0:
            for r in range(1, self.world):
                i = k * self.world + r
                if i < len(self.tiles):
                    f, y0, y1 = self.tiles[i]
                    ops.append(dist.P2POp(dist.irecv, self.full[f][y0:y1], r))
        else:
            i = k * self.world + self.rank
            if i < len(self.tiles):
                ops.append(dist.P2POp(dist.isend, local_outs[i], 0))
        return ops

    def run(self, local_outs: Dict[int, torch.Tensor], events: Dict[int, "torch.cuda.Event"] = None):
        """Issue every round; returns the works (wait on them, or on the comm
        stream). ``local_outs`` / ``events``: this rank's tiles by global index
        (rank 0 shades into ``full`` directly and passes none)."""
        works = []
        for k in range(self.rounds):
            i = k * self.world + self.rank
            if self.stream is not None:
                with torch.cuda.stream(self.stream):
                    if self.rank != 0 and events is not None and i in events:
                        self.stream.wait_event(events[i])
                    ops = self._round_ops(k, local_outs)
                    if ops:
                        works += dist.batch_isend_irecv(ops)
            else:
                ops = self._round_ops(k, local_outs)
                if ops:
                    works += dist.batch_isend_irecv(ops)
        return works


LAST_MAPPING = None      # how this process last mapped a peer buffer (tests)


class _DevicePointer:
    """A device pointer seen through __cuda_array_interface__ (no copy). The
    tensor torch builds over it keeps this object alive; when the last view
    goes, the IPC mapping ``mapped`` is closed."""

    def __init__(self, ptr, shape, strides_bytes, typestr, mapped=None):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "strides": tuple(strides_bytes), "version": 3}
        self._mapped = mapped

    def __del__(self):
        if self._mapped is not None:
            try:
                from cuda.bindings import runtime as rt
                rt.cudaIpcCloseMemHandle(self._mapped)
            except Exception:     # interpreter shutdown: the process exit unmaps it
                pass


def _ipc_open_here(args):
    """Map rank ``src``'s exported allocation into this process from THIS
    rank's device: cudaIpcOpenMemHandle with cudaIpcMemLazyEnablePeerAccess,
    called with the rank's own device current, enables peer access from it to
    the owner's device, which is what its kernels' stores need (torch's own
    rebuild opens the handle from the owner's device, whose peer mapping the
    rank's device would not have). Returns a tensor over the mapping, or None
    when the handle is not a plain cudaMalloc export."""
    (_cls, size, stride, toff, _scls, dtype, _sdev, handle, _sbytes, soff) = args[:10]
    # torch's handle: [version byte (2)] + type byte ('c': cudaMalloc) + cudaIpcMemHandle_t
    if len(handle) == 66 and handle[1:2] == b"c":
        raw = handle[2:]
    elif len(handle) == 65 and handle[:1] == b"c":
        raw = handle[1:]
    else:
        raw = handle
    if len(raw) != 64:
        return None
    try:
        from cuda.bindings import runtime as rt
    except ImportError:   # no cuda-python: torch's own mapping (same-device ranks only)
        return None
    dev = torch.cuda.current_device()
    (err,) = rt.cudaSetDevice(dev)
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"cudaSetDevice({dev}): {err}")
    h = rt.cudaIpcMemHandle_t()
    h.reserved = bytes(raw)
    err, ptr = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"cudaIpcOpenMemHandle on device {dev}: {err}")
    item = torch.empty((), dtype=dtype).element_size()
    typestr = {torch.float32: "<f4", torch.int32: "<i4", torch.uint8: "|u1"}[dtype]
    base = int(ptr) + int(soff) + int(toff) * item
    return torch.as_tensor(_DevicePointer(base, size, [st * item for st in stride], typestr, mapped=ptr))


def peer_buffer(shape, dtype=torch.float32, device=None, src: int = 0):
    """One device buffer owned by rank ``src`` and mapped into every rank's
    address space (CUDA IPC: cudaIpcGetMemHandle on the owner, then
    cudaIpcOpenMemHandle with lazy peer access from each rank's own device).
    A rank that passes a slice of it as ``out`` to glint_eval has its kernel
    store the radiance straight into rank ``src``'s HBM over NVLink: the
    gather to rank 0 becomes part of the shading kernel, overlapping it tile
    by tile, with no separate collective. Returns the buffer
    (``src``) or its mapping (others); the control plane only moves the IPC
    handle."""
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
            global LAST_MAPPING
            buf = _ipc_open_here(obj[0])
            LAST_MAPPING = "ipc-open on the rank's device"
            if buf is None:       # not a plain cudaMalloc export: torch's own mapping
                buf = rebuild_cuda_tensor(*obj[0])
                LAST_MAPPING = "torch rebuild"
    return buf
