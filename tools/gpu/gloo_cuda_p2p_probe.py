"""Probe: does torch.distributed's gloo backend move CUDA tensors with
batch_isend_irecv (so the NCCL-mode TileGather code path can be exercised on
one GPU by two processes)? Prints one line per rank."""
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    t = torch.full((4,), float(rank + 1), device="cuda")
    try:
        if rank == 0:
            r = torch.zeros(4, device="cuda")
            for w in dist.batch_isend_irecv([dist.P2POp(dist.irecv, r, 1)]):
                w.wait()
            print("rank0 got", r.tolist(), flush=True)
        else:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, t, 0)]):
                w.wait()
            print("rank1 sent", flush=True)
    except Exception as e:
        print(f"rank{rank} failed: {e!r}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(worker, args=(port,), nprocs=2)
