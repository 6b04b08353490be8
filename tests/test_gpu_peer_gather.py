"""The fused gather of SURVEY §8e on one GPU: two processes (gloo control
plane, 127.0.0.1), rank 0 owns one buffer for all frames and maps it into
rank 1 through CUDA IPC (dist.peer_buffer: the handle opened from rank 1's
own device with lazy peer access, the path a multi-GPU rank takes); each rank's kernel stores its
frames (f = rank mod 2) straight into that buffer. No kernel waits on another
rank: rank 1 only writes, then a host barrier. Rank 0 then checks every frame
bit for bit against its own local evaluation."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import torch.distributed as dist
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import dist as D
    from paper_2306_05051_b200 import synth
    try:
        D.init("gloo")
        torch.cuda.set_device(0)
        ctx = pkg.Context(0)
        frames = [synth.c2(e, window=(500, 564, 0, 256), device="cuda") for e in (15, 35, 55, 75, 90)]
        buf = D.peer_buffer((len(frames), 64, 256, 4), device=torch.device("cuda", 0))
        if rank == 1 and D.LAST_MAPPING != "ipc-open on the rank's device":
            raise RuntimeError(f"peer buffer mapped by {D.LAST_MAPPING}")
        if rank == 0:
            buf.fill_(float("nan"))
            torch.cuda.synchronize()
        D.barrier()
        for f in D.shard(range(len(frames)), rank, world):
            pkg.glint_eval(ctx, frames[f].gbuf, frames[f].scene, out=buf[f])
        torch.cuda.synchronize()
        D.barrier()
        ok = True
        if rank == 0:
            for f, fr in enumerate(frames):
                ref = pkg.glint_eval(ctx, fr.gbuf, fr.scene)
                torch.cuda.synchronize()
                ok &= torch.equal(ref.view(torch.int32), buf[f].view(torch.int32))
        D.barrier()
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))


def test_peer_gather_two_processes_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    assert res == {0: True, 1: True}, res
