"""Multi-rank host logic of the frame-sharded driver on CPU:
world_size 2 over gloo (127.0.0.1). Frames are shard-disjoint and complete,
the timing reduction is a max over ranks, and rank 0 can assemble every
frame's image from the other ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_05051_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r, w, _ = D.init("gloo")
    assert (r, w) == (rank, world)
    frames = list(range(10))
    mine = D.shard(frames, r, w)
    # each rank "shades" its frames: an image that encodes frame id and rank
    imgs = {f: torch.full((4, 6, 4), float(f * 10 + r)) for f in mine}
    t = D.max_over_ranks(1.0 + r)
    s = D.sum_over_ranks(len(mine))
    full = D.gather_frames(imgs, frames, shape=(4, 6, 4))
    D.barrier()
    if r == 0:
        q.put((mine, t, s, sorted(full), {f: float(full[f][0, 0, 0]) for f in full}))
    else:
        q.put((mine, t, s, None, None))
    dist.destroy_process_group()


def test_shard_covers_frames_once():
    for world in (1, 2, 3, 8):
        got = sorted(f for r in range(world) for f in D.shard(range(64), r, world))
        assert got == list(range(64))


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res0 = next(x for x in res if x[3] is not None)
    res1 = next(x for x in res if x[3] is None)
    assert sorted(res0[0] + res1[0]) == list(range(10))
    assert res0[1] == 2.0 and res1[1] == 2.0          # max over ranks
    assert res0[2] == 10.0                            # sum of shards
    assert res0[3] == list(range(10))                 # rank 0 has every frame
    for f, v in res0[4].items():
        assert v == f * 10 + (f % 2)                  # frame f came from rank f % 2
