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


def _shade_tile_oracle(f, y0, y1, W=64, H=48):
    """The test's stand-in for a rank's kernel: the oracle on one tile of a
    small C2 frame (elevation by frame), as an (rows, W, 4) float32 image
    (RGB rounded to fp32, flag bits in .w)."""
    import numpy as np
    import oracle
    from paper_2306_05051_b200 import synth
    fr = synth.c2(15 + 20 * f, width=W, height=H, window=(y0, y1, 0, W))
    rgb, fl, _ = oracle.eval(fr.gbuf, fr.scene)
    img = np.zeros((y1 - y0, W, 4), np.float32)
    img[..., :3] = rgb.reshape(y1 - y0, W, 3).astype(np.float32)
    img[..., 3] = fl.reshape(y1 - y0, W).view(np.float32)
    return torch.from_numpy(img)


def _tile_worker(rank, world, port, n_frames, q, band_rows=16):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        r, w, _ = D.init("gloo")
        H, W = 48, 64
        tiles = D.plan_tiles(n_frames, H, w, band_rows=band_rows)
        g = D.TileGather(tiles, r, w, full=[torch.full((H, W, 4), float("nan")) for _ in range(n_frames)]
                         if r == 0 else None)
        local = {}
        for i in g.mine:
            f, y0, y1 = tiles[i]
            img = _shade_tile_oracle(f, y0, y1)
            if r == 0:
                g.full[f][y0:y1] = img           # rank 0 shades in place
            else:
                local[i] = img
        for wk in g.run(local):
            wk.wait()
        D.barrier()
        q.put((r, [t.numpy().copy() for t in g.full] if r == 0 else None, tiles))
        dist.destroy_process_group()
    except Exception as e:   # report instead of hanging the parent
        q.put((rank, repr(e), None))


@pytest.mark.parametrize("world,n_frames", [(2, 1), (2, 3), (4, 1), (4, 3), (8, 1)])
def test_gloo_tile_gather_assembles_the_single_rank_image(world, n_frames):
    """SURVEY 8e at world sizes 2, 4 and 8 on CPU: one frame cut into bands (C2 /
    C3-style row-band sharding) or three frames (whole frames at 2 ranks,
    bands of every frame at 4: fewer frames than ranks), each tile shaded by its rank
    (the oracle stands in for the kernel) and gathered to rank 0 by the
    per-tile send/recv rounds of dist.TileGather: rank 0's assembled frames
    equal the whole frames shaded in one process, bit for bit."""
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    band = {2: 16, 4: 8, 8: 4}[world]
    ps = [ctx.Process(target=_tile_worker, args=(r, world, port, n_frames, q, band)) for r in range(world)]
    for p in ps:
        p.start()
    res = {r: (full, tiles) for r, full, tiles in (q.get(timeout=300) for _ in ps)}
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    full, tiles = res[0]
    assert not isinstance(full, str), full
    if n_frames == 1:
        assert len(tiles) == 48 // band                          # the frame's bands
    else:
        assert len(tiles) == (3 if world <= 3 else 3 * (48 // band))   # whole frames, or bands of every frame
    assert {i % world for i in range(len(tiles))} == set(range(world))   # every rank shaded something
    for f in range(n_frames):
        ref = _shade_tile_oracle(f, 0, 48).numpy()
        assert np.array_equal(full[f].view(np.uint32), ref.view(np.uint32)), f


def test_plan_tiles_partitions_every_row_once():
    for n_frames, H, world in ((1, 2160, 8), (10, 1080, 8), (10, 1080, 1), (64, 2160, 8), (8, 2160, 3), (1, 37, 4)):
        tiles = D.plan_tiles(n_frames, H, world)
        rows = {}
        for f, y0, y1 in tiles:
            for y in range(y0, y1):
                assert (f, y) not in rows
                rows[(f, y)] = 1
        assert len(rows) == n_frames * H
        per_rank = [len(D.shard(tiles, r, world)) for r in range(world)]
        assert max(per_rank) - min(per_rank) <= 1
