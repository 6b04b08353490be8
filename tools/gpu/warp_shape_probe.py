"""Dev probe (DESIGN.md §12 "warp pixel shape"): how much would 2D pixel
blocks per warp gain? Every pixel's result depends only on its own G-buffer
entry, so the same frames can be shaded with their pixels permuted in memory:
each aligned run of 32 pixels (what one warp shades per iteration) becomes a
bw x bh block of the image. The kernel is unchanged; only which pixels share
a warp changes. Checks that the permuted outputs equal the row-major ones bit
for bit, then times both with glint_eval_batch (CUDA events).

usage: python tools/gpu/warp_shape_probe.py [--config C2|C5] [--reps N]"""
import argparse
import json

import torch

import paper_2306_05051_b200 as pkg
from paper_2306_05051_b200 import synth


def permute(p, bw, bh):
    """(H, W, 4) -> (H*W/1024, 1024, 4), each run of 32 = one bw x bh block."""
    H, W, _ = p.shape
    q = p.reshape(H // bh, bh, W // bw, bw, 4).permute(0, 2, 1, 3, 4).reshape(-1, 1024, 4)
    return q.contiguous()


def unpermute(q, H, W, bw, bh):
    return q.reshape(H // bh, W // bw, bh, bw, 4).permute(0, 2, 1, 3, 4).reshape(H, W, 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ctx = pkg.Context(0)
    if args.config == "C2":
        frames = synth.c2_frames(device="cuda")
    else:
        frames = [synth.c5(f, device="cuda") for f in range(0, 64, 4)]
    H, W = frames[0].gbuf.height, frames[0].gbuf.width
    res = {"config": args.config, "frames": len(frames)}
    ref = pkg.glint_eval_batch(ctx, [f.gbuf for f in frames], [f.scene for f in frames])
    torch.cuda.synchronize()

    def timeit(gbs, scs):
        outs = pkg.glint_eval_batch(ctx, gbs, scs)
        for _ in range(3):
            pkg.glint_eval_batch(ctx, gbs, scs, outs=outs)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            pkg.glint_eval_batch(ctx, gbs, scs, outs=outs)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.reps, outs

    ms, _ = timeit([f.gbuf for f in frames], [f.scene for f in frames])
    res["32x1 ms"] = ms
    for bw, bh in ((16, 2), (8, 4)):
        gbs = [synth.GBuffer(*[permute(p, bw, bh) for p in f.gbuf.planes()]) for f in frames]
        ms, outs = timeit(gbs, [f.scene for f in frames])
        same = all(torch.equal(unpermute(o, H, W, bw, bh).view(torch.int32), r.view(torch.int32))
                   for o, r in zip(outs, ref))
        res[f"{bw}x{bh} ms"] = ms
        res[f"{bw}x{bh} bit-identical"] = same
        del gbs, outs
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
