"""Upper bound for a one-launch multi-frame kernel: the per-frame overhead
that chained launches (glint_eval_batch) still pay. Ten chained launches of
the same C2 frame vs one launch over the ten frames stacked vertically (same
scene, same pixels, 10x the tiles). CUDA events on the launch stream.

usage: python tools/gpu/frame_overhead.py [--elev 35] [--reps 30]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_2306_05051_b200 as pkg  # noqa: E402
from paper_2306_05051_b200 import synth  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elev", type=float, default=35.0)
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    ctx = pkg.Context(0)
    fr = synth.c2(a.elev, device="cuda")
    F = 10
    stacked = synth.GBuffer(*[torch.cat([p] * F, 0).contiguous() for p in fr.gbuf.planes()])
    outs = [torch.empty(fr.gbuf.height, fr.gbuf.width, 4, device="cuda") for _ in range(F)]
    gbs = [synth.GBuffer(*[p.clone() for p in fr.gbuf.planes()]) for _ in range(F)]
    big_out = torch.empty(stacked.height, stacked.width, 4, device="cuda")
    t_chain = timed(lambda: pkg.glint_eval_batch(ctx, gbs, [fr.scene] * F, outs=outs), a.reps)
    t_serial = timed(lambda: [pkg.glint_eval(ctx, g, fr.scene, out=o) for g, o in zip(gbs, outs)], a.reps)
    t_one = timed(lambda: pkg.glint_eval(ctx, stacked, fr.scene, out=big_out), a.reps)
    print(f"elev {a.elev}: {F} frames  one launch {t_one:.4f} ms  chained {t_chain:.4f} ms  serial {t_serial:.4f} ms  "
          f"chained overhead {100 * (t_chain / t_one - 1):.2f} %  serial overhead {100 * (t_serial / t_one - 1):.2f} %")
    ok = torch.equal(big_out.view(-1, 4)[: fr.gbuf.height * fr.gbuf.width].view(torch.int32),
                     outs[0].view(-1, 4).view(torch.int32))
    print("stacked frame 0 == chained frame 0:", ok)


if __name__ == "__main__":
    main()
