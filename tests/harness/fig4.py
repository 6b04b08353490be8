"""Fig. 4 at scale ("M scaled from 10^4 to 10^8").

N = 64 flakes per unit area, p = 1/2, footprint area 0.375 between the LOD
areas 0.25 and 0.5: the method distributes the trials, b(8) +
b(16) per (texel, angular node) pair of the two grids (Eq. 10); Zirr &
Kaplanyan blend the outputs of full-LOD draws (Eq. 7). The device's draws
(DEBUG records, production arithmetic) are accumulated over chunks of 2^20
pixels with distinct object ids (independent seeds) up to ~10^8 draws and
compared, at M = 10^4 .. 10^8, with the contract's exact law (the convolution
of the two enumerated gated laws, oracle/stats.py) and with Binomial(24, 1/2).

usage: python tests/harness/fig4.py [--out gpurun_out/fig4] [--chunks 8]
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2306_05051_b200 as pkg  # noqa: E402
from paper_2306_05051_b200 import synth  # noqa: E402
from oracle import stats  # noqa: E402

S30, C30 = math.sin(math.radians(30)), math.cos(math.radians(30))


def gbuffer(M, P, N, R, seed):
    H, W = M // 1024, 1024
    g = torch.Generator(device="cuda").manual_seed(seed)
    s = math.sqrt(P)
    duv = torch.zeros(H, W, 4, device="cuda")
    duv[..., 0] = s
    duv[..., 3] = s
    uvm = torch.zeros(H, W, 4, device="cuda")
    uvm[..., :2] = torch.rand(H, W, 2, generator=g, device="cuda")
    obj = torch.arange(H * W, dtype=torch.int64, device="cuda").reshape(H, W) * 2654435761 + seed * 1000003
    uvm[..., 2] = synth._bits_to_f32(obj)
    uvm[..., 3] = synth._bits_to_f32(torch.ones(H, W, dtype=torch.int64, device="cuda"))
    nrm = torch.zeros(H, W, 4, device="cuda")
    nrm[..., 2] = 1.0
    mat = torch.tensor([0.3, 0.3, N, R], device="cuda").expand(H, W, 4).contiguous()
    return synth.GBuffer(duv, uvm.contiguous(), nrm, torch.zeros(H, W, 4, device="cuda"), mat)


def scene():
    return synth.SceneParams(seed=1, ndf="ggx", view_kind="directional", view=(S30, 0.0, C30),
                             lights=[synth.Light("directional", (-S30, 0.0, C30), (1.0, 1.0, 1.0))])


def slot_counts(ctx, gb, sc, want=None):
    _, rec = pkg.glint_eval(ctx, gb, sc, debug=True)
    r = rec[:, 0]
    n = r["n"][0]
    slots = [int(i) for i in np.nonzero(n > 0)[0]] if want is None else want
    return r, slots


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/fig4")
    ap.add_argument("--chunks", type=int, default=8)
    a = ap.parse_args()
    ctx = pkg.Context(0)
    sc = scene()
    M = 1 << 20
    hist_d = np.zeros(64, np.int64)
    hist_z = np.zeros(256, np.int64)        # Zirr blend, in units of 1/2 count
    samples_d, samples_z = [], []
    law = None
    for ch in range(a.chunks):
        r, slots = slot_counts(ctx, gbuffer(M, 0.375, 64.0, 0.5, 100 + ch), sc)
        n = r["n"][0]
        assert sorted(np.round(n[n > 0], 4).tolist()) == [8.0, 16.0]
        p = float(r["p"][0])
        if law is None:
            law = np.convolve(stats.gated_pmf_enumerated(float(n[slots[0]]), p)[0],
                              stats.gated_pmf_enumerated(float(n[slots[1]]), p)[0])
        d = (r["count"][:, slots[0] * 12:(slots[0] + 1) * 12] + r["count"][:, slots[1] * 12:(slots[1] + 1) * 12])
        d = d.ravel().astype(np.int64)
        hist_d += np.bincount(d, minlength=64)[:64]
        samples_d.append(d[:2_000_000])
        # Zirr (Eq. 7): mix of full-LOD draws at areas 0.5 and 0.25, weight 1/2
        rh, sh = slot_counts(ctx, gbuffer(M, 0.5, 64.0, 0.5, 900 + ch), sc)
        rl, sl = slot_counts(ctx, gbuffer(M, 0.25, 64.0, 0.5, 900 + ch), sc)
        ih, il = int(np.argmax(rh["n"][0])), int(np.argmax(rl["n"][0]))
        z2 = (rh["count"][:, ih * 12:(ih + 1) * 12] + rl["count"][:, il * 12:(il + 1) * 12]).ravel().astype(np.int64)
        hist_z += np.bincount(z2, minlength=256)[:256]
        samples_z.append(z2[:2_000_000])
        print(f"chunk {ch}: {hist_d.sum():.3e} distributed draws", flush=True)
    sd = np.concatenate(samples_d)
    sz = np.concatenate(samples_z)
    binom = stats.binom_pmf(24, 0.5)
    rows = []
    for m in (10 ** 4, 10 ** 5, 10 ** 6, 10 ** 7, int(hist_d.sum())):
        if m <= len(sd):
            hd = np.bincount(sd[:m], minlength=64)[:64]
            hz = np.bincount(sz[:m], minlength=256)[:256]
        else:
            hd, hz = hist_d, hist_z
            m = int(hist_d.sum())
        k = np.arange(64)
        mean = float((hd * k).sum() / hd.sum())
        var = float((hd * k * k).sum() / hd.sum() - mean ** 2)
        kz = np.arange(256) / 2.0
        mz = float((hz * kz).sum() / hz.sum())
        vz = float((hz * kz * kz).sum() / hz.sum() - mz ** 2)
        rows.append(dict(M=m, mean=mean, var=var, chi2_p_exact_law=stats.chi2_gof(hd, law),
                         tv_exact_law=stats.total_variation(hd / hd.sum(), law),
                         tv_binom24=stats.total_variation(hd / hd.sum(), binom),
                         zirr_mean=mz, zirr_var=vz))
        print(rows[-1], flush=True)
    lm = stats.pmf_mean(law)
    lv = float(np.dot((np.arange(len(law)) - lm) ** 2, law))
    out = dict(law_mean=lm, law_var=lv, binom24_mean=12.0, binom24_var=6.0, rows=rows)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    L = [f"Exact contract law (gated b(8) * gated b(16), p = 1/2): mean {lm:.4f}, variance {lv:.4f}; "
         "Binomial(24, 1/2): mean 12, variance 6.", "",
         "| M (draws) | distributed mean | variance | chi2 p vs exact law | TV vs exact law | TV vs Bin(24, 1/2) "
         "| Zirr blend mean | Zirr blend variance |", "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        L.append(f"| {r['M']:.0e} | {r['mean']:.4f} | {r['var']:.4f} | {r['chi2_p_exact_law']:.3g} | "
                 f"{r['tv_exact_law']:.5f} | {r['tv_binom24']:.4f} | {r['zirr_mean']:.4f} | {r['zirr_var']:.4f} |")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
