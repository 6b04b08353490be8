"""Fig. 9 analogue over an (n, p) grid on the device (
P:L933-972): for each cell, 2^18 pixels x 12 draws of the gated Gaussian
binomial (DEBUG records, production arithmetic), compared with the contract's
exact gated law (chi-square, enumerated by oracle/stats.py) and with the
exact Binomial(n, p) (total variation: the approximation error Fig. 9 shows).

usage: python tests/harness/fig9.py [--out gpurun_out/fig9]
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

NS = [1, 2, 4, 8, 16, 32, 64, 128, 1024]
PS = [0.01, 0.05, 0.1, 0.3, 0.5, 0.7, 0.95]
S30, C30 = math.sin(math.radians(30)), math.cos(math.radians(30))


def gbuffer(M, n, R, seed):
    """Isotropic footprint P = 2^-12 (one grid, h = n: p = R), N = n 2^12."""
    H, W = M // 1024, 1024
    g = torch.Generator(device="cuda").manual_seed(seed)
    duv = torch.zeros(H, W, 4, device="cuda")
    duv[..., 0] = 1 / 64
    duv[..., 3] = 1 / 64
    uvm = torch.zeros(H, W, 4, device="cuda")
    uvm[..., :2] = torch.rand(H, W, 2, generator=g, device="cuda")
    obj = torch.arange(H * W, dtype=torch.int64, device="cuda").reshape(H, W) * 2654435761 + seed * 1000003
    uvm[..., 2] = synth._bits_to_f32(obj)
    uvm[..., 3] = synth._bits_to_f32(torch.ones(H, W, dtype=torch.int64, device="cuda"))
    nrm = torch.zeros(H, W, 4, device="cuda")
    nrm[..., 2] = 1.0
    mat = torch.tensor([0.3, 0.3, n * 4096.0, R], device="cuda").expand(H, W, 4).contiguous()
    return synth.GBuffer(duv, uvm.contiguous(), nrm, torch.zeros(H, W, 4, device="cuda"), mat)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/fig9")
    a = ap.parse_args()
    ctx = pkg.Context(0)
    sc = synth.SceneParams(seed=1, ndf="ggx", view_kind="directional", view=(S30, 0.0, C30),
                           lights=[synth.Light("directional", (-S30, 0.0, C30), (1.0, 1.0, 1.0))])
    cells = []
    for i, n in enumerate(NS):
        for j, p in enumerate(PS):
            _, rec = pkg.glint_eval(ctx, gbuffer(1 << 18, n, p, 1000 + 10 * i + j), sc, debug=True)
            r = rec[:, 0]
            pe = float(r["p"][0])
            c = r["count"][:, :12].ravel().astype(np.int64)
            law, _ = stats.gated_pmf_enumerated(float(r["n"][0, 0]), pe)
            h = np.bincount(c, minlength=len(law))
            cells.append(dict(n=n, p=p, p_device=pe, draws=int(c.size),
                              chi2_p=stats.chi2_gof(h, law),
                              tv_contract=stats.total_variation(h / h.sum(), law),
                              tv_binomial=stats.total_variation(h / h.sum(), stats.binom_pmf(n, pe)),
                              mean=float(c.mean()), binom_mean=n * pe))
            print(cells[-1], flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump(cells, f, indent=1)
    L = ["TV(device draws, exact Binomial(n, p)) -- the gated approximation's error (Fig. 9); each cell "
         f"{cells[0]['draws']:.2e} draws:", "",
         "| n \\ p | " + " | ".join(f"{p:g}" for p in PS) + " |", "|---|" + "---|" * len(PS)]
    for n in NS:
        L.append(f"| {n} | " + " | ".join(f"{c['tv_binomial']:.3f}" for c in cells if c["n"] == n) + " |")
    ps = np.array([c["chi2_p"] for c in cells])
    L += ["", f"Device draws vs the contract's exact gated law: chi-square p-values over the {len(cells)} cells: "
          f"min {ps.min():.3g}, median {np.median(ps):.3g}; max TV {max(c['tv_contract'] for c in cells):.4f}."]
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
