"""Re-check of one Fig. 9 cell on CPU with the oracle (bit-identical to the
device draws): for many seeds of the fig9.py G-buffer recipe (isotropic
footprint 2^-12, N = n 2^12, p = R, distinct object ids per pixel), the
pooled chi-square p-value of a pixel's 12 draws against the contract's exact
gated law must be uniform if the draws of a pixel are independent; also the
mean node-pair / texel-pair count correlation. Used for profiles/r1_gpu_stats.md
(the n = 128, p = 0.05 cell).

usage: python tests/harness/fig9_cell_cpu.py [--n 128] [--p 0.05] [--seeds 2000]
"""
import argparse
import math
import os
import sys

import numpy as np
import torch
from scipy import stats as st

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import stats  # noqa: E402
from paper_2306_05051_b200 import synth  # noqa: E402

S30, C30 = math.sin(math.radians(30)), math.cos(math.radians(30))


def gbuffer(M, n, R, seed):
    """The fig9.py recipe on CPU tensors."""
    H, W = M // 1024, 1024
    g = torch.Generator().manual_seed(seed)
    duv = torch.zeros(H, W, 4)
    duv[..., 0] = 1 / 64
    duv[..., 3] = 1 / 64
    uvm = torch.zeros(H, W, 4)
    uvm[..., :2] = torch.rand(H, W, 2, generator=g)
    obj = torch.arange(H * W, dtype=torch.int64).reshape(H, W) * 2654435761 + seed * 1000003
    uvm[..., 2] = synth._bits_to_f32(obj)
    uvm[..., 3] = synth._bits_to_f32(torch.ones(H, W, dtype=torch.int64))
    nrm = torch.zeros(H, W, 4)
    nrm[..., 2] = 1.0
    mat = torch.tensor([0.3, 0.3, n * 4096.0, R]).expand(H, W, 4).contiguous()
    return synth.GBuffer(duv, uvm.contiguous(), nrm, torch.zeros(H, W, 4), mat)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--p", type=float, default=0.05)
    ap.add_argument("--seeds", type=int, default=2000)
    ap.add_argument("--pixels", type=int, default=1 << 18)
    a = ap.parse_args()
    pooled, node_c, texel_c = [], [], []
    for seed in range(a.seeds):
        sc = synth.SceneParams(seed=1 + seed, ndf="ggx", view_kind="directional", view=(S30, 0.0, C30),
                               lights=[synth.Light("directional", (-S30, 0.0, C30), (1.0, 1.0, 1.0))])
        _, _, rec = oracle.eval(gbuffer(a.pixels, a.n, a.p, 1000 + seed), sc, debug=True)
        r = rec[:, 0]
        law, _ = stats.gated_pmf_enumerated(float(r["n"][0, 0]), float(r["p"][0]))
        c = r["count"][:, :12].astype(np.int64)
        pooled.append(stats.chi2_gof(np.bincount(c.ravel(), minlength=len(law)), law))
        if seed < 40:
            c3 = c.reshape(-1, 3, 4).astype(np.float64)
            for k in range(3):
                m = np.corrcoef(c3[:, k, :].T)
                node_c += [m[i, j] for i in range(4) for j in range(i + 1, 4)]
            for j in range(4):
                m = np.corrcoef(c3[:, :, j].T)
                texel_c += [m[i, k] for i in range(3) for k in range(i + 1, 3)]
    ps = np.array(pooled)
    print(f"cell n={a.n} p={a.p}: {len(ps)} seeds x {a.pixels} pixels x 12 draws")
    print(f"pooled chi2 p: frac<0.01 {np.mean(ps < 0.01):.4f} (SE {math.sqrt(0.0099 / len(ps)):.4f}), "
          f"frac<0.001 {np.mean(ps < 0.001):.4f}, KS uniformity p {st.kstest(ps, 'uniform').pvalue:.3g}")
    for nm, v in (("node-pair", np.array(node_c)), ("texel-pair", np.array(texel_c))):
        print(f"{nm} count corr: mean {v.mean():+.5f} +- {v.std() / math.sqrt(len(v)):.5f}, max |corr| {np.abs(v).max():.4f}")


if __name__ == "__main__":
    main()
