"""North-star check 3 at scale (Eq. 5-6, Fig. 13): as the number
of flakes per footprint N P grows, the glinty NDF D_P(h) converges to the
smooth D(h): the mean over surface points tends to D(h) and the per-pixel
spread shrinks like 1/sqrt(N P p).

A flat 1024x1024 quad with one isotropic footprint P for every pixel (distinct
object ids: independent seeds), one directional light and view placed so that
the half vector sits at theta_h from the normal. Radiance of the production
kernel; every factor but D_P is the same for all pixels, so L / L_ref = D_P / D(h)
with L_ref the same evaluation at N = 2^40 (D_P -> D(h), Eq. 6).

usage: python tools/gpu/convergence.py [--out gpurun_out/convergence]
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_2306_05051_b200 as pkg  # noqa: E402
from paper_2306_05051_b200 import synth  # noqa: E402

NPS = [1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8]


def quad(n, P, N, alpha, dev):
    iy, ix = torch.meshgrid(torch.arange(n, device=dev, dtype=torch.float64),
                            torch.arange(n, device=dev, dtype=torch.float64), indexing="ij")
    s = math.sqrt(P)
    u, v = torch.frac((ix + 0.37) * 0.618034), torch.frac((iy + 0.71) * 0.414214)
    duv = torch.zeros(n, n, 4, dtype=torch.float64, device=dev)
    duv[..., 0] = s
    duv[..., 3] = s
    mat = torch.tensor([alpha, alpha, N, 0.5], dtype=torch.float64, device=dev).expand(n, n, 4)
    nrm = torch.zeros(n, n, 3, dtype=torch.float64, device=dev)
    nrm[..., 2] = 1.0
    obj = (iy * n + ix).long() * 2654435761
    return synth._pack(u, v, obj, torch.ones_like(u, dtype=torch.bool), duv, nrm,
                       torch.zeros(n, n, 3, dtype=torch.float64, device=dev), mat)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/convergence")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = pkg.Context(0)
    n, P, alpha = 1024, 2.0 ** -10, 0.35
    rows = []
    for ndf in ("ggx", "beckmann"):
        for th in (0.0, 10.0, 20.0, 30.0, 45.0):
            t = math.radians(th)
            # view and light symmetric about h = (sin t, 0, cos t), 5 deg apart
            e = math.radians(5.0)
            wi = (math.sin(t + e), 0.0, math.cos(t + e))
            wo = (math.sin(t - e), 0.0, math.cos(t - e))
            sc = synth.SceneParams(seed=3, ndf=ndf, view_kind="directional", view=wi,
                                   lights=[synth.Light("directional", wo, (1.0, 1.0, 1.0))])
            ref = pkg.glint_eval(ctx, quad(n, P, 2.0 ** 40, alpha, dev), sc)[..., 0].double().mean().item()
            for NP in NPS:
                L = pkg.glint_eval(ctx, quad(n, P, NP / P, alpha, dev), sc)[..., 0].double() / ref
                rows.append(dict(ndf=ndf, theta_h=th, NP=NP, mean_rel=float(L.mean() - 1), spread=float(L.std())))
            print(ndf, th, [f"{r['mean_rel']:+.3f}/{r['spread']:.3f}" for r in rows[-len(NPS):]], flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    L = ["mean D_P / D(h) - 1 (and per-pixel spread std(D_P / D(h))) over 1024^2 independent surface points:", "",
         "| NDF | theta_h | " + " | ".join(f"N P = {x:.0e}" for x in NPS) + " |", "|---|---|" + "---|" * len(NPS)]
    for ndf in ("ggx", "beckmann"):
        for th in (0.0, 10.0, 20.0, 30.0, 45.0):
            rs = [r for r in rows if r["ndf"] == ndf and r["theta_h"] == th]
            L.append(f"| {ndf} | {th:g} | " + " | ".join(f"{r['mean_rel']:+.3f} ({r['spread']:.3f})" for r in rs) + " |")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
