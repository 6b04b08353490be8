"""Spatial statistics of the glint field (hash quality at image level): on a
flat 2048x2048 quad with one isotropic pixel footprint P (the method picks
texels of area ~P: one texel per pixel, neighbours sharing simplex vertices),
the radiance field's 2-D autocorrelation must vanish beyond the interpolation
support (adjacent pixels) and show no periodic peak anywhere in the lag plane
(a weak texel hash would repeat). Reports the autocorrelation profile along
x, y and the largest |rho| beyond 16 pixels.

usage: python tools/gpu/spatial_autocorr.py [--out gpurun_out/autocorr]
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


def field(ctx, n=2048, P=2.0 ** -20, N=2.0 ** 22, alpha=0.3, seed=5, dev="cuda"):
    iy, ix = torch.meshgrid(torch.arange(n, device=dev, dtype=torch.float64),
                            torch.arange(n, device=dev, dtype=torch.float64), indexing="ij")
    s = math.sqrt(P)
    u, v = (ix + 0.5) * s, (iy + 0.5) * s
    duv = torch.zeros(n, n, 4, dtype=torch.float64, device=dev)
    duv[..., 0] = s
    duv[..., 3] = s
    mat = torch.tensor([alpha, alpha, N, 0.3], dtype=torch.float64, device=dev).expand(n, n, 4)
    nrm = torch.zeros(n, n, 3, dtype=torch.float64, device=dev)
    nrm[..., 2] = 1.0
    gb = synth._pack(u, v, torch.zeros_like(u, dtype=torch.int64), torch.ones_like(u, dtype=torch.bool), duv, nrm,
                     torch.zeros(n, n, 3, dtype=torch.float64, device=dev), mat)
    t = math.radians(12.0)
    sc = synth.SceneParams(seed=seed, view_kind="directional", view=(math.sin(t), 0.0, math.cos(t)),
                           lights=[synth.Light("directional", (-math.sin(t) * 0.5, 0.2, 0.9), (1.0, 1.0, 1.0))])
    return pkg.glint_eval(ctx, gb, sc)[..., 0].double()


def autocorr(L):
    x = L - L.mean()
    F = torch.fft.rfft2(x)
    ac = torch.fft.irfft2(F * F.conj(), s=x.shape)
    return ac / ac[0, 0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/autocorr")
    a = ap.parse_args()
    ctx = pkg.Context(0)
    L = field(ctx)
    ac = autocorr(L)
    n = ac.shape[0]
    lag = torch.arange(n, device=ac.device)
    d = torch.minimum(lag, n - lag)
    dist = torch.sqrt(d[:, None].double() ** 2 + d[None, :].double() ** 2)
    far = ac[dist > 16]
    prof_x = ac[0, :33].tolist()
    prof_y = ac[:33, 0].tolist()
    res = dict(glint_fraction=float((L > 0).double().mean()), rho_x=prof_x, rho_y=prof_y,
               max_abs_rho_beyond_16px=float(far.abs().max()), rms_rho_beyond_16px=float(far.pow(2).mean().sqrt()),
               noise_level=1.0 / n)
    print(json.dumps({k: v for k, v in res.items() if not isinstance(v, list)}), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    lines = ["| lag (px) | " + " | ".join(str(i) for i in (0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32)) + " |",
             "|---|" + "---|" * 11]
    for name, pr in (("rho along x", prof_x), ("rho along y", prof_y)):
        lines.append(f"| {name} | " + " | ".join(f"{pr[i]:+.3f}" for i in (0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32)) + " |")
    lines += ["", f"max |rho| beyond 16 px over the whole 2048^2 lag plane: {res['max_abs_rho_beyond_16px']:.4f} "
              f"(rms {res['rms_rho_beyond_16px']:.5f}; 1/n = {1 / n:.5f}); glinting pixels {res['glint_fraction']:.3f}"]
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
