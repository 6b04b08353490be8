"""Workload characterisation asked for by SURVEY §8d: the footprint anisotropy
r histogram of C2 per elevation ("expect 1 ... >> 50; clamped beyond 256") and
the per-frame LOD (log2 footprint area, l_s) histogram of the C5 zoom path.
Input statistics only (fp64 from the synthetic G-buffers; no method
arithmetic): P = |det J|, r = sigma_max / sigma_min of J = [duv/dx | duv/dy].

usage: python tools/gpu/workload_stats.py [--out gpurun_out/workload]
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_2306_05051_b200 import synth  # noqa: E402

R_EDGES = [1, 1.5, 2, 4, 8, 16, 50, 256, float("inf")]


def footprint(gb):
    valid = (gb.uvm[..., 3].view(torch.int32) & 1) == 1
    d = gb.duv[valid].double()
    a = d[:, 0] ** 2 + d[:, 2] ** 2
    b = d[:, 0] * d[:, 1] + d[:, 2] * d[:, 3]
    c = d[:, 1] ** 2 + d[:, 3] ** 2
    P = (d[:, 0] * d[:, 3] - d[:, 1] * d[:, 2]).abs()
    lam = 0.5 * (a + c) + torch.sqrt((0.5 * (a - c)) ** 2 + b * b)
    r = lam / P.clamp_min(1e-300)
    return P, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/workload")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    c2 = []
    for e in synth.C2_ELEVATIONS:
        P, r = footprint(synth.c2(e, device=dev).gbuf)
        edges = torch.tensor(R_EDGES[:-1] + [1e300], dtype=torch.float64, device=dev)
        h = torch.histogram(r.cpu(), bins=edges.cpu())[0].tolist()
        c2.append(dict(elev=e, valid=int(r.numel()), r_hist=h, r_median=float(r.median()), r_max=float(r.max()),
                       log2P_min=float(torch.log2(P).min()), log2P_max=float(torch.log2(P).max())))
        print(c2[-1], flush=True)
    c5 = []
    for f in range(0, 64, 3):
        P, r = footprint(synth.c5(f, device=dev).gbuf)
        ls = torch.floor(torch.log2(P))
        lo, hi = int(ls.min()), int(ls.max())
        hist = torch.bincount((ls - lo).long()).tolist()
        c5.append(dict(frame=f, ls_min=lo, ls_max=hi, ls_hist=hist, ls_median=float(ls.median()),
                       r_median=float(r.median())))
        print(c5[-1], flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as fh:
        json.dump(dict(c2=c2, c5=c5, r_edges=R_EDGES), fh, indent=1)
    L = ["## C2: footprint anisotropy r per elevation (fraction of valid pixels per bin)", "",
         "| elevation | valid px | " + " | ".join(f"[{R_EDGES[i]:g}, {R_EDGES[i + 1]:g})" for i in range(len(R_EDGES) - 1))
         + " | median r | max r | log2 P range |", "|---|---|" + "---|" * (len(R_EDGES) - 1) + "---|---|---|"]
    for row in c2:
        n = max(1, row["valid"])
        L.append(f"| {row['elev']:g} | {row['valid']} | " + " | ".join(f"{x / n:.3f}" for x in row["r_hist"])
                 + f" | {row['r_median']:.2f} | {row['r_max']:.3g} | {row['log2P_min']:.1f} .. {row['log2P_max']:.1f} |")
    L += ["", "## C5: LOD l_s = floor(log2 P) per frame of the zoom path (every 3rd frame)", "",
          "| frame | l_s range | median l_s | median r |", "|---|---|---|---|"]
    for row in c5:
        L.append(f"| {row['frame']} | {row['ls_min']} .. {row['ls_max']} | {row['ls_median']:.0f} | {row['r_median']:.2f} |")
    with open(a.out + ".md", "w") as fh:
        fh.write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
