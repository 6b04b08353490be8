"""Table 1 analogue on B200: milliseconds per 1920x1080 frame of
the glint evaluation for the paper's method ("ours", 48 draws) and the
Zirr & Kaplanyan-style baseline ("zk"), on synthetic
stand-ins for the paper's scenes -- a screen-filling plane facing (90 deg) and
grazing (25 deg), and 32 spheres on a plane -- all with Beckmann alpha = 1.0 and
one light, sweeping the microfacet density N (uniform per frame). Reports, like
Table 1, the min and max time over the density sweep. Kernel time only (CUDA
events on the launch stream, inputs resident, after warm-up).

usage: python tools/gpu/table1.py [--out gpurun_out/table1] [--reps 20]
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

DENSITIES = [2.0 ** k for k in (4, 6, 8, 10, 12, 14, 16, 18, 20)]


def scene_frames(device):
    W, H = 1920, 1080
    out = {}
    for elev in (90, 25):
        fr = synth.c2(elev, W, H, ndf="beckmann", alpha=1.0, device=device)
        out[f"Plane {elev}deg"] = fr
    cam = (0.0, -35.0, 12.0)
    gb = synth.spheres_scene_gbuffer(W, H, cam, (0.0, 0.0, 1.0), 13, device=device)
    sc = synth.SceneParams(seed=1, ndf="beckmann", view_kind="point", view=cam,
                           lights=[synth.Light("point", (10.0, -10.0, 20.0), (900.0,) * 3)])
    out["Spheres"] = synth.Frame("spheres", gb, sc)
    for fr in out.values():
        fr.gbuf.mat[..., 0] = 1.0
        fr.gbuf.mat[..., 1] = 1.0
    return out


def time_frame(ctx, gb, scene, reps):
    st = torch.cuda.current_stream()
    out = torch.empty(gb.height, gb.width, 4, device=gb.duv.device)
    for _ in range(3):
        pkg.glint_eval(ctx, gb, scene, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        pkg.glint_eval(ctx, gb, scene, out=out)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/table1")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = pkg.Context(0)
    frames = scene_frames(dev)
    rows = []
    for name, fr in frames.items():
        valid = fr.gbuf.valid_count()
        for method in ("ours", "zk"):
            fr.scene.method = method
            ts = []
            for N in DENSITIES:
                fr.gbuf.mat[..., 2] = N
                ms = time_frame(ctx, fr.gbuf, fr.scene, a.reps)
                ts.append(ms)
                rows.append(dict(scene=name, method=method, N=N, ms=ms, evals_per_s=valid / (ms * 1e-3)))
            print(f"{name:14s} {method:4s} " + " ".join(f"{t:.3f}" for t in ts), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump(dict(densities=DENSITIES, rows=rows, device=torch.cuda.get_device_name(0)), f, indent=1)
    lines = ["| scene | ours (ms) min - max | zk baseline (ms) min - max | zk max / ours max |", "|---|---|---|---|"]
    for name in frames:
        o = [r["ms"] for r in rows if r["scene"] == name and r["method"] == "ours"]
        z = [r["ms"] for r in rows if r["scene"] == name and r["method"] == "zk"]
        lines.append(f"| {name} | {min(o):.3f} - {max(o):.3f} | {min(z):.3f} - {max(z):.3f} | {max(z) / max(o):.2f} |")
    lines += ["", "Per density (ms per frame):", "",
              "| scene | method | " + " | ".join(f"N=2^{int(math.log2(N))}" for N in DENSITIES) + " |",
              "|---|---|" + "---|" * len(DENSITIES)]
    for name in frames:
        for method in ("ours", "zk"):
            ts = [r["ms"] for r in rows if r["scene"] == name and r["method"] == method]
            lines.append(f"| {name} | {method} | " + " | ".join(f"{t:.3f}" for t in ts) + " |")
    # the C2 workload itself per elevation (GGX alpha 0.2, per-tile density 2^U(8,20)):
    # stable cost vs anisotropy
    lines += ["", "C2 workload per elevation (ms per 1920x1080 frame; valid-pixel evals/s):", "",
              "| elevation | valid px | ours ms | ours evals/s | zk ms | zk evals/s | zk / ours |", "|---|---|---|---|---|---|---|"]
    elev_rows = []
    for e in synth.C2_ELEVATIONS:
        fr = synth.c2(e, device=dev)
        valid = fr.gbuf.valid_count()
        res = {}
        for method in ("ours", "zk"):
            fr.scene.method = method
            res[method] = time_frame(ctx, fr.gbuf, fr.scene, a.reps)
        elev_rows.append(dict(elev=e, valid=valid, **{f"{k}_ms": v for k, v in res.items()}))
        lines.append(f"| {e:g} | {valid} | {res['ours']:.3f} | {valid / res['ours'] / 1e-3:.3e} | {res['zk']:.3f} | "
                     f"{valid / res['zk'] / 1e-3:.3e} | {res['zk'] / res['ours']:.2f} |")
    # the C5 zoom path (1080p, 4 lights): cost along a x10^6 change of footprint area
    lines += ["", "C5 zoom path at 1920x1080, 4 lights (ms per frame; area x10^6 from frame 0 to 63):", "",
              "| frame | ours ms | zk ms | zk / ours |", "|---|---|---|---|"]
    zoom_rows = []
    for f in range(0, 64, 9):
        fr = synth.c5(f, 1920, 1080, device=dev)
        res = {}
        for method in ("ours", "zk"):
            fr.scene.method = method
            res[method] = time_frame(ctx, fr.gbuf, fr.scene, a.reps)
        zoom_rows.append(dict(frame=f, **{f"{k}_ms": v for k, v in res.items()}))
        lines.append(f"| {f} | {res['ours']:.3f} | {res['zk']:.3f} | {res['zk'] / res['ours']:.2f} |")
    o = [r["ours_ms"] for r in zoom_rows]
    z = [r["zk_ms"] for r in zoom_rows]
    lines.append(f"| max / min | {max(o) / min(o):.2f} | {max(z) / min(z):.2f} | |")
    with open(a.out + ".json", "w") as f:
        json.dump(dict(densities=DENSITIES, rows=rows, c2_elevations=elev_rows, c5_zoom=zoom_rows,
                       device=torch.cuda.get_device_name(0)), f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
