#!/usr/bin/env python
"""Benchmark of the glint hot path (BASELINE.json metric: glint shading
evals/s, one eval = one ACTIVE (pixel, light) pair -- a valid pixel with a
non-degenerate footprint and the light above its horizon, the pairs whose
48 gated binomial draws the kernel performs; counted by glint_count_active).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C5|C2|C3|C4] [--gather p2p|nccl]

One step = one pass of the whole hot path (S0-S9) over one
batch of synthetic input. Default workload: C5 (BASELINE.json configs[4]),
the 64-frame 3840x2160 zoom path with 4 point lights, at every N (strong
scaling: the same 64 frames whatever the GPU count). Frames are dealt round-
robin to ranks (frame f on rank f mod N); C2 / C3 at N > 1 deal 64-row bands
instead. The gather of radiance to rank 0 is INSIDE the timed
region: by default fused into the kernels (each rank stores its tiles straight
into rank 0's full-frame buffers over NVLink, CUDA IPC), or with --gather nccl
as per-tile send/recv rounds on a communication stream overlapped with the
next tiles' shading. Inputs are resident in HBM when the timed region starts
and total > 126 MB L2 per rank (no flush needed).

``--gpus N`` without torchrun re-launches itself through torch.distributed.run
with N processes; a world size that differs from N prints no result line.
Prints ONE JSON line on rank 0. ``--impl reference`` times the CPU oracle
(oracle/) on the host cores over the same bounded sample our arm's
cpu_baseline uses.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "glint shading evals/s (pixel x light) at 1/2/4/8 B200; % of FP32 peak"
UNIT = "evals/s"
# Algorithmic work per eval (SURVEY §8d budget): 340 thread
# instructions per pixel (S0-S4a, shared by the L lights) + 1110 per
# (pixel, light) (S5-S9, of which 860 are the 48 draws).
W_PIXEL, W_EVAL = 340.0, 1110.0
# Algorithmic HBM bytes per pixel: 5 float4 planes in + 1 float4 out.
BYTES_PER_PIXEL = 96.0
LANES_PER_SM = 128


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period: float = 0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"], "samples": 0}
        names = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}

    def rejected(self):
        bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
        s = self.summary()
        if set(s["reasons"]) & bad:
            return True
        if s["sm_mhz"] and s["sm_max_mhz"] and s["sm_mhz"] < 0.6 * s["sm_max_mhz"] and not s["reasons"]:
            return True
        return False


# ----------------------------------------------------------------------------- workloads
def _gen(config):
    from paper_2306_05051_b200 import synth
    return {
        "C2": lambda f, win, dev: synth.c2(synth.C2_ELEVATIONS[f], window=win, device=dev),
        "C3": lambda f, win, dev: synth.c3(window=win, device=dev),
        "C4": lambda f, win, dev: synth.c4(f, window=win, device=dev),
        "C5": lambda f, win, dev: synth.c5(f, window=win, device=dev),
    }[config]


# (frames per step, height, width, description); BASELINE.json configs[1..4]
WORKLOADS = {
    "C2": (10, 1080, 1920, "C2: 1920x1080 infinite ground plane, pinhole 60deg FOV, elevations 5..85 + 90 deg "
                           "(10 frames per step), 1 point light, GGX alpha 0.2, N = 2^U(8,20) per uv tile, R = 0.034"),
    "C3": (1, 2160, 3840, "C3: 3840x2160, 32 analytic spheres on a plane, anisotropic GGX alpha U(0.05,0.6), "
                          "N log-U[1e3,1e7], 1 point light (1 frame per step)"),
    "C4": (8, 2160, 3840, "C4: 3840x2160, 32 spheres on a plane, anisotropic GGX alpha U(0.05,0.6), "
                          "N log-U[1e3,1e7], 16 point lights, 8 jittered frames per step"),
    "C5": (64, 2160, 3840, "C5: 64-frame 3840x2160 zoom path (distance 0.5 -> 500, elevation 30 deg) over the "
                           "32-sphere scene, 4 point lights, anisotropic GGX alpha U(0.05,0.6), N log-U[1e3,1e7]"),
}
# the bounded CPU sample shared by cpu_baseline and --impl reference: 8-row
# bands every `period` rows (centred), of the listed frames
SAMPLE = {"C2": (range(10), 16), "C3": ((0,), 16), "C4": (range(8), 256), "C5": (range(0, 64, 4), 270)}


def oracle_sample(config: str):
    """[(GBuffer on CPU, scene)] of the sample and its description."""
    from paper_2306_05051_b200 import synth
    frames, period = SAMPLE[config]
    _, H, W, _ = WORKLOADS[config]
    gen = _gen(config)
    subs = []
    for f in frames:
        parts, sc = [], None
        for y in range(period // 2 - 4, H, period):
            fr = gen(f, (y, min(H, y + 8), 0, W), "cpu")
            parts.append(fr.gbuf)
            sc = fr.scene
        subs.append((synth.GBuffer(*[torch.cat([p.planes()[k] for p in parts], 0) for k in range(5)]), sc))
    nf = len(list(frames))
    desc = f"8-row bands every {period} rows of {nf} frames of {config}" + (" (every 4th frame)" if config == "C5" else "")
    return subs, desc


def time_oracle(subs, threads=None):
    """One pass of the oracle over the sample: (active evals, seconds)."""
    import oracle
    t0 = time.perf_counter()
    ev = 0
    for gb, sc in subs:
        oracle.eval(gb, sc, threads=threads)
    dt = time.perf_counter() - t0
    for gb, sc in subs:
        ev += _active_pairs_oracle(gb, sc)
    return ev, dt


_ACTIVE_CACHE = {}


def _active_pairs_oracle(gb, sc):
    """Active (pixel, light) pairs of a sample part, from the oracle's records
    (light_active), computed once (outside any timing)."""
    import oracle
    key = (id(gb), id(sc))
    if key not in _ACTIVE_CACHE:
        n = 0
        planes = gb.planes()
        H = planes[0].shape[0]
        for y in range(0, H, 8):           # bounded record memory (one 8-row band at a time)
            sub = type(gb)(*[p[y:y + 8] for p in planes])
            _, _, rec = oracle.eval(sub, sc, debug=True)
            n += int(rec["light_active"].sum())
        _ACTIVE_CACHE[key] = n
    return _ACTIVE_CACHE[key]


def host_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def run_reference(args):
    from paper_2306_05051_b200 import dist as D
    rank, world, _ = D.env_rank_world()
    if rank != 0:
        return 0
    _, _, _, desc = WORKLOADS[args.config]
    subs, sample = oracle_sample(args.config)
    for gb, sc in subs:
        sc.draws = args.draws
        sc.method = args.method
        _active_pairs_oracle(gb, sc)
    cores = host_cores()
    for _ in range(args.warmup):
        time_oracle(subs)
    ev_tot, t_tot = 0, 0.0
    for _ in range(args.steps):
        ev, t = time_oracle(subs)
        ev_tot += ev
        t_tot += t
    value = ev_tot / t_tot
    sample = f"{sample} ({ev_tot // args.steps} active evals per step; the same sample as our arm's cpu_baseline)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_tot / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": desc, "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def read_profile_traffic(config):
    """The committed ncu evidence for this config (profiles/ncu_counts_<config>.json,
    tools/ncu_step_counts.py: SASS thread-instructions and DRAM bytes per pixel
    over every launch of a step) and, for C2 / C5, the full capture of one frame
    (profiles/ncu_summary_<config>.json). Returns (DRAM bytes per pixel, counts)."""
    def load(name):
        p = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(p):
            return None
        with open(p) as f:
            return json.load(f)
    counts = load(f"ncu_counts_{config.lower()}.json")
    if counts is None:
        return None, None
    counts["full"] = load(f"ncu_summary_{config.lower()}.json")
    return counts.get("dram_bytes_per_launch_per_pixel"), counts


def measure_h2d_gbs(dev, nbytes=1 << 29, reps=3) -> float:
    """Best-of-3 pinned host -> device copy bandwidth (GB/s, CUDA events)."""
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def run_ours(args):
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import build as B
    from paper_2306_05051_b200 import dist as D
    if int(os.environ.get("RANK", "0")) == 0:
        B.build()
    # GLINT_BENCH_BACKEND=gloo and GLINT_BENCH_DEVICE=<d> exist for the
    # functional test of the N > 1 code path on one GPU
    # (tests/test_bench_contract.py::test_our_arm_two_ranks_one_gpu); a
    # measurement always runs NCCL with one GPU per rank
    backend = os.environ.get("GLINT_BENCH_BACKEND", "nccl")
    rank, world, local = D.init(backend)
    local = int(os.environ.get("GLINT_BENCH_DEVICE", local))
    if world > 1:
        D.barrier()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = pkg.Context(local)
    n_frames, H, W, desc = WORKLOADS[args.config]
    gen = _gen(args.config)
    tiles = D.plan_tiles(n_frames, H, world)
    mine = [i for i in range(len(tiles)) if i % world == rank]
    frames = {}
    for i in mine:
        f, y0, y1 = tiles[i]
        fr = gen(f, (y0, y1, 0, W), dev)
        fr.scene.draws, fr.scene.method = args.draws, args.method
        frames[i] = fr
    if args.draws != 48:
        desc += f"; ABLATION: {args.draws} draws per pixel-light (P:L749/L758)"
    if args.method == "zk":
        desc += "; BASELINE: Zirr & Kaplanyan-style path (DESIGN.md section 10), not the paper's method"
    L = len(next(iter(frames.values())).scene.lights) if frames else 0

    # ---- the metric's unit, counted outside the timed region
    active = {i: pkg.glint_count_active(ctx, fr.gbuf, fr.scene) for i, fr in frames.items()}
    valid = {i: fr.gbuf.valid_count() for i, fr in frames.items()}
    evals = sum(active.values())
    evals_replicated = sum(valid[i] * len(frames[i].scene.lights) for i in frames)
    px = sum(frames[i].gbuf.height * frames[i].gbuf.width for i in frames)

    # ---- outputs: rank 0 owns the step's full frames; the gather is in the timed region
    use_nccl = world > 1 and args.gather == "nccl"
    if use_nccl and backend != "nccl":
        raise SystemExit("--gather nccl needs the NCCL backend")
    comm = torch.cuda.Stream(dev) if use_nccl else None
    if use_nccl:
        full = torch.empty((n_frames, H, W, 4), dtype=torch.float32, device=dev) if rank == 0 else None
        gatherer = D.TileGather(tiles, rank, world, full=full, comm_stream=comm)
        local_outs = {} if rank == 0 else {i: torch.empty((tiles[i][2] - tiles[i][1], W, 4), dtype=torch.float32,
                                                          device=dev) for i in mine}
        outs = [full[tiles[i][0]] if rank == 0 else local_outs[i] for i in mine]
        origins = [(0, tiles[i][1]) if rank == 0 else (0, 0) for i in mine]
    else:
        full = D.peer_buffer((n_frames, H, W, 4), device=dev)     # rank 0's buffer, mapped everywhere
        outs = [full[tiles[i][0]] for i in mine]
        origins = [(0, tiles[i][1]) for i in mine]
    gbs = [frames[i].gbuf for i in mine]
    scenes = [frames[i].scene for i in mine]
    stream = torch.cuda.current_stream(dev)
    comm_done = torch.cuda.Event() if use_nccl else None

    def step(evs=None):
        if use_nccl:
            tile_ev = {}
            for k, i in enumerate(mine):
                pkg.glint_eval_batch(ctx, [gbs[k]], [scenes[k]], outs=[outs[k]], stream=stream, origins=[origins[k]])
                e = torch.cuda.Event()
                e.record(stream)
                tile_ev[i] = e
            works = gatherer.run({i: outs[k] for k, i in enumerate(mine)} if rank != 0 else {}, tile_ev)
            with torch.cuda.stream(comm):
                for w in works:
                    w.wait()
                comm_done.record(comm)
            # the step ends when its gather has landed (and the next step's kernels
            # may then overwrite the local buffers the sends read)
            stream.wait_event(comm_done)
            return
        if evs is None and not args.no_batch:
            # this rank's tiles in one call: launches chained with programmatic
            # dependent launch (tile t+1 fills the SMs tile t frees at its tail)
            pkg.glint_eval_batch(ctx, gbs, scenes, outs=outs, stream=stream, origins=origins)
            return
        for k in range(len(mine)):
            if evs is not None:
                evs[k][0].record(stream)
            pkg.glint_eval(ctx, gbs[k], scenes[k], out=outs[k], stream=stream, origin=origins[k])
            if evs is not None:
                evs[k][1].record(stream)

    args.warmup = max(args.warmup, 3)      # contract: W >= 3
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    D.barrier()

    # per-launch durations of serialised launches (outside the timed region)
    ev_pairs = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in mine]
    if not use_nccl:
        step(ev_pairs)
        torch.cuda.synchronize()
        serial_launch_ms = [a.elapsed_time(b) for a, b in ev_pairs]
    else:
        serial_launch_ms = [float("nan")]
    D.barrier()

    def timed():
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = ctx.launch_count()
        with ClockSampler(local) as clk:
            D.barrier()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_push("glint_timed")   # ncu --nvtx-include "glint_timed/": the step's launches
            start.record(stream)
            for _ in range(args.steps):
                step()
            end.record(stream)
            torch.cuda.nvtx.range_pop()
            torch.cuda.synchronize()
            D.barrier()
        return start.elapsed_time(end), ctx.launch_count() - n0, clk

    ms, launches, clk = timed()
    if clk.rejected():
        ms, launches, clk = timed()
    ms_max = D.max_over_ranks(ms, device=dev)
    ms_rank0 = ms            # printed by rank 0: its own timed region (with NCCL, its last receive)
    evals_all = D.sum_over_ranks(evals, device=dev) * args.steps
    evals_repl_all = D.sum_over_ranks(evals_replicated, device=dev) * args.steps
    launches_all = int(round(D.sum_over_ranks(float(launches), device=dev)))
    value = evals_all / (ms_max / 1e3)

    # ---- verification of the gathered step: rank 0's frames all written, and
    # tiles shaded on other ranks equal rank 0's own evaluation bit for bit
    if rank == 0:
        full.fill_(float("nan"))
        torch.cuda.synchronize()
    D.barrier()
    step()
    torch.cuda.synchronize()
    D.barrier()
    check = None
    if rank == 0:
        assert not torch.isnan(full[..., 3]).any().item(), "a pixel of the gathered frames was never written"
        remote = [i for i in range(len(tiles)) if i % world != 0][:3]
        for i in remote:
            f, y0, y1 = tiles[i]
            fr = gen(f, (y0, y1, 0, W), dev)
            fr.scene.draws, fr.scene.method = args.draws, args.method
            ref = pkg.glint_eval(ctx, fr.gbuf, fr.scene)
            torch.cuda.synchronize()
            if not torch.equal(ref.view(torch.int32), full[f][y0:y1].view(torch.int32)):
                raise SystemExit(f"tile {i} gathered from rank {i % world} differs from rank 0's evaluation")
        check = (f"all {n_frames} frames written at rank 0; {len(remote)} tiles from other ranks "
                 f"re-evaluated on rank 0: bit-identical") if remote else f"all {n_frames} frames written"
    D.barrier()

    # ---- compute-only scaling (N > 1): the same steps with each rank's tiles
    # shaded into local buffers, no gather; max over ranks of the device time
    compute_only = None
    if world > 1:
        louts = [torch.empty((tiles[i][2] - tiles[i][1], W, 4), dtype=torch.float32, device=dev) for i in mine]
        for _ in range(2):
            pkg.glint_eval_batch(ctx, gbs, scenes, outs=louts, stream=stream)
        torch.cuda.synchronize()
        D.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            pkg.glint_eval_batch(ctx, gbs, scenes, outs=louts, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        c_ms = D.max_over_ranks(a.elapsed_time(b), device=dev)
        compute_only = {"value": evals_all / (c_ms / 1e3), "ms_per_step": c_ms / args.steps,
                        "how": "each rank's tiles into local buffers, no gather; max over ranks"}
        del louts

    # ---- roofline of the dominant (only) kernel: issue-bound ALU path
    peaks, peak_src = load_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    issue_peak = sms * LANES_PER_SM * f_max                   # thread-instructions/s
    w_eval = W_EVAL + W_PIXEL / max(L, 1)
    launches_per_step = len(mine)
    # the kernel's average launch duration inside the timed region: the
    # launches are back to back on one stream (chained, so one launch's tail
    # overlaps the next one's start): this rank's step time / its launches
    mean_launch_s = ms / 1e3 / max(launches, 1)
    evals_per_launch = evals / max(launches_per_step, 1)
    achieved = evals_per_launch * w_eval / mean_launch_s
    traffic_pp, prof = read_profile_traffic(args.config)
    px_per_launch = px / max(launches_per_step, 1)
    roofline = {
        "bound": "alu", "achieved": achieved, "peak": issue_peak, "unit": "thread-inst/s",
        "frac": achieved / issue_peak,
        "frac_note": ("W is SURVEY 8d's dense-draw budget; the kernel skips the count work of warp-grids with no "
                      "passing gate (exact: production == DEBUG bit for bit), so it issues fewer instructions than W "
                      "per eval and issue_frac_warp is the measured issue-slot utilisation"),
        "traffic": (traffic_pp * px_per_launch) if traffic_pp else None,
        "peak_source": f"{sms} SMs x 128 lanes x sm_max_mhz {f_max / 1e6:.0f} ({peak_src} MEASURED_PEAKS.json)",
        "algorithmic_inst_per_eval": w_eval,
        "evals_per_launch": evals_per_launch,
        "hbm_achieved_gbs": BYTES_PER_PIXEL * px_per_launch / mean_launch_s / 1e9,
        "hbm_frac": BYTES_PER_PIXEL * px_per_launch / mean_launch_s / 1e9 / float(peaks.get("hbm_gbs", 6458.7)),
        "mean_launch_ms": mean_launch_s * 1e3,
        "launch_ms_basis": "rank 0's timed region / its launches (glint_eval_batch: chained launches)",
        "serial_median_launch_ms": float(np.nanmedian(serial_launch_ms)) if not use_nccl else None,
        "serial_min_launch_ms": float(np.nanmin(serial_launch_ms)) if not use_nccl else None,
    }
    if prof and prof.get("sass_thread_inst_per_pixel") and args.draws == 48 and args.method == "ours":
        roofline["sass_thread_inst_per_pixel"] = prof["sass_thread_inst_per_pixel"]
        roofline["issue_frac_sass"] = px_per_launch * prof["sass_thread_inst_per_pixel"] / mean_launch_s / issue_peak
        if prof.get("warp_inst_per_pixel"):
            roofline["warp_inst_per_pixel"] = prof["warp_inst_per_pixel"]
            roofline["issue_frac_warp"] = px_per_launch * prof["warp_inst_per_pixel"] / mean_launch_s / (sms * 4 * f_max)
        roofline["traffic_source"] = (f"profiles/ncu_counts_{args.config.lower()}.json ({prof.get('source')}, "
                                      f"{prof.get('launches')} launches: every frame of a step)")
        full_cap = prof.get("full")
        if full_cap and full_cap.get("fp32_flop_per_pixel") and full_cap.get("sass_thread_inst_per_pixel"):
            fl_pp = (full_cap["fp32_flop_per_pixel"] * prof["sass_thread_inst_per_pixel"]
                     / full_cap["sass_thread_inst_per_pixel"])
            fl = px_per_launch * fl_pp / mean_launch_s
            roofline["fp32_tflops"] = fl / 1e12
            roofline["fp32_frac"] = fl / (2 * sms * LANES_PER_SM * f_max)
    cs = clk.summary()
    if cs.get("sm_mhz"):
        roofline["frac_at_measured_clock"] = achieved / (sms * LANES_PER_SM * cs["sm_mhz"] * 1e6)

    # ---- end to end through the public C ABI with host buffers (each rank
    # its own tiles: pinned host G-buffers in, host radiance out)
    e2e = None
    if not args.no_e2e:
        sub = mine[:args.e2e_tiles if args.e2e_tiles else (4 if H >= 2160 else 10)]
        hosts = [frames[i].gbuf.to("cpu").pin() for i in sub]
        houts = [torch.empty((frames[i].gbuf.height, W, 4), dtype=torch.float32).pin_memory() for i in sub]
        e_px = sum(frames[i].gbuf.height * W for i in sub)
        e_ev = sum(active[i] for i in sub)
        n_e2e = max(1, min(args.steps, args.e2e_steps))
        e_scenes = [frames[i].scene for i in sub]

        def e2e_step():
            if args.no_batch:
                for hb, sc, ho in zip(hosts, e_scenes, houts):
                    pkg.glint_eval_host(ctx, hb, sc, out=ho)
            else:   # one call per step: the copy/compute pipeline runs across the tiles
                pkg.glint_eval_host_batch(ctx, hosts, e_scenes, outs=houts)
        e2e_step()
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        torch.cuda.synchronize()
        t_e2e = D.max_over_ranks(time.perf_counter() - t0, device=dev)
        e2e = {"value": D.sum_over_ranks(e_ev * n_e2e, device=dev) / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(D.sum_over_ranks(e_px * 80, device=dev)),
               "d2h_bytes_per_step": int(D.sum_over_ranks(e_px * 16, device=dev)),
               "steps": n_e2e, "api": ("glint_eval_host" if args.no_batch else "glint_eval_host_batch")
               + " (pinned host G-buffers -> host radiance), every rank on its own tiles",
               "sample": f"first {len(sub)} of each rank's {len(mine)} tiles (host pinned memory bound)"}
        h2d_peak = measure_h2d_gbs(dev)
        e2e["h2d_gbs_achieved"] = e_px * 80 * n_e2e / t_e2e / 1e9
        e2e["h2d_gbs_measured_peak"] = h2d_peak
        e2e["h2d_frac"] = e2e["h2d_gbs_achieved"] / h2d_peak
        # sanity: host path reproduces the device path bit for bit
        ref0 = pkg.glint_eval(ctx, gbs[0], scenes[0])
        torch.cuda.synchronize()
        if not torch.equal(houts[0].view(torch.int32), ref0.cpu().view(torch.int32)):
            raise SystemExit("host-buffer entry output differs from glint_eval")
        del hosts, houts

    # ---- CPU baseline (oracle on host cores, the same sample as --impl reference), rank 0 at N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        subs, sample = oracle_sample(args.config)
        for gb, sc in subs:
            sc.draws, sc.method = args.draws, args.method
        ev, t = time_oracle(subs)
        cpu = {"value": ev / t, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
               "sample": f"{sample} ({ev} active evals, {t:.1f} s wall, {t * host_cores():.0f} core-s)"}
        # the single-core figure beside the all-core one (the first frame's part of the sample)
        ev1, t1 = time_oracle(subs[:1], threads=1)
        cpu["value_1core"] = ev1 / t1
        cpu["sample_1core"] = f"the first frame's bands of the sample, 1 thread ({ev1} active evals, {t1:.1f} s)"

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "pixels_per_step_per_rank": px,
                       "evals_per_step_per_rank": evals,
                       "evals_replicated_per_step_per_rank": evals_replicated,
                       "evals_note": "evals = active (pixel, light) pairs (glint_count_active: valid pixel, "
                                     "non-degenerate footprint, light above the horizon, R-27b); replicated = "
                                     "valid pixels x lights",
                       "value_replicated_pairs": evals_repl_all / (ms_max / 1e3),
                       "lights": L, "tiles_per_step": len(tiles), "launches_per_step_per_rank": launches_per_step,
                       "launch_path": ("glint_eval (one launch per tile)" if args.no_batch else
                                       "glint_eval_batch (one call per step and rank; tiles chained by "
                                       "programmatic dependent launch)") if not use_nccl else
                                      "glint_eval_batch per tile + an event, NCCL round per tile",
                       "l2": "inputs > 126 MB L2 per rank: no flush between steps",
                       "parallelism": (f"{len(tiles)} tiles ({'whole frames' if tiles[0][2] - tiles[0][1] == H else '64-row bands'}) "
                                       f"dealt round-robin to {world} ranks"),
                       "gather": ("none (one rank: the frames are shaded in place)" if world == 1 else
                                  "fused: the kernels store every tile into rank 0's full frames (CUDA IPC peer "
                                  "memory over NVLink), inside the timed region" if not use_nccl else
                                  "NCCL grouped send/recv per tile round on a comm stream, each send after its "
                                  "tile's kernel event, inside the timed region"),
                       "verified": check, "rank0_ms_per_step": ms_rank0 / args.steps,
                       **({"compute_only": compute_only} if compute_only else {})},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_all,
            "clocks": cs, "gpu": props.name,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--method", default="ours", choices=["ours", "zk"],
                    help="ours = the paper's method; zk = the Zirr & Kaplanyan-style baseline (eval_mode 3)")
    ap.add_argument("--gather", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: fuse the gather to rank 0 into the kernels (peer stores) or NCCL per tile")
    ap.add_argument("--draws", type=int, default=48, choices=[48, 64, 160],
                    help="draws per pixel-light: 48 = the method; 64 / 160 = its section-6 ablations")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-tiles", type=int, default=0,
                    help="tiles per rank in the host-buffer (e2e) leg (default: 4 of a 4K config, else 10)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-batch", action="store_true",
                    help="one glint_eval per tile instead of one glint_eval_batch per step (A/B)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch through torchrun
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}: refusing to report\n")
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
