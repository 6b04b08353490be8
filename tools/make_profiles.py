"""Summarise an ncu --set full capture (+ optional launch list) into profiles/.

usage: python tools/make_profiles.py <report.ncu-rep> <tag> [launches.csv] [--pix N --json PATH --launch TEXT]
writes profiles/ncu_summary.json (the C2 frame's full capture; bench.py reads
its FP32 op counts) or --json PATH for another config's frame (--pix = its
pixels), and profiles/<tag>_ncu.md (human summary)."""
import csv
import io
import json
import os
import subprocess
import sys

args = sys.argv[1:]
opts = {}
for k in ("--pix", "--json", "--launch", "--skip"):
    if k in args:
        i = args.index(k)
        opts[k] = args[i + 1]
        del args[i:i + 2]
rep, tag = args[0], args[1]
launches = args[2] if len(args) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
units = dict(zip(h, u))


def f(k):
    try:
        return float(d[k])
    except (KeyError, ValueError):
        return None


def to_bytes(k):
    x = f(k)
    s = units.get(k, "")
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(s, 1) if x is not None else None


PIX = int(opts.get("--pix", 1920 * 1080))   # default: one C2 frame (bench --steps 1 --warmup 3, -s 3 -c 1)
OUT_JSON = opts.get("--json", "profiles/ncu_summary.json")
LAUNCH = opts.get("--launch", "one C2 1920x1080 frame (elevation 35 deg), bench.py --steps 1 --warmup 3")
rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
tinst = f("sass__thread_inst_executed_true_per_opcode") or f("smsp__thread_inst_executed.sum")
dur_ns = f("gpu__time_duration.sum") * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
                                         "second": 1e9, "s": 1e9}.get(
    units.get("gpu__time_duration.sum", "nsecond"), 1)
summary = {
    "source": os.path.basename(rep), "tag": tag, "launch": LAUNCH,
    "pixels_per_launch": PIX,
    "gpu_time_us": dur_ns / 1e3,
    "sm_clock_ghz": f("sm__cycles_elapsed.avg.per_second"),
    "dram_read_bytes": rd, "dram_write_bytes": wr,
    "dram_bytes_per_launch_per_pixel": (rd + wr) / PIX,
    "sass_thread_inst_per_launch": tinst,
    "sass_thread_inst_per_pixel": tinst / PIX,
    "warp_inst_per_launch": f("smsp__inst_executed.sum"),
    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "pipe_alu_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "pipe_fma_pct": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "pipe_xu_pct": f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    "pipe_lsu_pct": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
    "stalls_per_issue": {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: f(k)
                         for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                         and k.endswith("_per_issue_active.ratio") and (f(k) or 0) >= 0.05},
}
# FP32 arithmetic: FFMA = 2 flops; vs 2 x 128 lanes x SMs x f
ffma = f("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum")
fadd = f("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum")
fmul = f("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum")
if None not in (ffma, fadd, fmul):
    flop = 2 * ffma + fadd + fmul
    sms = f("device__attribute_multiprocessor_count") or 148
    clk = (summary["sm_clock_ghz"] or 1.965) * 1e9     # ncu reports GHz
    summary["fp32_flop_per_pixel"] = flop / PIX
    summary["fp32_tflops"] = flop / (dur_ns * 1e-9) / 1e12
    summary["fp32_frac_of_peak_at_clock"] = flop / (dur_ns * 1e-9) / (2 * 128 * sms * clk)
os.makedirs("profiles", exist_ok=True)
with open(OUT_JSON, "w") as fh:
    json.dump(summary, fh, indent=1)
lines = [f"# ncu summary `{tag}` ({os.path.basename(rep)})", "",
         "Captured with `ncu --set full --clock-control none --import-source on -k regex:glint_eval_kernel -s " + opts.get("--skip", "3") + " -c 1` (tools/gpu/r2_full.sh)",
         f"on {LAUNCH}.", "",
         "| metric | value |", "|---|---|"]
for k, val in summary.items():
    if k != "stalls_per_issue":
        lines.append(f"| {k} | {val} |")
lines += ["", "Warp stalls per issued instruction (>= 0.05):", ""]
lines += [f"- {k}: {val:.3f}" for k, val in sorted(summary["stalls_per_issue"].items(), key=lambda kv: -kv[1])]
if launches and os.path.exists(launches):
    txt = open(launches).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:]))) if i >= 0 else []
    if rows:
        hh = rows[0]
        ki, mi, vi = hh.index("Kernel Name"), hh.index("Metric Name"), hh.index("Metric Value")
        per = {}
        for r in rows[1:]:
            if len(r) > vi and r[mi] == "gpu__time_duration.sum":
                per.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
        tot = sum(sum(x) for x in per.values())
        cmdf = launches.replace(".csv", ".cmd")
        nvtx = os.path.exists(cmdf) and "--nvtx-include" in open(cmdf).read()
        if os.path.exists(cmdf):
            lines += ["", "Launch-list command: `" + open(cmdf).read().strip() + "`"]
        lines += ["", "Launch list (ncu `--metrics gpu__time_duration.sum --clock-control none`, cold-cache, "
                  "serialised" + (", timed region only: `--nvtx --nvtx-include glint_timed/`" if nvtx else "") + "):", "",
                  "| kernel | launches | total us | mean us/launch | share |", "|---|---|---|---|---|"]
        for k, x in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(x)} | {sum(x) / 1e3:.1f} | {sum(x) / 1e3 / len(x):.1f} | "
                         f"{100 * sum(x) / tot:.1f}% |")
        with open(f"profiles/{tag}_launches.csv", "w") as fh:
            fh.write(txt[i:])
with open(f"profiles/{tag}_ncu.md", "w") as fh:
    fh.write("\n".join(lines) + "\n")
print("\n".join(lines))
