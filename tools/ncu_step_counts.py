"""Per-config instruction and DRAM counts over one whole bench step (every
frame's launch), for the bench lines whose workload varies across frames
(C5's zoom path) or which the full C2 capture does not cover (C4, C5).

Input: an ncu CSV of the serialised per-frame launches that bench.py runs
outside its timed region (`--metrics smsp__thread_inst_executed_pred_on.sum,
smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum -s <warmup x frames> -c <frames>`).
Output: profiles/ncu_counts_<config>.json (read by bench.py: issue_frac_sass).

usage: python tools/ncu_step_counts.py <ncu.csv> <C2|C4|C5> [cmd-file]
"""
import csv
import io
import json
import os
import sys

PIX = {"C2": 1920 * 1080, "C4": 3840 * 2160, "C5": 3840 * 2160}


def main():
    path, cfg = sys.argv[1], sys.argv[2]
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    h = rows[0]
    ii, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        per.setdefault(r[ii], {})[r[mi]] = v
    n = len(per)
    tot = {k: sum(d.get(k, 0.0) for d in per.values()) for k in next(iter(per.values()))}
    px = PIX[cfg] * n
    out = {
        "config": cfg, "launches": n, "pixels": px,
        "sass_thread_inst_per_pixel": tot["smsp__thread_inst_executed_pred_on.sum"] / px,
        "warp_inst_per_pixel": tot["smsp__inst_executed.sum"] / px,
        "dram_bytes_per_launch_per_pixel": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / px,
        "serial_time_us_total": tot["gpu__time_duration.sum"] / 1e3,
        "source": os.path.basename(path),
        "command": open(sys.argv[3]).read().strip() if len(sys.argv) > 3 else None,
    }
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/ncu_counts_{cfg.lower()}.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
