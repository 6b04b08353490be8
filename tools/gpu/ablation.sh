#!/bin/bash
# section-6 ablation on B200: 48 (method) vs 64 vs 160 draws per pixel-light, C2 and C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_abl.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_abl.log
for cfg in C2 C4; do for d in 48 64 160; do
  st=50; [ $cfg = C4 ] && st=5
  timeout 600 python bench.py --config $cfg --draws $d --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abl_${cfg}_$d.json 2> gpurun_out/abl_${cfg}_$d.err
  python -c "import json; d=json.load(open('gpurun_out/abl_${cfg}_$d.json')); print('$cfg', $d, d['value'], d['ms_per_step'])"
done; done
