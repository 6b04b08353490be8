#!/bin/bash
# section-6 ablation on B200: 48 (method) vs 64 vs 160 draws per pixel-light, and the
# Zirr & Kaplanyan-style baseline, on C2 and C4
mkdir -p gpurun_out
for cfg in C2 C4; do for v in "48 ours" "64 ours" "160 ours" "48 zk"; do
  set -- $v; d=$1; m=$2
  st=50; [ $cfg = C4 ] && st=5
  timeout 900 python bench.py --config $cfg --draws $d --method $m --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abl_${cfg}_${d}_$m.json 2> gpurun_out/abl_${cfg}_${d}_$m.err
  python -c "import json; d=json.loads(open('gpurun_out/abl_${cfg}_${d}_$m.json').read().strip().splitlines()[-1]); print('$cfg', $d, '$m', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
