#!/bin/bash
# Bench each variant library under variants/ (built with build.py --out ... -D ...) on C2 and C4.
# usage: bash tools/gpu/sweep.sh [lib ...]
mkdir -p gpurun_out
libs=${@:-variants/*.so}
for l in paper_2306_05051_b200/libglint.so $libs; do
  for cfg in C2 C4; do
    n=$(basename $l .so)_$cfg
    GLINT_LIB=$PWD/$l timeout 300 python bench.py --config $cfg --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw_$n.json 2> gpurun_out/sw_$n.err
    v=$(tail -1 gpurun_out/sw_$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e' % d['value'], d['clocks']['sm_mhz'])" 2>/dev/null)
    echo "$l $cfg $v"
  done
done
