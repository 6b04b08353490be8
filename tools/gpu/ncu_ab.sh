#!/bin/bash
# ncu --set full of one C5 frame (31) for the product library and variants
# usage: bash tools/gpu/ncu_ab.sh "<variant libs>" [config] [skip]
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
cfg=${2:-C5}; skip=${3:-223}
for l in paper_2306_05051_b200/libglint.so $1; do
  n=$(basename $l .so)
  GLINT_LIB=$PWD/$l timeout 900 ncu --set full --clock-control none --import-source on -k regex:glint_eval_kernel -s $skip -c 1 \
    -o gpurun_out/ab_$n python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ab_$n.log 2>&1
  echo "$n rc=$?"
done
