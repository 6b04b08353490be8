#!/bin/bash
# Round-2 GPU cycle: GPU tests, bench lines (C5 default, C2, C4), round-1 A/B.
# usage: bash tools/gpu/r2_cycle.sh [tests|bench|ab|all]
set -u
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
if [[ $what == bench || $what == all ]]; then
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
  timeout 600 python bench.py --config C2 --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
  timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
fi
if [[ $what == ab || $what == all ]]; then
  (cd build_variants/r1 && timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline) > gpurun_out/r1_c2.json 2> gpurun_out/r1_c2.err
  (cd build_variants/r1 && timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline) > gpurun_out/r1_c5.json 2> gpurun_out/r1_c5.err
fi
