#!/bin/bash
# Full GPU cycle: all -m gpu tests (with the parity error log), smoke, bench
# lines (C5 default, C2, C4), ncu launch list of the default bench and a full
# capture of one C5 frame and one C2 frame, whole-step counts.
# usage: bash tools/gpu/r2_full.sh <tag> [notests]
cd "$(dirname "$0")/../.."
tag=${1:-r2}
mkdir -p gpurun_out
if [ "${2:-}" != notests ]; then
  GLINT_PARITY_LOG=$PWD/gpurun_out/parity_err_$tag.txt timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$tag.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_$tag.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$tag.log
fi
timeout 900 python bench.py > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err
timeout 600 python bench.py --config C2 > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 600 python bench.py --config C4 --steps 10 > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
# launch list of the default bench command (short), per the profiling recipe
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_launch_$tag.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "glint_timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
# full captures: C5 frame 31 (serial pass: warmup 3 x 64 launches, then frames in order) and C2 35 deg
M=smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:glint_eval_kernel -s $((3*64+31)) -c 1 \
  -o gpurun_out/full_c5_$tag python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c5_$tag.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:glint_eval_kernel -s 33 -c 1 \
  -o gpurun_out/full_c2_$tag python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c2_$tag.log 2>&1; echo "ncu c2 rc=$?"
bash tools/gpu/step_counts.sh C2 C4 C5
