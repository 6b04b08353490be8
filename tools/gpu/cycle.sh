#!/bin/bash
# One build->measure cycle on the GPU box: parity tests, bench, ncu capture.
# usage: bash tools/gpu/cycle.sh <tag> [full|launches|none]
tag=${1:-x}; prof=${2:-full}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$tag.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_$tag.log
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench_rc=$?
cat gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if [ "$prof" = "full" ] || [ "$prof" = "both" ]; then
  $CMD > gpurun_out/plain_$tag.log 2>&1 && \
  ncu --set full --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum --clock-control none --import-source on -k regex:glint_eval_kernel -s 3 -c 1 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1; echo ncu_full_rc=$?
fi
if [ "$prof" = "launches" ] || [ "$prof" = "both" ]; then
  echo "ncu --nvtx --nvtx-include glint_timed/ --metrics gpu__time_duration.sum --clock-control none --csv $CMD" > gpurun_out/launches_$tag.cmd
  $CMD > gpurun_out/plain2_$tag.log 2>&1 && \
  ncu --nvtx --nvtx-include "glint_timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1; echo ncu_launch_rc=$?
fi
