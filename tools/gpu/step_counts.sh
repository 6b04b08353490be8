#!/bin/bash
# Whole-step ncu counts (instructions, DRAM bytes, time) of the serialised
# per-frame launches bench.py runs outside its timed region, per config.
# usage: bash tools/gpu/step_counts.sh [C2 C4 C5]
mkdir -p gpurun_out
for cfg in ${@:-C2 C4 C5}; do
  case $cfg in C2) f=10;; C4) f=8;; C5) f=64;; esac
  CMD="python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  M=smsp__thread_inst_executed_pred_on.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
  echo "ncu --metrics $M --clock-control none -k regex:glint_eval_kernel -s $((3 * f)) -c $f --csv $CMD" > gpurun_out/counts_$cfg.cmd
  $CMD > gpurun_out/counts_plain_$cfg.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:glint_eval_kernel -s $((3 * f)) -c $f --csv \
      --log-file gpurun_out/counts_$cfg.csv $CMD > gpurun_out/counts_ncu_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
