#!/bin/bash
# A/B timing of variant libraries (build_variants/exp/*.so, A/B only) against
# the product library on C2 and C5; optional ncu --set full capture of one C2
# frame (35 deg) of the product library.
# usage: bash tools/gpu/ab.sh "<lib ...>" [ncu]
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for l in paper_2306_05051_b200/libglint.so $1; do
  for cfg in ${AB_CONFIGS:-C2 C5}; do
    st=30; [ $cfg = C5 ] && st=5; [ $cfg = C4 ] && st=10
    n=$(basename $l .so)_$cfg
    GLINT_LIB=$PWD/$l timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
    v=$(tail -1 gpurun_out/ab_$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e %.3f ms %s' % (d['value'], d['ms_per_step'], d['clocks']['sm_mhz']))" 2>/dev/null)
    echo "$l $cfg $v" | tee -a gpurun_out/ab_summary.txt
  done
done
if [ "${2:-}" = ncu ]; then
  CMD="python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/ncu_plain.log 2>&1 && \
  ncu --set full --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed_pipe_fp64.sum \
    --clock-control none --import-source on -k regex:glint_eval_kernel -s 33 -c 1 -o gpurun_out/prof_c2_$3 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
fi
