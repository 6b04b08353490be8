#!/bin/bash
# bench the default library and each build_variants/*.so (no e2e / cpu legs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_var.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_var.log
for lib in paper_2306_05051_b200/libglint.so build_variants/*.so; do
  echo "== $lib"
  GLINT_LIB=$PWD/$lib python bench.py --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print(d['value'], d['roofline']['mean_launch_ms'], d['clocks'])"
done
