#!/bin/bash
for lib in paper_2306_05051_b200/libglint.so build_variants/*.so; do
  echo "== $lib"
  GLINT_LIB=$PWD/$lib timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; t=sys.stdin.read().strip().split(chr(10)); d=json.loads(t[-1]) if t[-1].startswith('{') else None; print(d['value'] if d else t[-5:], d and d['roofline']['mean_launch_ms'])"
done
