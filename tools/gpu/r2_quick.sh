#!/bin/bash
# quick GPU checks: selected pytest files + the reference arm's default line
# usage: bash tools/gpu/r2_quick.sh "<pytest args>"
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1800 python -m pytest $1 -x -q -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/pytest_quick.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_default.json 2> gpurun_out/ref_default.err; echo "ref rc=$?" >> gpurun_out/pytest_quick.log
