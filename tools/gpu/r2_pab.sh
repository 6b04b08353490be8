#!/bin/bash
# parity tests (optionally against a variant library: PARITY_LIB=...) + A/B
# timing of variant libraries + optional ncu capture
# usage: [PARITY_LIB=lib.so] bash tools/gpu/r2_pab.sh "<variant libs>" <ncu tag|none> [pytest args]
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
if [ -n "${PARITY_LIB:-}" ]; then export GLINT_LIB=$PWD/$PARITY_LIB; fi
GLINT_PARITY_LOG=$PWD/gpurun_out/parity_err.txt timeout 1500 python -m pytest ${3:-tests/test_gpu_parity.py} -x -q -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1
echo "exit $? (lib ${GLINT_LIB:-product})" >> gpurun_out/pytest_parity.log
unset GLINT_LIB
if [ "$2" = none ]; then bash tools/gpu/ab.sh "$1"; else bash tools/gpu/ab.sh "$1" ncu $2; fi
