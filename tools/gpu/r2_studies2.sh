#!/bin/bash
# After gates-before-counts: parity, then the timing studies whose numbers the
# kernel change moves (section-6 ablation + ZK baseline, Table 1 analogue).
# Fig. 4 / Fig. 9 statistics and the coherence metrics depend only on the
# draws and the radiance, which are unchanged bit for bit.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_parity_s2.log 2>&1; echo "parity rc=$?"
bash tools/gpu/ablation.sh > gpurun_out/r2_ablation.txt 2>&1; echo "ablation rc=$?"
timeout 1200 python tools/gpu/table1.py --out gpurun_out/r2_table1 > gpurun_out/r2_table1.log 2>&1; echo "table1 rc=$?"
