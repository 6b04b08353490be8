#!/bin/bash
# Round-2 refresh of the section-8(f) studies with the final kernel (bijective
# draw hash, exact shell): ablation 48/64/160 + ZK baseline, Table 1 analogue,
# GPU statistics (Fig. 4 / Fig. 9), temporal coherence.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/gpu/ablation.sh > gpurun_out/r2_ablation.txt 2>&1
timeout 1200 python tools/gpu/table1.py --out gpurun_out/r2_table1 > gpurun_out/r2_table1.log 2>&1; echo "table1 rc=$?"
timeout 1200 python tests/harness/fig4.py --out gpurun_out/r2_fig4 > gpurun_out/r2_fig4.log 2>&1; echo "fig4 rc=$?"
timeout 1200 python tests/harness/fig9.py --out gpurun_out/r2_fig9 > gpurun_out/r2_fig9.log 2>&1; echo "fig9 rc=$?"
timeout 1500 python tools/gpu/coherence.py --out gpurun_out/r2_coherence > gpurun_out/r2_coherence.log 2>&1; echo "coherence rc=$?"
