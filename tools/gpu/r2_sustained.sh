#!/bin/bash
# sustained runs of the default bench workload (C5) and of C2: clocks and
# throttle reasons over ~30-60 s timed regions
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 480 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sus_c5.json 2> gpurun_out/sus_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config C2 --steps 35000 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sus_c2.json 2> gpurun_out/sus_c2.err; echo "c2 rc=$?"
