#!/bin/bash
# Per-config bench lines: our arm and the reference arm
# for BASELINE configs 0-3 (config 4 is the default bench line).
# Usage (on the GPU box): bash tools/bench_configs.sh <tag>
cd ${GRAFT_REPO_ROOT:-.}
tag=${1:-r02}
mkdir -p gpurun_out
for c in 0 1 2 3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 \
    > gpurun_out/bench_${tag}_cfg$c.json 2> gpurun_out/bench_${tag}_cfg$c.err
  echo "cfg$c ours rc=$?"
  timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 1 \
    > gpurun_out/bench_ref_${tag}_cfg$c.json 2> gpurun_out/bench_ref_${tag}_cfg$c.err
  echo "cfg$c ref rc=$?"
done
