#!/bin/bash
# C4 walker iteration: parity tests touching the per-target walker, then the C4 bench leg
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/c4
TAG=${1:-x}
python -m pytest tests -m gpu -q -x -k "rgg or c4 or shapes or sharding or option_matrix" 2>&1 | tail -3 > gpurun_out/c4/tests_$TAG.txt
for i in 1 2; do
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --skip-extra > gpurun_out/c4/bench_${TAG}_$i.json 2> gpurun_out/c4/bench_${TAG}_$i.err
done
