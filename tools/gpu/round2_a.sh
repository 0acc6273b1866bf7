#!/bin/bash
# tests + bench legs (default, reference algorithms) for round 2
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/r2a
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2a/tests.txt
python bench.py > gpurun_out/r2a/bench_default.json 2> gpurun_out/r2a/bench_default.err
python bench.py --algorithm maco-p --config c2 --steps 200 --warmup 5 > gpurun_out/r2a/bench_macop_c2.json 2> gpurun_out/r2a/bench_macop_c2.err
python bench.py --algorithm maco --config c3 --steps 100 --warmup 5 --cpu-seconds 20 > gpurun_out/r2a/bench_maco_c3.json 2> gpurun_out/r2a/bench_maco_c3.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2a/ref_default.json 2>&1
