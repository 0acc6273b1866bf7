#!/bin/bash
# A/B/...: tools/gpu/abn.sh CONFIG TAG STEPS lib1 lib2 ... -- interleaved ab_bench runs (3 rounds) + stage traces (C2)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/ab
CFG=$1; TAG=$2; N=$3; shift 3
for r in 1 2 3; do
  for L in "$@"; do
    python tools/ab_bench.py $L $CFG $N 5 >> gpurun_out/ab/${TAG}.jsonl 2>>gpurun_out/ab/${TAG}.err
  done
done
if [ "$CFG" = c2 ]; then
  for L in "$@"; do LIB=$L TAG=$(basename $L) python tools/stage_trace.py 2>&1 | grep "V=1000 flushed" >> gpurun_out/ab/${TAG}_trace.txt; done
fi
