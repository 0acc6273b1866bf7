#!/bin/bash
# C2 A/B: stage traces and event-timed steps, old (_lib_ab/libgmaco_old.so) vs new build
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/ab
TAG=$1
OLD=paper_2010_14244_b200/_lib_ab/libgmaco_old.so; NEW=paper_2010_14244_b200/_lib/libgmaco.so
for L in old new; do
  LIBP=$OLD; [ $L = new ] && LIBP=$NEW
  LIB=$LIBP TAG=$L python tools/stage_trace.py >> gpurun_out/ab/${TAG}_trace.txt 2>&1
done
for r in 1 2 3; do
  python tools/ab_bench.py $OLD c2 50 5 >> gpurun_out/ab/${TAG}.jsonl 2>>gpurun_out/ab/${TAG}.err
  python tools/ab_bench.py $NEW c2 50 5 >> gpurun_out/ab/${TAG}.jsonl 2>>gpurun_out/ab/${TAG}.err
done
