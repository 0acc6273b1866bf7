#!/bin/bash
# A/B: tools/gpu/ab.sh CONFIG TAG [steps] -- old (_lib_ab/libgmaco_old.so) vs new (_lib/libgmaco.so), interleaved
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/ab
CFG=$1; TAG=$2; N=${3:-10}
OLD=paper_2010_14244_b200/_lib_ab/libgmaco_old.so; NEW=paper_2010_14244_b200/_lib/libgmaco.so
for r in 1 2 3; do
  python tools/ab_bench.py $OLD $CFG $N 3 >> gpurun_out/ab/${TAG}.jsonl 2>>gpurun_out/ab/${TAG}.err
  python tools/ab_bench.py $NEW $CFG $N 3 >> gpurun_out/ab/${TAG}.jsonl 2>>gpurun_out/ab/${TAG}.err
done
if [ -n "$NCU" ]; then
  for L in old new; do
    LIB=$OLD; [ $L = new ] && LIB=$NEW
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab/${TAG}_ncu_$L.csv \
      python tools/ab_bench.py $LIB $CFG 3 2 > /dev/null 2>&1
  done
fi
