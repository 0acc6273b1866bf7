#!/bin/bash
# Bench lines, launch lists and ncu captures for profiles/ (round TAG).
cd "$(dirname "$0")/../.."
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for c in c1 c3 c4 c5; do
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
python bench.py --algorithm maco-p --config c2 --steps 200 --warmup 5 > $O/bench_macop_c2.json 2> $O/bench_macop_c2.err
python bench.py --algorithm maco --config c3 --steps 100 --warmup 5 --cpu-seconds 20 > $O/bench_maco_c3.json 2> $O/bench_maco_c3.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err
python tools/stage_trace.py > $O/stage_trace.txt 2>&1
# launch list (serialised, cold) of the default bench leg
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-secondary --skip-extra > $O/ncu_launch.log 2>&1
L=paper_2010_14244_b200/_lib/libgmaco.so
bash tools/gpu/ncu_kernel.sh $L c2 k_colony_grid 8 ${T}_c2_walk
bash tools/gpu/ncu_kernel.sh $L c2 k_tail_coop 8 ${T}_c2_tail
bash tools/gpu/ncu_kernel.sh $L c4 k_colony_qt 3 ${T}_c4_qt 5
bash tools/gpu/ncu_kernel.sh $L c3 k_colony_grid 4 ${T}_c3_walk 6
bash tools/gpu/ncu_kernel.sh $L c5 k_colony_grid 4 ${T}_c5_walk 6
bash tools/gpu/ncu_kernel.sh $L ref:maco-p:c2 k_tail_coop 8 ${T}_macop_step
# summaries on the box (the .ncu-rep files would exceed gpurun's 64 MiB copy-back)
for f in gpurun_out/ncu/${T}_*.ncu-rep; do
  python tools/ncu_summary.py report $f --json ${f%.ncu-rep}.json > /dev/null 2>&1
done
rm -f gpurun_out/ncu/${T}_*.ncu-rep
