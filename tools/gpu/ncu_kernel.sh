#!/bin/bash
# ncu --set full of one kernel launch: tools/gpu/ncu_kernel.sh LIB CONFIG KERNEL_REGEX SKIP OUT [steps]
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/ncu
LIB=$1; CFG=$2; K=$3; SKIP=$4; OUT=$5; N=${6:-12}
python tools/ab_bench.py $LIB $CFG 3 2 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k "regex:$K" --launch-skip $SKIP --launch-count 1 \
    -o gpurun_out/ncu/$OUT -f python tools/ab_bench.py $LIB $CFG $N 2 > gpurun_out/ncu/$OUT.log 2>&1
echo "ncu rc=$?"
