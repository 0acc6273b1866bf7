#!/bin/bash
# e2e loop A/B: tools/gpu/abe2e.sh TAG lib1 lib2 ... (create_profile with LIB)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/ab
TAG=$1; shift
for r in 1 2; do for L in "$@"; do
  echo "== $L" >> gpurun_out/ab/${TAG}_e2e.txt
  LIB=$L python tools/create_profile.py c2 20 2>/dev/null | grep "^rep [12]" >> gpurun_out/ab/${TAG}_e2e.txt
done; done
