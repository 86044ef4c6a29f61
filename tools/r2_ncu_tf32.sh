#!/bin/bash
# Full ncu capture (source counters) of the 3xTF32 GEMM launches of cfg1 N=1.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_ncu_tf32
mkdir -p $out
timeout 300 python bench.py --config cfg1 --steps 2 --warmup 3 > $out/plain.log 2>&1
echo "plain rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tf32x3 -c 2 -o $out/tf32 \
  python bench.py --config cfg1 --steps 2 --warmup 3 > $out/ncu.log 2>&1
echo "ncu rc=$?"
