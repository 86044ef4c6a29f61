#!/bin/bash
# ncu --set full of the cfg3 expert GEMM pair of one timed step (after 3 warm-up steps).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_ncu
python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/r2_ncu/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 6 -c 2 \
    -o gpurun_out/r2_ncu/gemm_cfg3 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/r2_ncu/ncu.log 2>&1
echo "ncu rc=$?"
