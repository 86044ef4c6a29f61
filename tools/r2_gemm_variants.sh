#!/bin/bash
# cfg3 GEMM shapes: deep (6-stage) vs staged (5-stage) CTA-pair kernel, schedule sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_gemm
for deep in 1 0; do
  HEP_GEMM_DEEP=$deep timeout 300 python tools/gemm_bench.py --sched-up 2,822,12 --sched-down 822,2,422,1022,12,a22 \
    > gpurun_out/r2_gemm/deep$deep.log 2>&1
  echo "deep=$deep rc=$?"
done
