#!/bin/bash
# cfg3 GEMM shapes: 6- vs 5-stage CTA-pair kernel, schedule sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_gemm
for st in 6 5; do
  HEP_GEMM_STAGES=$st timeout 300 python tools/gemm_bench.py --sched-up 2,822,12 --sched-down 822,2,422,1022,12,a22 \
    > gpurun_out/r2_gemm/stages$st.log 2>&1
  echo "stages=$st rc=$?"
done
