#!/bin/bash
# cfg3 N=1: dynamic tile queue on the down-projection only (HEP_GEMM_DYN=down) vs the
# static schedule, interleaved x3, plus ncu DRAM bytes of both.  Logs -> gpurun_out/r2_dyn_down/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_dyn_down${SUFFIX}
mkdir -p $out
for rep in 1 2 3 4 5 6; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > $out/static_r$rep.log 2>&1; echo "static rc=$?"
  HEP_GEMM_DYN=down timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > $out/dyn_r$rep.log 2>&1; echo "dyn rc=$?"
done
HEP_GEMM_DYN=down timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:grouped_gemm_bf16_2cta -s 14 -c 2 --csv python bench.py --steps 2 --warmup 3 --no-cpu \
  > $out/ncu_dyn.csv 2>&1; echo "ncu rc=$?"
HEP_GEMM_DYN=down timeout 600 python -m pytest tests/test_gpu_headline.py -q -m gpu > $out/headline.log 2>&1; echo "headline rc=$?"; tail -1 $out/headline.log
