#!/bin/bash
# 3xTF32 GEMM with raw B split in shared memory vs pre-split hi/lo weights (cfg1, N=1).
# Logs -> gpurun_out/r2_tf32raw/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_tf32raw
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "f32 or tf32" > $out/tests_kernels.log 2>&1
echo "kernel tests rc=$?"; tail -1 $out/tests_kernels.log
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_vranks.py -q -m gpu -x -k "f32 or fp32 or cfg1 or cfg2" > $out/tests_layer.log 2>&1
echo "layer tests rc=$?"; tail -1 $out/tests_layer.log
for rep in 1 2; do
  timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 > $out/cfg1_raw_r$rep.log 2>&1; echo "raw rc=$?"
  HEP_TF32_PRESPLIT=1 timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 > $out/cfg1_pre_r$rep.log 2>&1; echo "pre rc=$?"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:tf32x3 -c 4 --csv python bench.py --config cfg1 --steps 2 --warmup 3 > $out/ncu_raw.csv 2>&1
echo "ncu rc=$?"
HEP_TF32_PRESPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:tf32x3 -c 4 --csv python bench.py --config cfg1 --steps 2 --warmup 3 > $out/ncu_pre.csv 2>&1
echo "ncu pre rc=$?"
