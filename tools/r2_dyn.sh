#!/bin/bash
# Dynamic tile scheduler: correctness (GEMM + layer tests) then A/B timing and ncu DRAM bytes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_dyn
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_headline.py -q -m gpu -x -k "gemm or layer or headline" > gpurun_out/r2_dyn/tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2_dyn/tests.log
timeout 600 python tools/gemm_ab.py --proj down --variants 822:5:0,822:5:1,2:5:1,422:5:1 --rounds 6 > gpurun_out/r2_dyn/ab_down.log 2>&1
timeout 600 python tools/gemm_ab.py --proj up --variants 2:5:0,2:5:1 --rounds 6 > gpurun_out/r2_dyn/ab_up.log 2>&1
python tools/gemm_sched_dram.py > gpurun_out/r2_dyn/sched_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:grouped_gemm --log-file gpurun_out/r2_dyn/sched_dram.csv python tools/gemm_sched_dram.py > gpurun_out/r2_dyn/sched_ncu.log 2>&1
echo "ncu rc=$?"
