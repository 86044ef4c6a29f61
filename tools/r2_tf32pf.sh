#!/bin/bash
# 3xTF32 GEMM: L2 prefetch distance of the weight stream (HEP_TF32_PF), cfg1 N=1,
# interleaved; ncu time / DRAM / tensor-active per launch.  Logs -> gpurun_out/r2_tf32pf/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_tf32pf
mkdir -p $out
HEP_TF32_PF=8 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "f32 or tf32" > $out/tests.log 2>&1
echo "tests rc=$?"; tail -1 $out/tests.log
for rep in 1 2 3; do
  for pf in 0 4 8 16; do
    HEP_TF32_PF=$pf timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 > $out/cfg1_pf${pf}_r$rep.log 2>&1; echo "pf$pf rc=$?"
  done
done
for pf in 0 8 16; do
  HEP_TF32_PF=$pf timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:tf32x3 -c 4 --csv python bench.py --config cfg1 --steps 2 --warmup 3 > $out/ncu_pf$pf.csv 2>&1
  echo "ncu pf$pf rc=$?"
done
