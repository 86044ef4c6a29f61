#!/bin/bash
# ncu per-kernel time and DRAM bytes of the SR codec: the unfused step + encode and the
# fused step-with-encode (tools/bench_sr_fused.py, one process, no cross-rank waits).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_ncu
python tools/bench_sr_fused.py > gpurun_out/r2_ncu/sr_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"sr_|sgd_" -c 400 --log-file gpurun_out/r2_ncu/sr_kernels.csv python tools/bench_sr_fused.py > gpurun_out/r2_ncu/sr_ncu.log 2>&1
echo "ncu rc=$?"
