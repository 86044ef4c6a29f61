#!/bin/bash
# DRAM bytes of the cfg3 expert GEMM pair (final build), three separate ncu captures of
# one timed step each.  Logs -> gpurun_out/r2_traffic/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_traffic
mkdir -p $out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu > $out/plain.log 2>&1; echo "plain rc=$?"
for r in 1 2 3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:grouped_gemm_bf16_2cta -s 14 -c 2 --csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > $out/ncu_r$r.csv 2>&1; echo "ncu r$r rc=$?"
done
