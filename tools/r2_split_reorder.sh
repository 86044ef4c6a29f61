#!/bin/bash
# SR split with the tile copy issued before the dependent mode load: codec parity tests,
# encode batch time, ncu per-kernel list.  Logs -> gpurun_out/r2_split_reorder/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_split_reorder
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_oracle.py -q -m gpu -x -k "sr or SR or encode or decode or wire" > $out/tests.log 2>&1
echo "tests rc=$?"; tail -1 $out/tests.log
for b in 16 32; do timeout 120 python tools/sr_encode_probe.py --batch $b > $out/time_b$b.log 2>&1; echo "b$b rc=$?"; tail -1 $out/time_b$b.log; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
  -k regex:"sr_" -c 8 python tools/sr_encode_probe.py --batch 16 --reps 2 > $out/launches_b16.csv 2>&1; echo "ncu rc=$?"
