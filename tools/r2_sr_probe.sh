#!/bin/bash
# SR encode chain of a cfg4 batch (16, 32): graph-replay time, ncu launch list, and a full
# capture of the sample / finish kernels.  Logs -> gpurun_out/r2_sr_probe/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_sr_probe
mkdir -p $out
for b in 16 32; do timeout 120 python tools/sr_encode_probe.py --batch $b > $out/time_b$b.log 2>&1; echo "b$b rc=$?"; cat $out/time_b$b.log | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv \
  -k regex:"sr_" python tools/sr_encode_probe.py --batch 16 --reps 2 > $out/launches_b16.csv 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sr_sample|sr_finish|sr_split" -c 3 -o $out/sr_full \
  python tools/sr_encode_probe.py --batch 16 --reps 2 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
