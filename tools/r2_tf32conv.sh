#!/bin/bash
# 3xTF32 converter variants: accuracy and cfg1 N=1 timing.  Logs -> gpurun_out/r2_tf32conv/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_tf32conv
mkdir -p $out
for m in 4 8 5 6; do HEP_TF32_CONV=$m timeout 120 python tools/tf32_conv_exp.py >> $out/acc.jsonl 2>>$out/acc.err; done
HEP_TF32_PRESPLIT=1 timeout 120 python tools/tf32_conv_exp.py >> $out/acc.jsonl 2>>$out/acc.err
echo "acc rc=$?"
for rep in 1 2; do
  for m in 4 8 5 6 pre; do
    if [ $m = pre ]; then env="HEP_TF32_PRESPLIT=1"; else env="HEP_TF32_CONV=$m"; fi
    env $env timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 > $out/cfg1_${m}_r$rep.log 2>&1; echo "$m rc=$?"
  done
done
