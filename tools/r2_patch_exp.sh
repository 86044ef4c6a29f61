#!/bin/bash
# Fused-decode GEMM cost split: real patch lists vs empty blocks (same pipeline, no entries).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_patch
for v in real empty real empty; do
  if [ $v = empty ]; then export HEP_PATCH_EXP=empty; else unset HEP_PATCH_EXP; fi
  HEP_SR_FUSED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --config cfg4 \
    > gpurun_out/r2_patch/$v.$RANDOM.log 2>&1
  echo "$v rc=$?"
done
