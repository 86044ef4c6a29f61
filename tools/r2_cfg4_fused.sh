#!/bin/bash
# cfg4 (SR migration) at N=2: fused SR decode (default) vs the dense decode (HEP_SR_FUSED=0).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_cfg4
for mode in 1 0; do
  HEP_SR_FUSED=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --config cfg4 \
    > gpurun_out/r2_cfg4/n2_fused$mode.log 2>&1
  echo "fused=$mode rc=$?"
done
