#!/bin/bash
# cfg5 (8-layer stack) and cfg4 at N=4 after the per-layer-gate change.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_cfg5
for c in cfg5 cfg4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 20 --warmup 5 --config $c \
    > gpurun_out/r2_cfg5/${c}_n4.log 2>&1
  echo "$c rc=$?"
done
