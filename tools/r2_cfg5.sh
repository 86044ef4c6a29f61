#!/bin/bash
# cfg5 (8-layer stack on the residual stream) at N = 4, 2, 1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_cfg5
for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 --config cfg5 \
    > gpurun_out/r2_cfg5/cfg5_n$n.log 2>&1
  echo "cfg5 n$n rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 --config cfg5 > gpurun_out/r2_cfg5/cfg5_n1.log 2>&1
echo "cfg5 n1 rc=$?"
