#!/bin/bash
# Interleaved A/B of HEP_GEMM_SPIN at N=4 (3 rounds per config), to separate the effect
# from run-to-run variance.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_spin
for round in 1 2 3; do
  for c in cfg4 cfg3; do
    for sp in 0 1; do
      HEP_GEMM_SPIN=$sp HEP_P2P_TIMEOUT_S=60 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 20 --warmup 5 \
        --config $c --no-cpu > gpurun_out/r2_spin/${c}_spin${sp}_r$round.log 2>&1
      echo "$c spin=$sp round=$round rc=$?"
    done
  done
done
