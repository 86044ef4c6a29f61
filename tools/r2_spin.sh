#!/bin/bash
# In-kernel dispatch gating (HEP_GEMM_SPIN=1: one launch over own + received groups) vs the
# event-gated launches, cfg4 and cfg3 at N=4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_spin
for c in cfg4 cfg3; do
  for sp in 0 1; do
    HEP_GEMM_SPIN=$sp HEP_P2P_TIMEOUT_S=60 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 20 --warmup 5 \
      --config $c --no-cpu > gpurun_out/r2_spin/${c}_spin$sp.log 2>&1
    echo "$c spin=$sp rc=$?"
  done
done
