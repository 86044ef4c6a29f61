#!/bin/bash
# cfg5 (8 Mixtral-shaped layers, residual stream) at N=4: every S_ED of SF=[2,2].
# Logs -> gpurun_out/r2_cfg5_sweep/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_cfg5_sweep
mkdir -p $out
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 --no-cpu "$@" \
    > $out/$name.log 2>&1
  echo "$name rc=$?"
}
for sed in 1,1 1,2 2,1 2,2; do run cfg5_n4_sed${sed/,/} 4 --config cfg5 --sed $sed; done
