#!/bin/bash
# The bench's default planner (reference model + measured routing imbalance) at N=2/4 for
# cfg5 and cfg3.  Logs -> gpurun_out/r2_planner_imb/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_planner_imb
mkdir -p $out
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 "$@" \
    > $out/$name.log 2>&1
  echo "$name rc=$?"
}
run cfg5_n4 4 --config cfg5
run cfg3_n4 4
run cfg5_n2 2 --config cfg5
run cfg3_n2 2
