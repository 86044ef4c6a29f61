#!/bin/bash
# bench.py with the collector off in the timed passes: cfg1 (launch-bound) at N=1/2/4 and
# cfg3 at N=1.  Logs -> gpurun_out/r2_gc/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_gc
mkdir -p $out
timeout 300 python bench.py --steps 20 --warmup 5 > $out/cfg3_n1.log 2>&1; echo "cfg3 n1 rc=$?"
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 > $out/cfg1_n1.log 2>&1; echo "cfg1 n1 rc=$?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 --config cfg1 > $out/cfg1_n$n.log 2>&1
  echo "cfg1 n$n rc=$?"
done
