#!/bin/bash
# Round-2 bench check on a 2-GPU box: N=1 cfg3 (the driver's line), the reference arm,
# and N=2 cfg3 / cfg5 / cfg4 through the planner path.  Logs -> gpurun_out/r2_bench/.
mkdir -p gpurun_out/r2_bench
cd "$(dirname "$0")/.."
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench/cfg3_n1.log 2>&1
echo "cfg3 n1 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench/reference_cfg3.log 2>&1
echo "reference rc=$?"
for c in cfg3 cfg5 cfg4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --config $c > gpurun_out/r2_bench/${c}_n2.log 2>&1
  echo "$c n2 rc=$?"
done
