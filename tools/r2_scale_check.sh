#!/bin/bash
# Round-2 4-GPU check: cfg3 / cfg5 / cfg4 at N=4 (cfg4 with and without the fused SR
# decode) plus the fused-encode microbenchmark.  Logs -> gpurun_out/r2_n4/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_n4
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 10 --warmup 3 --no-cpu "$@" \
    > gpurun_out/r2_n4/$name.log 2>&1
  echo "$name rc=$?"
}
run cfg4_n4 4 --config cfg4
HEP_SR_FUSED=0 run cfg4_n4_dense 4 --config cfg4
run cfg3_n4 4 --config cfg3
run cfg5_n4 4 --config cfg5
run cfg1_n4 4 --config cfg1
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/bench_sr_fused.py > gpurun_out/r2_n4/sr_fused.log 2>&1; echo "sr_fused rc=$?"
