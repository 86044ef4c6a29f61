#!/bin/bash
# A/B of the capped remote-dispatch grid (HEP_DISPATCH_CTAS) at N=4, interleaved.
# Logs -> gpurun_out/r2_dispatch/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_dispatch
timeout 900 python -m pytest tests/test_gpu_vranks.py -q -m gpu -x > gpurun_out/r2_dispatch/vranks.log 2>&1
echo "vranks rc=$?"; tail -2 gpurun_out/r2_dispatch/vranks.log
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 "$@" \
    > gpurun_out/r2_dispatch/$name.log 2>&1
  echo "$name rc=$?"
}
for rep in 1 2; do
  for cap in 0 148 296; do
    HEP_DISPATCH_CTAS=$cap run cfg4_n4_cap${cap}_r$rep 4 --config cfg4
    HEP_DISPATCH_CTAS=$cap run cfg3_n4_cap${cap}_r$rep 4
  done
done
