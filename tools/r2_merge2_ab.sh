#!/bin/bash
# cfg4 / cfg3 at N=4 and cfg4 at N=2: own+received GEMMs merged (HEP_MERGE_GEMMS=2) vs
# the default split launches, interleaved x3.  Logs -> gpurun_out/r2_merge2/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_merge2
mkdir -p $out
HEP_MERGE_GEMMS=2 timeout 900 python -m pytest tests/test_gpu_vranks.py -q -m gpu -x -k "test_virtual_ranks_layer and not fused" > $out/vranks_merge2.log 2>&1
echo "vranks merge2 rc=$?"; tail -1 $out/vranks_merge2.log
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 "$@" \
    > $out/$name.log 2>&1
  echo "$name rc=$?"
}
for rep in 1 2 3; do
  for m in 0 2; do
    HEP_MERGE_GEMMS=$m run cfg4_n4_m${m}_r$rep 4 --config cfg4
    HEP_MERGE_GEMMS=$m run cfg3_n4_m${m}_r$rep 4
  done
done
for m in 0 2; do HEP_MERGE_GEMMS=$m run cfg4_n2_m${m} 2 --config cfg4; done
