#!/bin/bash
# One GEMM launch per projection over all groups (HEP_MERGE_GEMMS=1) vs the split
# own / remote / gathered launches, N=4, interleaved.  Logs -> gpurun_out/r2_merge/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_merge
mkdir -p $out
HEP_MERGE_GEMMS=1 timeout 900 python -m pytest tests/test_gpu_vranks.py -q -m gpu -x -k "test_virtual_ranks_layer and not fused" > $out/vranks_merge.log 2>&1
echo "vranks merge rc=$?"; tail -1 $out/vranks_merge.log
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 "$@" \
    > $out/$name.log 2>&1
  echo "$name rc=$?"
}
for rep in 1 2; do
  for m in 0 1; do
    HEP_MERGE_GEMMS=$m run cfg4_n4_m${m}_r$rep 4 --config cfg4
    HEP_MERGE_GEMMS=$m run cfg4_n2_m${m}_r$rep 2 --config cfg4
  done
done
for m in 0 1; do HEP_MERGE_GEMMS=$m run cfg3_n4_m${m} 4; done
