#!/bin/bash
# cfg4 at N=2/4: All-Gather stream priority (HEP_AG_PRIORITY) x one GEMM launch per
# projection (HEP_MERGE_GEMMS), interleaved; cfg3 N=4 merge A/B.  Logs -> gpurun_out/r2_agprio/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_agprio
mkdir -p $out
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 "$@" \
    > $out/$name.log 2>&1
  echo "$name rc=$?"
}
for rep in 1 2; do
  for p in 0 1; do
    for m in 0 1; do
      HEP_AG_PRIORITY=$p HEP_MERGE_GEMMS=$m run cfg4_n4_p${p}_m${m}_r$rep 4 --config cfg4
    done
  done
  for m in 0 1; do HEP_AG_PRIORITY=1 HEP_MERGE_GEMMS=$m run cfg4_n2_p1_m${m}_r$rep 2 --config cfg4; done
  for m in 0 1; do HEP_MERGE_GEMMS=$m run cfg3_n4_m${m}_r$rep 4; done
done
