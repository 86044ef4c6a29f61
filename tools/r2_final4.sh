#!/bin/bash
# Round-2 closing evidence on a 4-GPU box (final build): the real multi-process parity
# tests (peer-memory and NCCL paths) and bench lines at N=2 / N=4 for every config, plus
# pinned pure-All-Gather hierarchies for cfg5 / cfg3.  Logs -> gpurun_out/r2_final4/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_final4
mkdir -p $out
timeout 2400 python -m pytest tests/test_gpu_multi.py -v -m gpu > $out/test_gpu_multi_4gpu.log 2>&1
echo "multi tests rc=$?"; tail -1 $out/test_gpu_multi_4gpu.log
run() {  # name, N, extra args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 20 --warmup 5 "$@" \
    > $out/$name.log 2>&1
  echo "$name rc=$?"
}
for n in 2 4; do
  run cfg3_n$n $n
  run cfg4_n$n $n --config cfg4
  run cfg5_n$n $n --config cfg5
  run cfg1_n$n $n --config cfg1
done
run cfg5_n4_sed22 4 --config cfg5 --sed 2,2
run cfg5_n2_sed2 2 --config cfg5 --sed 2
run cfg3_n4_sed22 4 --sed 2,2
