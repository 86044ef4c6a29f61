#!/bin/bash
# Every BASELINE config at 1, 2 and 4 GPUs of one box (run under `gpurun --gpus 4`), plus
# the cfg2 S_ED sweep of the cfg1 shape at 4 GPUs.  One JSON line per run in
# gpurun_out/sweep/<config>_n<N>[_sed..].log; summarise with tools/sweep_report.py.
mkdir -p gpurun_out/sweep
port=29600
run() {  # run <name> <N> <args...>
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --gpus 1 "$@" > gpurun_out/sweep/$name.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $n "$@" > gpurun_out/sweep/$name.log 2>&1
  fi
  echo "$name rc=$?"
}
for cfg in cfg3 cfg4 cfg1 cfg5; do
  steps=30; [ $cfg = cfg5 ] && steps=10
  run ${cfg}_n1 1 --config $cfg --steps $steps --warmup 3 --no-cpu
  run ${cfg}_n2 2 --config $cfg --steps $steps --warmup 3
  run ${cfg}_n4 4 --config $cfg --steps $steps --warmup 3
done
for sed in 1,1 1,2 2,1 2,2; do
  run cfg2_n4_sed${sed/,/_} 4 --config cfg1 --sed $sed --steps 30 --warmup 3
done
