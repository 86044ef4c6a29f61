#!/bin/bash
# The round-end bench subset (run under `gpurun --gpus 4`): the headline cfg3 at 1/2/4
# GPUs, cfg1 (fp32), cfg4 (fine-grained + SR) and cfg5 (8 layers) at 1 and 4, the
# reference arm, and smoke().  One JSON line per run in gpurun_out/final/<name>.log; summarise with
# python tools/sweep_report.py gpurun_out/final.
mkdir -p gpurun_out/final
port=29700
run() {  # run <name> <N> <args...>
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --gpus 1 "$@" > gpurun_out/final/$name.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $n "$@" > gpurun_out/final/$name.log 2>&1
  fi
  echo "$name rc=$?"
}
run cfg3_n1 1 --config cfg3 --steps 30 --warmup 3
run cfg3_n2 2 --config cfg3 --steps 30 --warmup 3
run cfg3_n4 4 --config cfg3 --steps 30 --warmup 3
run cfg1_n1 1 --config cfg1 --steps 30 --warmup 3
run cfg1_n4 4 --config cfg1 --steps 30 --warmup 3
run cfg4_n1 1 --config cfg4 --steps 30 --warmup 3
run cfg4_n4 4 --config cfg4 --steps 30 --warmup 3
run cfg5_n1 1 --config cfg5 --steps 10 --warmup 3
run cfg5_n4 4 --config cfg5 --steps 10 --warmup 3
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/reference_cfg3_n1.txt 2>&1
echo "reference rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1
echo "smoke rc=$?"
