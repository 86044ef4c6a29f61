#!/bin/bash
# Full one-GPU check: every -m gpu test, smoke(), the cfg3 bench line, and the ncu
# launch list + GEMM capture of a short cfg3 bench.  Logs -> gpurun_out/r2_full/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_full
export HEP_ACCURACY_LOG=gpurun_out/r2_full/accuracy.jsonl
rm -f $HEP_ACCURACY_LOG
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_full/tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r2_full/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_full/cfg3_n1.log 2>&1; echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_full/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_full/launches_cfg3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_full/ncu_launches.log 2>&1; echo "ncu rc=$?"
