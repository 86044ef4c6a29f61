#!/bin/bash
# One-GPU round-2 evidence: layer tests, cfg3 / cfg1 / cfg4 bench lines, the reference arm,
# then the ncu launch list of a short cfg3 bench.  Logs -> gpurun_out/r2_n1/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2_n1
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_cpp_api.py -q -m gpu -x > gpurun_out/r2_n1/tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_n1/cfg3_n1.log 2>&1; echo "cfg3 rc=$?"
timeout 600 python bench.py --steps 50 --warmup 5 --config cfg1 > gpurun_out/r2_n1/cfg1_n1.log 2>&1; echo "cfg1 rc=$?"
HEP_GRAPH=0 timeout 600 python bench.py --steps 50 --warmup 5 --config cfg1 --no-cpu > gpurun_out/r2_n1/cfg1_n1_nograph.log 2>&1; echo "cfg1 nograph rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --config cfg4 --no-cpu > gpurun_out/r2_n1/cfg4_n1.log 2>&1; echo "cfg4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_n1/reference_cfg3.log 2>&1; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_n1/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_n1/launches_cfg3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_n1/ncu_launches.log 2>&1; echo "ncu rc=$?"
