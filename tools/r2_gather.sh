#!/bin/bash
# Permute fused into the up-projection's A load (tile::gather4) vs the explicit permute:
# parity tests, then cfg3 / cfg4 N=1 bench A/B.  Logs -> gpurun_out/r2_gather/.
cd "$(dirname "$0")/.."
out=gpurun_out/r2_gather
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_headline.py -q -m gpu -x > $out/tests.log 2>&1
echo "tests rc=$?"; tail -3 $out/tests.log
for rep in 1 2; do
  for ga in 1 0; do
    HEP_GATHER_A=$ga timeout 300 python bench.py --steps 20 --warmup 5 > $out/cfg3_g${ga}_r$rep.log 2>&1; echo "cfg3 g$ga rc=$?"
    HEP_GATHER_A=$ga timeout 300 python bench.py --config cfg4 --steps 20 --warmup 5 > $out/cfg4_g${ga}_r$rep.log 2>&1; echo "cfg4 g$ga rc=$?"
  done
done
