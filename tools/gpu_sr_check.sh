#!/bin/bash
# SR codec check on one B200 (run under gpurun): parity tests, bench_sr, launch list.
mkdir -p gpurun_out
tag=${1:-v}
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "sr or shared" > gpurun_out/t_sr_$tag.log 2>&1
tail -2 gpurun_out/t_sr_$tag.log
timeout 300 python tools/bench_sr.py --reps 20 > gpurun_out/bench_sr_$tag.log 2>&1
python tools/prof_sr.py > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/sr_launches_$tag.csv python tools/prof_sr.py > /dev/null 2>&1
echo done
