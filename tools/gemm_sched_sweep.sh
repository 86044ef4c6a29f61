# GEMM schedule sweep (L2 policy / raster) on one B200: phase times + ncu DRAM bytes.
# Usage: bash tools/gemm_sched_sweep.sh "UP DOWN" ...   (hex sched words, see kernels.h)
mkdir -p gpurun_out
for cfg in "$@"; do
  set -- $cfg
  echo "UP=$1 DOWN=$2" >> gpurun_out/sweep.log
  HEP_GEMM_SCHED_UP=$1 HEP_GEMM_SCHED_DOWN=$2 timeout -s KILL 200 python bench.py --steps 20 --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print({k: round(v,3) for k,v in d['phase_ms'].items()}, round(d['roofline']['achieved']), d['clocks'])" >> gpurun_out/sweep.log 2>&1
  HEP_GEMM_SCHED_UP=$1 HEP_GEMM_SCHED_DOWN=$2 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped_gemm -s 2 -c 2 --csv --log-file gpurun_out/ncu_sched_$1_$2.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
done
