#!/bin/bash
# ncu time + DRAM bytes of the cfg3 down-projection GEMM per L2 schedule (HEP_GEMM_SCHED_DOWN).
mkdir -p gpurun_out/dsched
python tools/kernel_roofline.py run --config cfg3 > /dev/null || exit 1
for sch in ${SCHEDS:-2 12 822 422 1022 6 a 22}; do
  HEP_GEMM_SCHED_DOWN=$sch ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    -k regex:grouped_gemm --launch-skip 2 --launch-count 2 --log-file gpurun_out/dsched/$sch.csv \
    python tools/kernel_roofline.py run --config cfg3 > /dev/null 2>&1
done
echo done
