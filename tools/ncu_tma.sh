#!/bin/bash
# ncu: launch list + full capture of the TMA GEMM on the c3 solve steps (not plan build)
export BTD_GRAPHS=0
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
$CMD > gpurun_out/plain_c3.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > /dev/null 2>&1
n=$(grep -c "gemm_tma_kernel" gpurun_out/launches_c3.csv)
skip=$((n - 12))
echo "tma launches=$n skip=$skip"
ncu --set full --clock-control none --import-source on -k regex:gemm_tma -s $skip -c 2 -o gpurun_out/prof_c3_tma $CMD > gpurun_out/ncu_c3_tma.log 2>&1
echo rc=$?
