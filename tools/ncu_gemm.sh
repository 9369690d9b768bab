#!/bin/bash
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
export BTD_GRAPHS=0
$CMD > gpurun_out/plain_c3.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > /dev/null 2>&1
n=$(grep -c "gemm_pipe_kernel" gpurun_out/launches_c3.csv)
skip=$((n - 30))
echo "gemm launches=$n skip=$skip"
ncu --set full --clock-control none --import-source on -k regex:gemm_pipe -s $skip -c 4 -o gpurun_out/prof_c3_gemm $CMD > gpurun_out/ncu_c3_gemm.log 2>&1
echo rc=$?
