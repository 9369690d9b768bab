#!/bin/bash
# ncu full capture of the warp-specialised GEMM (c3 mode-1 steps), BTD_GEMM_WS=$1
export BTD_GEMM_WS=${1:-1} BTD_GRAPHS=0
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
$CMD > gpurun_out/plain_ws.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:gemm_ws -s 20 -c 2 -o gpurun_out/prof_ws$1 $CMD > gpurun_out/ncu_ws.log 2>&1
echo rc=$?
