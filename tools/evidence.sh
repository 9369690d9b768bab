#!/bin/bash
# Full evidence run: bench lines for every config, ncu launch lists and one full
# capture of the forward + backward sweep kernels (GEMM for c3).
set -u
OUT=gpurun_out/ev
mkdir -p $OUT
export BTD_GRAPHS=0   # ncu replays individual kernels; graphs off for the captures only
for c in c1 c0 c2 c3 c4; do
  BTD_GRAPHS=1 timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$?"
done
for c in c1 c2 c4 c3; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
  $CMD > $OUT/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv $CMD > /dev/null 2>&1
  if [ $c = c3 ]; then
    n=$(grep -c "gemm_pipe_kernel" $OUT/launches_$c.csv); skip=$((n - 20))
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pipe -s $skip -c 3 -o $OUT/prof_$c $CMD > $OUT/ncu_$c.log 2>&1
  else
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:chain_|stream_" -s 2 -c 2 -o $OUT/prof_$c $CMD > $OUT/ncu_$c.log 2>&1
  fi
  echo "ncu $c rc=$?"
done
