#!/bin/bash
# Full evidence run: bench lines for every config, ncu launch lists and one full
# capture of the dominant kernels.  Heavy files stay in /tmp/ev on the box; only
# bench JSON, launch shares and text summaries come back in gpurun_out/ev (<64 MiB).
set -u
T=/tmp/ev
OUT=gpurun_out/ev
mkdir -p $T $OUT
export BTD_GRAPHS=0   # ncu replays individual kernels; graphs off for the captures only
for c in ${CONFIGS:-c1 c0 c2 c3 c4 c3dd}; do
  BTD_GRAPHS=1 timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $T/bench_$c.err
  echo "bench $c rc=$?"
done
for c in ${NCU_CONFIGS:-c1 c2 c4 c3}; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
  $CMD > $T/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_$c.csv $CMD > /dev/null 2>&1
  if [ $c = c3 ]; then
    n=$(grep -c "gemm_tma_kernel" $T/launches_$c.csv); skip=$((n - 12))
    timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:gemm_tma -s $skip -c 2 -o $T/prof_$c $CMD > $T/ncu_$c.log 2>&1
  else
    timeout 900 ncu -f --set full --clock-control none --import-source on -k "regex:chain_|stream_" -s 2 -c 2 -o $T/prof_$c $CMD > $T/ncu_$c.log 2>&1
  fi
  echo "ncu $c rc=$?"
  python tools/ncu_summary.py $T/prof_$c.ncu-rep > $OUT/ncu_full_$c.txt 2>&1
  python tools/launch_shares.py $OUT/launch_shares_$c.json $c:$T/launches_$c.csv:$T/plain_$c.log > /dev/null 2>&1
  grep -E "btd::|anonymous namespace|Kernel Name" $T/launches_$c.csv | tail -n 400 > $OUT/launches_$c.csv
  cp $T/plain_$c.log $OUT/
done
du -sh $OUT
