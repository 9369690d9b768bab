#!/bin/bash
# ncu evidence for the bench configs: launch list (device times of every
# kernel, cold/serialised) + one full capture of the forward and backward sweep.
set -u
OUT=gpurun_out
for c in "$@"; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu --no-check"
  $CMD > $OUT/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv $CMD > $OUT/ncu_launch_$c.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:chain_ -s 2 -c 2 -o $OUT/prof_$c $CMD > $OUT/ncu_full_$c.log 2>&1
  echo "$c done rc=$?"
done
