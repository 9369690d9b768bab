#!/bin/bash
# ncu launch lists (gpu__time_duration per launch) of one solve step per config -> launch shares
T=/tmp/ll; OUT=gpurun_out/ll; mkdir -p $T $OUT
export BTD_GRAPHS=0
for c in ${CONFIGS:-c1 c2 c3 c4 c0}; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
  $CMD > $T/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_$c.csv $CMD > /dev/null 2>&1
  echo "ncu $c rc=$?"
  python tools/launch_shares.py $OUT/launch_shares_$c.json $c:$T/launches_$c.csv:$T/plain_$c.log
  python - "$T/launches_$c.csv" "$OUT/launches_$c.csv" <<'PY'
import sys
lines = open(sys.argv[1]).read().splitlines()
keep = [l for l in lines if "btd::" in l or "anonymous namespace" in l or "Kernel Name" in l]
open(sys.argv[2], "w").write("\n".join(keep[-400:]) + "\n")
PY
done
du -sh $OUT
