#!/bin/bash
# ncu launch lists (gpu__time_duration.sum per kernel, cold-cache and serialised) of one
# bench step per config plus the plain bench line giving gpu_launches per step; the per-
# kernel share of a step: tools/launch_shares.py profiles/r02/launch_shares.json c4:...:...
O=gpurun_out/r02
mkdir -p $O
for c in c4 c1 c2 c3; do
  python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/plain_$c.log 2>/dev/null
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/build_launches_c3.csv \
    python tools/build_profile.py c3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/build_launches_c1.csv \
    python tools/build_profile.py c1 > /dev/null 2>&1
ls -la $O
