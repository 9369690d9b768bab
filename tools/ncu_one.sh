#!/bin/bash
# full ncu capture of the chain kernels of one config (one fwd + one bwd launch)
c=$1; tag=$2
CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
$CMD > gpurun_out/plain_$c.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:chain_ -s 2 -c 2 -o gpurun_out/prof_${c}_$tag $CMD > gpurun_out/ncu_${c}_$tag.log 2>&1
echo "$c rc=$?"
