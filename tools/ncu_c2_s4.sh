c=c2
CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
$CMD > gpurun_out/plain_$c.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:chain_ -s 2 -c 2 -o gpurun_out/prof_${c}_s4 $CMD > gpurun_out/ncu_${c}_s4.log 2>&1
echo "$c rc=$?"
