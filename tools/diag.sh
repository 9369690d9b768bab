python bench.py --config c3 > gpurun_out/diag_c3.json 2> gpurun_out/diag_c3.err; echo c3 rc=$?
CMD="python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check"
BTD_GRAPHS=0 $CMD > /dev/null 2>&1 && BTD_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:chain_" -s 2 -c 2 -o /tmp/prof_c1_new $CMD > gpurun_out/diag_ncu.log 2>&1; echo ncu rc=$?
tail -20 gpurun_out/diag_ncu.log
