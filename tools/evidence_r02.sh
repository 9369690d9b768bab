#!/bin/bash
# Round-2 evidence run on one B200 (gpurun): GPU tests, smoke, bench lines for every
# config, the reference arm, ncu launch list of the default bench and one full ncu
# capture of its dominant kernel.  Outputs under gpurun_out/r02/ (summaries are copied
# to profiles/r02/ by hand).
set -x
O=gpurun_out/r02
mkdir -p $O
nvidia-smi -q -d CLOCK,POWER > $O/nvsmi_before.txt 2>&1
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
for c in c0 c1 c2 c3; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --config c3dd --steps 5 --warmup 2 > $O/bench_c3dd.json 2> $O/bench_c3dd.err
python bench.py --impl reference > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stream_fwd_kernel -s 3 -c 1 \
    -o $O/ncu_full_c4_fwd python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gjc_panel_kernel -c 1 \
    -o $O/ncu_full_gjc_c1 python tools/build_profile.py c1 > $O/ncu_full_gjc.log 2>&1
ls -la $O
