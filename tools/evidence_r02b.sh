#!/bin/bash
# Round-2 final evidence on one B200 (gpurun): GPU tests, smoke, bench lines for every config,
# the reference arm, ncu launch lists of one solve step (c4, c1), full ncu captures of the
# default bench's dominant kernel and of the scalar-coupled forward sweep (c1).
# Outputs under gpurun_out/r02b/ (summaries copied to profiles/r02/ by hand).
set -x
O=gpurun_out/r02b
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
for c in c0 c1 c2 c3; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --config c3dd --steps 5 --warmup 2 > $O/bench_c3dd.json 2> $O/bench_c3dd.err
python bench.py --impl reference > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
for c in c4 c1; do
  python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/plain_$c.log 2>/dev/null
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:stream_fwd_kernel -s 3 -c 1 \
    -o $O/ncu_full_c4_fwd python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/ncu_full_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chain_fwd_sc_kernel -s 3 -c 1 \
    -o $O/ncu_full_c1_fwd_sc python bench.py --config c1 --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/ncu_full_c1.log 2>&1
ls -la $O
