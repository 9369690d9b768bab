#!/bin/bash
# Functional check of bench.py's multi-rank path on ONE GPU: W ranks share the device,
# collectives over gloo (host), so no kernel waits on another rank.  Timings are not
# scaling numbers (the ranks time-share one GPU); the residual checks the sharded solve.
OUT=${OUT:-gpurun_out/shard_gloo}; mkdir -p $OUT
port=29600
for spec in "c4 2" "c1 2" "c2 4" "c4 4" "c3 2"; do
  set -- $spec; c=$1; w=$2; port=$((port+1))
  BTD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w \
    --master-addr 127.0.0.1 --master-port $port bench.py --gpus $w --config $c --steps 3 --warmup 3 \
    > $OUT/bench_${c}_w$w.json 2> $OUT/bench_${c}_w$w.err
  echo "$c w=$w rc=$? $(python -c "
import json,sys
try:
  d=json.loads(open('$OUT/bench_${c}_w$w.json').read().strip().splitlines()[-1])
  print('RHS/s=%.0f res=%s e2e=%s launches=%s' % (d['value'], d['rel_residual'], (d['e2e'] or {}).get('value'), d['gpu_launches']))
except Exception as e: print('no json', e)")"
done
