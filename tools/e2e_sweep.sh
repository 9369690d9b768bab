#!/bin/bash
# e2e (host API) rate vs host-pipeline chunk count
for c in ${CONFIGS:-c1 c2}; do
  for ch in ${CHUNKS:-1 2 4 8}; do
    BTD_HOST_CHUNKS=$ch python bench.py --config $c --no-cpu --no-check --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'chunks=$ch', round(d['e2e']['value'],1), round(d['value'],1))"
  done
done
