#!/bin/bash
run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'RHS/s=%.0f'%d['value'], d.get('phases_ms'), d['solve_roofline']['frac'])"
}
run base "X=0" --config c2
run f20 "BTD_CHAIN_VARIANT=20 BTD_CHAIN_VARIANT_BWD=0" --config c2
run base "X=0" --config c3dd
run f7 "BTD_CHAIN_VARIANT=7 BTD_CHAIN_VARIANT_BWD=0" --config c3dd
run f12 "BTD_CHAIN_VARIANT=12 BTD_CHAIN_VARIANT_BWD=0" --config c1
