#!/bin/bash
# A/B of chain-kernel shapes after per-column-group named barriers (BTD_CHAIN_VARIANT[_BWD])
run() { # label "ENV=.. ENV=.." --config cX
  lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'P=%d'%c['ranks'], 'RHS/s=%.0f'%d['value'], 'fwd=%.2f tree=%.2f bwd=%.2f'%(d['phases_ms']['forward'],d['phases_ms']['interface_tree'],d['phases_ms']['backward']), 'solve_frac=%.3f'%d['solve_roofline']['frac'])"
}
run base "BTD_CHAIN_VARIANT=0" --config c2
run v17 "BTD_CHAIN_VARIANT=17" --config c2
run b7 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=7" --config c2
run f15 "BTD_CHAIN_VARIANT=15 BTD_CHAIN_VARIANT_BWD=0" --config c2
run f16 "BTD_CHAIN_VARIANT=16 BTD_CHAIN_VARIANT_BWD=0" --config c2
run f18b18 "BTD_CHAIN_VARIANT=18" --config c2
run base "BTD_CHAIN_VARIANT=0" --config c3dd
