#!/bin/bash
run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'P=%d split=%d'%(c['ranks'],c['split']), 'RHS/s=%.0f'%d['value'], 'fwd=%.2f tree=%.2f bwd=%.2f'%(d['phases_ms']['forward'],d['phases_ms']['interface_tree'],d['phases_ms']['backward']), 'solve_frac=%.3f'%d['solve_roofline']['frac'])"
}
run base "X=0" --config c1
run b10 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=10" --config c1
run b13 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=13" --config c1
run f11 "BTD_CHAIN_VARIANT=11 BTD_CHAIN_VARIANT_BWD=0" --config c1
run f12 "BTD_CHAIN_VARIANT=12 BTD_CHAIN_VARIANT_BWD=0" --config c1
run base "X=0" --config c1
