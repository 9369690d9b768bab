#!/bin/bash
run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'RHS/s=%.0f'%d['value'], {k:round(v,2) for k,v in d.get('phases_ms').items()}, round(d['solve_roofline']['frac'],3))"
}
run base "X=0" --config c1
run b14 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=14" --config c1
run b15 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=15" --config c1
run b17 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=17" --config c1
