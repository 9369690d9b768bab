#!/bin/bash
run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'P=%d'%c['ranks'], 'RHS/s=%.0f'%d['value'], 'fwd=%.2f tree=%.2f bwd=%.2f'%(d['phases_ms']['forward'],d['phases_ms']['interface_tree'],d['phases_ms']['backward']), 'solve_frac=%.3f'%d['solve_roofline']['frac'])"
}
run base "BTD_CHAIN_VARIANT=0" --config c2
run b5 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=5" --config c2
run b10 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=10" --config c2
run b19 "BTD_CHAIN_VARIANT=0 BTD_CHAIN_VARIANT_BWD=19" --config c2
run b13P74 "BTD_CHAIN_VARIANT=0" --config c2 --ranks 74
run c4r8 "BTD_CHAIN_VARIANT=0" --config c4 --ranks 8 --split 74
run c4r16 "BTD_CHAIN_VARIANT=0" --config c4 --ranks 16 --split 37
run c4r32 "BTD_CHAIN_VARIANT=0" --config c4 --ranks 32 --split 19
run c4r64 "BTD_CHAIN_VARIANT=0" --config c4 --ranks 64 --split 10
