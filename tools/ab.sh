#!/bin/bash
# A/B chain-kernel variants: prints value, ms/step, phases
run() { # env... -- bench args
  python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print(c['workload'], 'P=%d split=%d'%(c['ranks'],c['split']), 'RHS/s=%.0f'%d['value'], 'ms=%.2f'%d['ms_per_step'], 'fwd=%.2f tree=%.2f bwd=%.2f'%(d['phases_ms']['forward'],d['phases_ms']['interface_tree'],d['phases_ms']['backward']), 'solve_frac=%.3f'%d['solve_roofline']['frac'])"
}
for v in 0 1 2; do echo -n "v$v "; BTD_CHAIN_VARIANT=$v run --config c1; done
for v in 0 1 2; do echo -n "v$v "; BTD_CHAIN_VARIANT=$v run --config c2; done
echo -n "v0 P18 "; BTD_CHAIN_VARIANT=0 run --config c2 --ranks 18
echo -n "v2 P18 "; BTD_CHAIN_VARIANT=2 run --config c1 --ranks 36
echo -n "c4 s148 "; run --config c4 --split 148
echo -n "c4 s37 "; run --config c4 --split 37
