#!/bin/bash
run() {
  python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print(c['workload'], 'P=%d split=%d'%(c['ranks'],c['split']), 'RHS/s=%.0f'%d['value'], 'ms=%.2f'%d['ms_per_step'], 'fwd=%.2f tree=%.2f bwd=%.2f'%(d['phases_ms']['forward'],d['phases_ms']['interface_tree'],d['phases_ms']['backward']), 'solve_frac=%.3f'%d['solve_roofline']['frac'])"
}
for v in 0 2 3 4; do echo -n "v$v "; BTD_CHAIN_VARIANT=$v run --config c2; done; run --config c4
