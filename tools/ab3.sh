#!/bin/bash
run() {
  python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print(c['workload'], 'P=%d split=%d'%(c['ranks'],c['split']), 'RHS/s=%.0f'%d['value'], 'ms=%.2f'%d['ms_per_step'], 'fwd=%.2f tree=%.2f bwd=%.2f'%(d['phases_ms']['forward'],d['phases_ms']['interface_tree'],d['phases_ms']['backward']), 'solve_frac=%.3f'%d['solve_roofline']['frac'])"
}
python -m pytest tests -m gpu -q -x 2>&1 | tail -1; for c in c3 c1 c4 c2; do run --config $c; done; echo -n "legacy "; BTD_GEMM_LEGACY=1 run --config c3
