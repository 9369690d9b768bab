#!/bin/bash
run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'P=%d split=%d'%(c['ranks'],c['split']), 'RHS/s=%.0f'%d['value'], 'fwd=%.2f tree=%.2f bwd=%.2f'%(d['phases_ms']['forward'],d['phases_ms']['interface_tree'],d['phases_ms']['backward']), 'solve_frac=%.3f'%d['solve_roofline']['frac'])"
}
run base "X=0" --config c2
run base "X=0" --config c1
run c4r8 "X=0" --config c4
run c4r32s37 "X=0" --config c4 --ranks 32 --split 37
run c4r64s37 "X=0" --config c4 --ranks 64 --split 37
run c4r128s37 "X=0" --config c4 --ranks 128 --split 37
run c4r512s37 "X=0" --config c4 --ranks 512 --split 37
