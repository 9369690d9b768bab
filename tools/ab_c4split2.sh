run() { lab=$1; shift
  python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'P=%d split=%d'%(c['ranks'],c['split']), 'RHS/s=%.0f'%d['value'], {k:round(v,3) for k,v in d['phases_ms'].items()}, round(d['solve_roofline']['frac'],3))"
}
for s in 74 148 222 296 370 444; do run s$s --config c4 --ranks 8 --split $s; done
run p64s37 --config c4 --ranks 64 --split 37
run s74again --config c4 --ranks 8 --split 74
