run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', 'P=%d split=%d'%(c['ranks'],c['split']), 'RHS/s=%.0f'%d['value'], {k:round(v,3) for k,v in d['phases_ms'].items()}, round(d['solve_roofline']['frac'],3))"
}
for rep in 1 2; do
run n3s74 "X=0" --config c4 --ranks 8 --split 74
run n4s55 "BTD_STREAM_NSTG=4" --config c4 --ranks 8 --split 55
run n4s74 "BTD_STREAM_NSTG=4" --config c4 --ranks 8 --split 74
run n4s111 "BTD_STREAM_NSTG=4" --config c4 --ranks 8 --split 111
done
