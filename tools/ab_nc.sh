run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-check "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'RHS/s=%.0f'%d['value'], {k:round(v,2) for k,v in (d.get('phases_ms') or {}).items()}, round(d['solve_roofline']['frac'],3))"
}
for c in c1 c2 c4 c3; do
run cg "X=0" --config $c
run nc "BTD_LIB_PATH=paper_1108_4181_b200/_lib/alt/nc.so" --config $c
done
run cg "X=0" --config c3dd
run nc "BTD_LIB_PATH=paper_1108_4181_b200/_lib/alt/nc.so" --config c3dd
