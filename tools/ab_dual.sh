run() { lab=$1; envs=$2; shift 2
  env $envs python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print('$lab', c['workload'], 'RHS/s=%.0f'%d['value'], {k:round(v,3) for k,v in d['phases_ms'].items()}, round(d['solve_roofline']['frac'],3), d['rel_residual'])"
}
for rep in 1 2; do
run base "X=0" --config c1
run dual4 "BTD_CHAIN_VARIANT=18 BTD_CHAIN_VARIANT_BWD=0" --config c1
run dual8 "BTD_CHAIN_VARIANT=19 BTD_CHAIN_VARIANT_BWD=0" --config c1
run base "X=0" --config c2
run dual4 "BTD_CHAIN_VARIANT=21 BTD_CHAIN_VARIANT_BWD=0" --config c2
done
