for c in c1 c3 c2; do python bench.py --config $c --steps 10 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['solve_roofline']['frac'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, d['rel_residual'])"; done
