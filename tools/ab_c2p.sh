for r in 37 74 111; do for rep in 1 2; do python bench.py --config c2 --ranks $r --split 1 --steps 10 --no-e2e --no-cpu --no-check 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2 P=$r', round(d['value']), round(d['solve_roofline']['frac'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})"; done; done
