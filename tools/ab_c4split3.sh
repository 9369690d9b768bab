for rep in 1 2; do for s in 74 296 222; do
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-check --config c4 --ranks 8 --split $s 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('split $s', round(d['value']), round(d['ms_per_step'],3), round(d['solve_roofline']['frac'],3), round(d['phases_ms']['total'],3))"
done; done
