for c in c2 c1; do for r in 36 37 48 56 72 74 96 111 148; do
python bench.py --config $c --ranks $r --split 1 --steps 5 --warmup 3 --no-e2e --no-cpu --no-check 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$c',$r,round(d['value']),round(d['solve_roofline']['frac'],3),{k:round(v,2) for k,v in d['phases_ms'].items()})"
done; done
