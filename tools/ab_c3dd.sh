for r in 144 148; do python bench.py --config c3dd --steps 3 --warmup 2 --ranks $r 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$r', d['value'], d['solve_roofline']['frac'], d['config'])"; done
