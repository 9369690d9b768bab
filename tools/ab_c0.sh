for s in 1 4 8 16 32; do python bench.py --config c0 --split $s --steps 20 --no-cpu --no-check 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split $s', round(d['value']), round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['phases_ms'].items()}, 'e2e', round(d['e2e']['value']))"; done
