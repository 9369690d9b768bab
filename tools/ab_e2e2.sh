for c in c1 c2; do for w in 32 64 128; do BTD_HOST_MINW=$w python bench.py --config $c --steps 5 --no-cpu --no-check 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c minw $w', round(d['value']), 'e2e', round(d['e2e']['value']))"; done; done
