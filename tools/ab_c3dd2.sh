for v in "0 0" "9 0" "9 9"; do set -- $v; BTD_CHAIN_VARIANT=$1 BTD_CHAIN_VARIANT_BWD=$2 python bench.py --config c3dd --steps 3 --warmup 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fwd v$1 bwd v$2', d['value'], d['solve_roofline']['frac'])"; done
