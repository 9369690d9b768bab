# e2e (host-buffer API) vs host-pipeline chunk width (BTD_HOST_MINW) and chunk count
for spec in "c4 32 8" "c4 16 8" "c4 8 8" "c1 64 8" "c1 32 8" "c2 128 8" "c2 64 8"; do
set -- $spec
BTD_HOST_MINW=$2 BTD_HOST_CHUNKS=$3 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu --no-check 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$1 minw=$2 chunks=$3',round(d['value']),'e2e',round(d['e2e']['value']))"
done
