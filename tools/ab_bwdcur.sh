python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_shard.py -q -m gpu -x > gpurun_out/t_bc.log 2>&1; echo tests rc=$?
for rep in 1 2; do for c in c1 c2; do python bench.py --config $c --steps 10 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['solve_roofline']['frac'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, d['rel_residual'])"; done; done
python bench.py --config c3dd --steps 3 --warmup 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3dd', round(d['value'],1), d['grid_rel_residual'])"
