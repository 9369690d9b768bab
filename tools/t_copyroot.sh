python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_shard.py tests/test_gpu_plan_io.py tests/test_gpu_schur_system.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/t_cr.log 2>&1; echo tests rc=$?
for c in c1 c3; do python bench.py --config $c --steps 10 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['solve_roofline']['frac'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, d['rel_residual'])"; done
