python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_schur_system.py -q -m gpu -x > gpurun_out/t_fork.log 2>&1; echo tests rc=$?
for r in 1 2; do python bench.py --config c3 --steps 10 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value']), round(d['solve_roofline']['frac'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, round(d['e2e']['value']), d['rel_residual'])"; done
python tools/shard_projection.py --config c3 --worlds 2 8
