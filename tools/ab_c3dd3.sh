python -m pytest tests/test_gpu_parity.py -q -m gpu -k "schur_dd" > gpurun_out/t_dd.log 2>&1; echo tests rc=$?
for r in 1 2; do python bench.py --config c3dd --steps 5 --warmup 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3dd', round(d['value'],1), round(d['ms_per_step'],2), d['grid_rel_residual'])"; done
