python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_c3split.log 2>&1; echo tests rc=$?
python tools/shard_projection.py --config c3 --worlds 1 2 4 8 > gpurun_out/proj5.txt 2>&1
python bench.py --config c3 --steps 5 --no-e2e --no-cpu > gpurun_out/b_c3.json 2>&1
