python -m pytest tests/test_gpu_shard.py tests/test_abi.py -q -m gpu -x > gpurun_out/t_shard.log 2>&1; echo rc=$?
python bench.py --config c1 --sharded --steps 3 --warmup 3 --no-cpu > gpurun_out/b_c1_sh.json 2>gpurun_out/b_c1_sh.err; echo rc=$?
OUT=gpurun_out/shard_gloo2 bash tools/shard_gloo_1gpu.sh
