python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_fshard2.log 2>&1; echo tests rc=$?
python tools/shard_projection.py --config c4 --worlds 1 2 4 8 > gpurun_out/proj3.txt 2>&1
python tools/shard_projection.py --config c4 --worlds 4 --split 37 >> gpurun_out/proj3.txt 2>&1
python tools/shard_projection.py --config c4 --worlds 8 --split 18 >> gpurun_out/proj3.txt 2>&1
python tools/shard_projection.py --config c4 --worlds 8 --split 12 >> gpurun_out/proj3.txt 2>&1
python tools/shard_projection.py --config c0 --worlds 1 2 4 >> gpurun_out/proj3.txt 2>&1
python bench.py --config c4 > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err
