python -m pytest tests/test_gpu_shard.py -q -m gpu -x > gpurun_out/t_fshard.log 2>&1; echo tests rc=$?
python tools/shard_projection.py --config c4 --worlds 1 2 4 8 > gpurun_out/proj2.txt 2>&1
python tools/shard_projection.py --config c4 --worlds 8 --split 9 >> gpurun_out/proj2.txt 2>&1
python tools/shard_projection.py --config c4 --worlds 8 --split 5 >> gpurun_out/proj2.txt 2>&1
python tools/shard_projection.py --config c4 --worlds 8 --split 1 >> gpurun_out/proj2.txt 2>&1
