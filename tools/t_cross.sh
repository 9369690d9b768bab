python -m pytest tests/test_gpu_shard.py -q -m gpu -x > gpurun_out/t_cross.log 2>&1; echo tests rc=$?
python tools/shard_projection.py --config c1 --worlds 1 2 4 8 > gpurun_out/proj4.txt 2>&1
python tools/shard_projection.py --config c2 --worlds 1 2 4 8 >> gpurun_out/proj4.txt 2>&1
python tools/shard_projection.py --config c3 --worlds 1 2 4 8 >> gpurun_out/proj4.txt 2>&1
