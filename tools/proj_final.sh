python tools/shard_projection.py --config c1 --worlds 1 2 4 8
python tools/shard_projection.py --config c2 --worlds 1 2 4 8
python tools/shard_projection.py --config c2 --worlds 4 --ranks-per-gpu 37
python tools/shard_projection.py --config c4 --worlds 1 2 4 8
python tools/shard_projection.py --config c3 --worlds 1 2 4 8
