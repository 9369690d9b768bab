python tools/shard_projection.py --config c4 --worlds 1 2 4 8
python tools/shard_projection.py --config c4 --worlds 8 --split 9
python tools/shard_projection.py --config c4 --worlds 8 --split 5
python tools/shard_projection.py --config c1 --worlds 1 2 4 8
python tools/shard_projection.py --config c2 --worlds 1 2 4 8
