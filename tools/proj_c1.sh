for rpg in 18 24 28 37 74; do python tools/shard_projection.py --config c1 --worlds 8 --ranks-per-gpu $rpg; done > gpurun_out/proj6.txt 2>&1
for rpg in 18 28 37; do python tools/shard_projection.py --config c1 --worlds 4 --ranks-per-gpu $rpg; done >> gpurun_out/proj6.txt 2>&1
for rpg in 18 37 74; do python tools/shard_projection.py --config c2 --worlds 8 --ranks-per-gpu $rpg; done >> gpurun_out/proj6.txt 2>&1
