# c4 cross-product: 8/16/32/64 subdomains per GPU x 1/2/4/8 GPUs,
# split = floor(592 / subdomains per GPU) (one wave of device ranges per GPU)
for w in 1 2 4 8; do for spg in 8 16 32 64; do
  python tools/shard_projection.py --config c4 --worlds $w --ranks-per-gpu $spg --split $((592 / spg))
done; done > gpurun_out/proj_cross.txt 2>&1
