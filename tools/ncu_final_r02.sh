#!/bin/bash
# full ncu captures (one launch each) of the sweep kernels of c4, c1, c2 with the final round-2 code
O=gpurun_out/r02c; mkdir -p $O
for spec in "c4 stream_bwd_kernel" "c1 chain_bwd_kernel" "c2 chain_fwd_kernel" "c2 chain_bwd_kernel"; do
  set -- $spec; c=$1; k=$2
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu --no-check"
  $CMD > /dev/null 2>&1 && ncu -f --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/ncu_${c}_$k $CMD > $O/ncu_${c}_$k.log 2>&1
  echo "$c $k rc=$?"
done
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f; done > $O/ncu_full_sweeps_final.txt 2>&1
rm -f $O/*.ncu-rep
