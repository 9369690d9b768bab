# the NCCL flavour of the sharded path at world 1 (bench.py --sharded): ShardedPlan, the 3-phase
# shard API with fused shard-tree kernels (M <= 32), NCCL all-gathers, pipelined host solve
for c in c4 c1 c0; do python bench.py --config $c --sharded --steps 5 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c sharded(w1,nccl)', round(d['value']), 'e2e', round(d['e2e']['value']), 'res', d['rel_residual'], d['config']['parallelism'])"; done
