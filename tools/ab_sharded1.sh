# One-GPU cost of the multi-GPU machinery: plain, 1-rank sharded (NCCL chunks), fused all-gather
# (barrier only), fused all-gather with stores through the rank's own LSA alias.
for c in 5 4; do
  python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c plain', round(d['value'],1), d['config']['parallelism'], d['config'].get('allgather'))"
  python bench.py --config $c --sharded --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c sharded', round(d['value'],1), d['config']['parallelism'], d['config'].get('allgather'))"
  python bench.py --config $c --sharded --fused-allgather --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c fused', round(d['value'],1), d['config']['parallelism'], d['config'].get('allgather'))"
  CPG_P2P_SELF=1 python bench.py --config $c --sharded --fused-allgather --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c fused+self-stores', round(d['value'],1), d['config']['parallelism'], d['config'].get('allgather'))"
done
