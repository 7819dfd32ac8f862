# e2e with deferred pipelined calls on configs 1, 2, 4, 5; the one-rank sharded bench path; the bench
# under torchrun with one rank; the GPU suite.
for cfg in 1 2 4; do
  python bench.py --config $cfg --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'same', d['e2e_matches_device_run'], 'mass', d['mass_err_max'])"
done
python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg 5', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'same', d['e2e_matches_device_run'], 'mass', d['mass_err_max'], 'frac', d['roofline']['frac'])"
python bench.py --config 4 --sharded --no-cpu-baseline --steps 3 --warmup 3 2>gpurun_out/sharded_c4.err | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg 4 sharded(1 rank NCCL)', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['config']['parallelism'], d['config']['allgather'], 'same', d['e2e_matches_device_run'])"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --config 2 --no-cpu-baseline --steps 3 --warmup 3 2>gpurun_out/torchrun1.err | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('torchrun nproc1 cfg2', round(d['value'],1), d['n_gpus'])"

