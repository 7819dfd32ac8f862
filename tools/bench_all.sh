# Every config's bench line (+ CPU baseline) into gpurun_out/configs/, the default
# headline run and the reference arm.  Used to refresh profiles/<round>/configs.
mkdir -p gpurun_out/configs
run() { name=$1; shift; python bench.py "$@" > gpurun_out/configs/$name.json.tmp 2> gpurun_out/configs/$name.log; tail -1 gpurun_out/configs/$name.json.tmp > gpurun_out/configs/$name.json; rm -f gpurun_out/configs/$name.json.tmp; python -c "import json; d=json.load(open('gpurun_out/configs/$name.json')); print('$name', round(d['value'],1), d.get('e2e',{}).get('value'), (d.get('cpu_baseline') or {}).get('value'))" || tail -3 gpurun_out/configs/$name.log; }
run cfg_1_single --config 1 --mode single --steps 5 --warmup 3
run cfg_1_batched --config 1 --mode batched --tile 16 --steps 5 --warmup 3
run cfg_2_single --config 2 --mode single --steps 5 --warmup 3
run cfg_2_batched --config 2 --mode batched --tile 64 --steps 5 --warmup 3
run cfg_3_single --config 3 --steps 3 --warmup 3
run cfg_3_batched --config 3 --mode batched --tile 64 --steps 3 --warmup 3
run cfg_4_batched --config 4 --steps 3 --warmup 3
run cfg_5_single --config 5 --mode single --steps 2 --warmup 3
run bench_default_c5 --steps 5 --warmup 3
run bench_reference_c5 --impl reference --steps 2 --warmup 1
