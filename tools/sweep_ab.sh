python -m pytest tests/test_gpu_parity.py -q -x -k "column_sweep or column_blocked" 2>&1 | tail -3
run() { env "$@" python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['value'],1), round(d['roofline']['launch_ms'],2), d['gpu_launches'])" || tail -3 /tmp/err.txt; }
run CPG_SWEEP=0
run CPG_SWEEP=1 CPG_CB_DEBUG=1
grep "\[cpg\]" /tmp/err.txt
run CPG_SWEEP=1 CPG_HOT_MB=0
run CPG_SWEEP=1 CPG_SWEEP_MB=24
run CPG_SWEEP=1 CPG_SWEEP_MB=64
run CPG_SWEEP=1 CPG_SWEEP_DRIFT=2 CPG_SWEEP_MB=24
run CPG_SWEEP=1 CPG_SWEEP_CFG=43
run CPG_SWEEP=1 CPG_SWEEP_CFG=83
run CPG_SWEEP=1 CPG_SWEEP_DEG=128
run CPG_SWEEP=1 CPG_CB_DEG=0
