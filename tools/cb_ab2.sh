python -m pytest tests/test_gpu_parity.py -q -x -k "column_sweep_chunked" 2>&1 | grep -E "Error|assert|max_abs|passed|failed" | head -20
run() { env "$@" python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['value'],1), round(d['roofline']['launch_ms'],2), d['gpu_launches'])" || tail -3 /tmp/err.txt; }
run CPG_CB_DEG=0
run CPG_CB_DEG=4096 CPG_CB_DEBUG=1
grep "\[cpg\]" /tmp/err.txt
run CPG_CB_DEG=4096 CPG_HOT_MB=0
run CPG_CB_DEG=4096 CPG_CB_MB=32
run CPG_CB_DEG=4096 CPG_CB_MB=32 CPG_HOT_MB=0
run CPG_CB_DEG=2048 CPG_CB_DEBUG=1
grep "\[cpg\]" /tmp/err.txt
run CPG_CB_DEG=2048 CPG_HOT_MB=0
run CPG_CB_DEG=8192
run CPG_CB_DEG=1024 CPG_CB_MB=32 CPG_HOT_MB=0
