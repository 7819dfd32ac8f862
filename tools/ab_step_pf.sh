# A/B of the software-pipelined single-source step (CPG_STEP_PF) on configs 1,2,3 and 5-single.
CPG_STEP_PF=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -x 2>&1 | tail -2
run() { pf=$1; shift; CPG_STEP_PF=$pf python bench.py --no-cpu-baseline --steps 3 --warmup 3 "$@" 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('PF=$pf $*', round(d['value'],1), round(d['roofline']['launch_ms'],4))" || tail -3 /tmp/err.txt; }
for c in 3 1 2; do run 0 --config $c; run 1 --config $c; done
run 0 --config 5 --mode single
run 1 --config 5 --mode single
