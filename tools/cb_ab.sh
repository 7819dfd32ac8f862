set -x
python -m pytest tests/test_gpu_parity.py -q -x -k "column_blocked or split_and_fused" 2>&1 | tail -3
for cfg in "0 48" "32768 48" "16384 48" "65536 48" "32768 32" "32768 80"; do
  set -- $cfg
  CPG_CB_DEG=$1 CPG_CB_MB=$2 python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('CB', '$1', '$2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
done
for c in 4 3; do for deg in 0 32768 16384; do
  CPG_CB_DEG=$deg python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('C$c', '$deg', d['value'], d['ms_per_step'])"
done; done
