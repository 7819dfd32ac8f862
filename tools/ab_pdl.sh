set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build4.log 2>&1 || exit 1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; tail -2 gpurun_out/pytest_gpu4.log
for cfg in "1" "2" "1 --mode single" "2 --mode single" "3 --mode single" "3" "4"; do
  for pdl in 0 1 0 1; do
    CPG_PDL=$pdl python bench.py --config $cfg --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg pdl=$pdl', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1))"
  done
done > gpurun_out/pdl_ab.txt 2>&1
cat gpurun_out/pdl_ab.txt
ncu --set full -k regex:k_ldg -c 1 -o gpurun_out/ncu_gather_ldg ./tools/gather_l2 > gpurun_out/ncu_gather.log 2>&1
