# PDL A/B (CPG_PDL=0/1) on the paths that use it, interleaved on one box.
for cfg in "1" "2" "3" "1 --mode single" "2 --mode single" "5 --mode single --steps 2"; do
  for pdl in 0 1 0 1; do
    CPG_PDL=$pdl python bench.py --config $cfg --no-cpu-baseline --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg pdl=$pdl', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'mass_err', d.get('mass_err_max'))"
  done
done
