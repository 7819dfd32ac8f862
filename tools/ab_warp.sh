# Warp-tile single-source step (CPG_WARP_TILES=1) vs the CTA tiles, interleaved, configs 3 and 5 (+ 1, 2 groups unaffected).
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "warp_tile or tile_widths or large_graph" 2>&1 | tail -2
for cfg in "3" "5 --mode single --steps 2"; do
  for rep in 1 2; do
    for wt in 0 1; do
      CPG_WARP_TILES=$wt python bench.py --config $cfg --no-cpu-baseline --warmup 2 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg warp=$wt', round(d['value'],1), round(d['ms_per_step'],2), 'launch_ms', round(r['launch_ms'],4), 'gather_frac', round(r.get('frac_gather_ceiling') or 0,3), 'mass', d['mass_err_max'])"
    done
  done
done
