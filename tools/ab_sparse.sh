#!/bin/bash
# A/B of the sparse early steps: CPG_SPARSE_STEPS = 0 (off) vs the
# default vs other M, per config/path.  Lines into gpurun_out/ab_sparse/.
mkdir -p gpurun_out/ab_sparse
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_sparse/$name.json 2> gpurun_out/ab_sparse/$name.log; python -c "import json; d=json.load(open('gpurun_out/ab_sparse/$name.json')); print('$name', round(d['value'],1), round(d['e2e']['value'],1), d['config'].get('sparse_early_steps'), round(d['roofline']['launch_ms'],3))" || tail -3 gpurun_out/ab_sparse/$name.log; }
for cfgargs in "${@}"; do :; done
