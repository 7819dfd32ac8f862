set -x
python -m pytest tests/test_gpu_sparse_steps.py -x -q 2>&1 | tail -15
source tools/ab_sparse.sh
for M in 0 2 3; do CPG_SPARSE_STEPS=$M run c5_b16_M$M --steps 4 --warmup 3; done
for M in 0 3 4; do CPG_SPARSE_STEPS=$M run c3_single_M$M --config 3 --steps 3 --warmup 3; done
