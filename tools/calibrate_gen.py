"""Calibrate generator draw counts against the BASELINE.json config sizes (GPU)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2412_10789_b200 as P

for spec in sys.argv[1:]:
    kind, *args = spec.split(":")
    t = time.time()
    if kind == "rmat":
        scale, samples = int(args[0]), int(float(args[1]))
        csr = P.gen_rmat(scale, samples, seed=5, device=0)
    else:
        n_ids, samples, expo, mean, cap = int(args[0]), int(float(args[1])), float(args[2]), float(args[3]), int(args[4])
        csr = P.gen_chunglu(n_ids, samples, expo, mean, cap, seed=4, device=0)
    print(spec, "n", csr.n, "m", csr.nnz // 2, "mean_deg", csr.nnz / csr.n, f"{time.time()-t:.1f}s", flush=True)
    csr.close()
