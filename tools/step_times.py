"""Per-step kernel times of one query (tile) of a bench config, for several
CPG_SPARSE_STEPS settings (diagnostics for DESIGN.md 4.7).

    python tools/step_times.py --config 5 --mode batched --M 0,1,2,3

Prints the library's per-step CUDA-event times (CPG_PROF_DUMP) for each M.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--M", default="0,1,2,3")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_2412_10789_b200 as P

    cfg = dict(bench.CONFIGS[args.config])
    if args.mode:
        cfg["mode"] = args.mode
    kernel = P.Kernel.ppr(cfg["param"]) if cfg["family"] == bench.PPR else P.Kernel.hkpr(cfg["param"])
    K = P.plan_truncation(kernel, cfg["eps"]).cheby_steps
    c_np = np.ascontiguousarray(kernel.cheby_coeffs(K))
    csr = bench.make_device_csr(cfg, 0)
    dg = P.DeviceGraph.from_device(csr)
    torch.cuda.synchronize()
    sources = P.select_sources_uniform(csr.n, cfg["sources"], 1)
    batched = cfg["mode"] == "batched"
    tile = int(cfg.get("tile", min(64, len(sources))))
    src = np.ascontiguousarray(sources[:tile] if batched else sources[:1], dtype=np.uint32)
    L = P._lib.lib()
    os.environ["CPG_PROF_DUMP"] = "1"
    os.environ["CPG_GROUP_Q"] = "1"
    for M in args.M.split(","):
        os.environ["CPG_SPARSE_STEPS"] = M
        for rep in range(args.reps):
            L.cpg_set_profiling(1)
            s = P._lib.cpg_stats()
            print(f"M={M} rep={rep}", file=sys.stderr, flush=True)
            if batched:
                P._check(L.cpg_chebypower_batched(dg.handle, P._f64p(c_np), K, P._u32p(src), len(src), tile, None,
                                                  ctypes.byref(s)))
            else:
                P._check(L.cpg_chebypower(dg.handle, P._f64p(c_np), K, P._u32p(src), len(src), None,
                                          ctypes.byref(s)))
            L.cpg_set_profiling(0)
            print(f"M={M} rep={rep} step_ms_total={s.step_ms:.3f} device_ms={s.device_ms:.3f}", flush=True)
    dg.close()


if __name__ == "__main__":
    main()
