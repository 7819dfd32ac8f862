"""Fraction of the gathers (edge endpoints) that land in the top-X rows of the degree order,
for a BASELINE config: the L2 hit rate a perfect hot-row cache of X rows would give.
    python tools/degree_coverage.py <config>"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

cfg = bench.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
csr = bench.make_device_csr(cfg, 0)
off = np.empty(csr.n + 1, dtype=np.uint64)
import ctypes  # noqa: E402

import paper_2412_10789_b200 as P  # noqa: E402

off, _ = csr.to_host()
deg = np.sort(np.diff(off.astype(np.int64)))[::-1]
cum = np.cumsum(deg) / deg.sum()
n = len(deg)
B = 16 if cfg.get("tile", 64) == 16 else 64
for mb in (16, 32, 64, 96, 126, 256, 512, 1024):
    rows = min(n, (mb << 20) // (8 * B))
    print(f"top {rows:>10d} rows ({mb:4d} MB of the B={B} iterate): {100 * cum[rows - 1]:5.1f}% of gathers")
print("n", n, "nnz", int(deg.sum()), "max deg", int(deg[0]))
