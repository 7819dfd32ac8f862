"""How many gathers of hub rows land in the warm tier of the degree order (rows past the
L2-resident hot prefix but still gathered hundreds of times per step): the gathers a
column-window schedule of the hub pieces could turn into L2 hits.
    python tools/cb_stats.py [config]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

cfg = bench.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
csr = bench.make_device_csr(cfg, 0)
off, nb = csr.to_host()
csr.close()
n = len(off) - 1
dev = torch.device("cuda:0")
deg = torch.from_numpy(np.diff(off.astype(np.int64))).to(dev)
order = torch.argsort(deg, descending=True, stable=True)
rank = torch.empty(n, dtype=torch.int32, device=dev)
rank[order] = torch.arange(n, dtype=torch.int32, device=dev)
nnz = int(deg.sum())
B = 16 if cfg.get("tile", 64) == 16 else 64
hot = (64 << 20) // (8 * B)
tiers = [(mb, (mb << 20) // (8 * B)) for mb in (128, 256, 512, 1024, 2048)]
Ts = (32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768)
res = {T: {"rows": int((deg > T).sum()), "edges": 0, "hot": 0, **{mb: 0 for mb, _ in tiers}} for T in Ts}
nbt = torch.from_numpy(nb.view(np.int32))
off_t = torch.from_numpy(off.astype(np.int64))
CH = 1 << 22  # rows per chunk
for r0 in range(0, n, CH):
    r1 = min(n, r0 + CH)
    e0, e1 = int(off_t[r0]), int(off_t[r1])
    if e1 == e0:
        continue
    d = deg[r0:r1]
    rowdeg = torch.repeat_interleave(d, d)
    cr = rank[nbt[e0:e1].to(dev).long()]
    for T in Ts:
        m = rowdeg > T
        c = cr[m]
        res[T]["edges"] += int(m.sum())
        res[T]["hot"] += int((c < hot).sum())
        for mb, rows in tiers:
            res[T][mb] += int(((c >= hot) & (c < rows)).sum())
print(f"n {n} nnz {nnz} B {B} hot prefix {hot} rows (64 MB)")
for T in Ts:
    r = res[T]
    line = f"rows with degree > {T:6d}: {r['rows']:8d} rows, {r['edges'] / 1e6:8.1f} M edges ({100 * r['edges'] / nnz:4.1f}% of nnz); "
    line += f"hot prefix {r['hot'] / 1e6:7.1f} M; warm up to " + ", ".join(f"{mb} MB: {r[mb] / 1e6:6.1f} M" for mb, _ in tiers)
    print(line)
