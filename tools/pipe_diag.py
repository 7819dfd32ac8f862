import sys, time, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import bench, paper_2412_10789_b200 as P
cfg = dict(bench.CONFIGS[4])
csr = bench.make_device_csr(cfg, 0)
dg = P.DeviceGraph.from_device(csr)
n = csr.n
kern = P.Kernel.hkpr(5.0); K = 15; c = np.ascontiguousarray(kern.cheby_coeffs(K))
src = np.ascontiguousarray(P.select_sources_uniform(n, 64, 1), dtype=np.uint32)
L = P._lib.lib()
outs = [torch.empty((64, n), dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
def call(i, fn):
    st = P._lib.cpg_stats()
    P._check(getattr(L, fn)(dg.handle, P._f64p(c), K, P._u32p(src), 64, 64, outs[i % 2].ctypes.data, ctypes.byref(st)))
    return st
for fn in ["cpg_chebypower_batched", "cpg_chebypower_batched_async"]:
    call(0, fn); L.cpg_graph_sync(dg.handle)
    ts = []
    t0 = time.perf_counter()
    for i in range(4):
        t = time.perf_counter(); st = call(i, fn); ts.append(time.perf_counter() - t)
    L.cpg_graph_sync(dg.handle)
    tot = time.perf_counter() - t0
    print(fn, "per-call s", [round(x, 4) for x in ts], "total", round(tot, 4), "device_ms", round(st.device_ms, 2), "wall", round(st.wall_seconds, 4))
