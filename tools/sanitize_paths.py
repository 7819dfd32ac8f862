"""Run every kernel path of libcpg once on a small graph, checked against the oracle,
so compute-sanitizer (memcheck / racecheck / synccheck) can watch each of them:

    compute-sanitizer --tool memcheck python tools/sanitize_paths.py <path>

Paths: single (combined step kernel, PDL), single_split (hub + tile kernels), group
(query-group kernel), fused16 / fused64 (fused batched kernel, PDL), split16 / split64
(hub-piece + plain-row kernels), loopback (sharded layout, R = 3, C = 2, one GPU),
p2p_self (fused all-gather through the NCCL symmetric window, own LSA alias),
measure, topk.  Exits non-zero on a parity failure.
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(path: str) -> None:
    env = {
        "single_split": {"CPG_STEP_SPLIT": "1"},
        "group": {"CPG_GROUP_Q": "4"},
        "split16": {"CPG_BATCH_SPLIT": "1"},
        "split64": {"CPG_BATCH_SPLIT": "1"},
        "fused16": {"CPG_BATCH_SPLIT": "0"},
        "fused64": {"CPG_BATCH_SPLIT": "0"},
        "p2p_self": {"CPG_P2P": "1", "CPG_P2P_SELF": "1"},
    }.get(path, {})
    os.environ.update(env)
    import paper_2412_10789_b200 as P
    from oracle import Port

    off, nb = P.gen_chunglu(6000, 40000, 2.1, 12.0, 3000, seed=4)  # hub rows split into pieces
    n = len(off) - 1
    k = P.Kernel.ppr(0.2)
    K = 12
    c = k.cheby_coeffs(K)
    src = [0, 5, n // 2, n - 1]
    want = np.stack([Port.cheby_power(off, nb, c, K, s)[0] for s in src])
    g = P.Graph.from_csr(off, nb)
    if path in ("single", "single_split"):
        got = np.stack([P.cheby_power(g, k, s, K).values for s in src])
    elif path == "group":
        got, _ = P.cheby_power_many(g, k, src, K)
    elif path in ("fused16", "split16", "fused64", "split64"):
        got, _ = P.cheby_power_many(g, k, src, K, batched=True, tile=16 if path.endswith("16") else 64)
    elif path == "loopback":  # R = 3 shards on one GPU, one host thread per rank
        import threading

        os.environ["CPG_CHUNKS"] = "2"
        grp = P.LoopbackGroup(3)
        parts = [P.DeviceGraph.loopback(off, nb, r, grp) for r in range(3)]
        res = [None] * 3

        def work(r):
            res[r] = (P.cheby_power_many(parts[r], k, src, K)[0],
                      P.cheby_power_many(parts[r], k, src, K, batched=True, tile=8)[0])

        th = [threading.Thread(target=work, args=(r,)) for r in range(3)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        got = res[0][0]
        for r in range(3):
            for a in res[r]:
                assert np.abs(a - want).max() <= 1e-12, r
    elif path == "p2p_self":
        import torch  # noqa: F401  (the torch-bundled NCCL carries the device API)

        offs = np.ascontiguousarray(off, np.uint64)
        nbs = np.ascontiguousarray(nb, np.uint32)
        dg = P.DeviceGraph.sharded(offs.ctypes.data_as(ctypes.c_void_p), nbs.ctypes.data_as(ctypes.c_void_p), n,
                                   len(nb), False, 0, 0, 1, P.nccl_unique_id())
        got, _ = P.cheby_power_many(dg, k, src, K, batched=True, tile=4)
    elif path == "measure":
        r = P.measure(want[0], want[1], g)
        assert r.l1 > 0
        got = want
    elif path == "topk":
        ids, vals, _ = P.cheby_power_topk(g, k, src, K, k=20)
        for j in range(len(src)):
            order = sorted(range(n), key=lambda v: (-want[j][v], v))[:20]
            assert list(ids[j]) == order, (j, list(ids[j])[:5], order[:5])
        got = want
    else:
        raise SystemExit(f"unknown path {path}")
    err = np.abs(got - want).max()
    print(f"{path}: max_abs {err:.2e}")
    if err > 1e-12:
        raise SystemExit(1)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
