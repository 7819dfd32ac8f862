"""GPU: golden vectors, the C++ drop-in against the reference's own types, and the
sharded (NCCL) code path with one rank."""
import os
import subprocess

import numpy as np
import pytest

from conftest import assert_parity

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def test_gpu_matches_golden_vectors(cpg, gpu):
    g = np.load(GOLDEN)
    names = sorted({k.split("/")[1] for k in g.files if k.startswith("graph/")})
    for name in names:
        graph = cpg.Graph.from_csr(g[f"graph/{name}/offsets"], g[f"graph/{name}/neighbors"])
        for tag, kern in (("ppr", cpg.Kernel.ppr(0.2)), ("hkpr", cpg.Kernel.hkpr(5.0))):
            K = int(g[f"graph/{name}/{tag}/K"])
            src = g[f"graph/{name}/sources"]
            got, st = cpg.cheby_power_many(graph, kern, src, K)
            for j in range(len(src)):
                assert_parity(got[j], g[f"graph/{name}/{tag}/values"][j])
            got_b, _ = cpg.cheby_power_many(graph, kern, src, K, batched=True, tile=len(src))
            for j in range(len(src)):
                assert_parity(got_b[j], g[f"graph/{name}/{tag}/values"][j])
        y = cpg.apply_walk(graph, g[f"graph/{name}/walk_x"])
        np.testing.assert_allclose(y, g[f"graph/{name}/walk_y"], rtol=1e-13, atol=1e-15)


def test_cpp_dropin_with_reference_types(gpu):
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK (0 failures)" in r.stdout


def test_sharded_handle_single_rank_nccl(cpg, gpu):
    """cpg_graph_create_sharded with nranks = 1: NCCL communicator, in-place
    all-gathers and the final gather all run (as copies) on one GPU."""
    from oracle import Port

    off, nb = cpg.gen_chunglu(30000, 300000, 2.2, 20.0, 5000, seed=2)
    uid = cpg.nccl_unique_id()
    import ctypes

    offs = np.ascontiguousarray(off, np.uint64)
    nbs = np.ascontiguousarray(nb, np.uint32)
    dg = cpg.DeviceGraph.sharded(offs.ctypes.data_as(ctypes.c_void_p), nbs.ctypes.data_as(ctypes.c_void_p),
                                 len(off) - 1, len(nb), False, 0, 0, 1, uid)
    assert dg.info.nranks == 1 and dg.info.n_local == len(off) - 1
    k = cpg.Kernel.hkpr(5.0)
    got, st = cpg.cheby_power_many(dg, k, [0, 17, 29000], 15)
    got_b, _ = cpg.cheby_power_many(dg, k, [0, 17, 29000], 15, batched=True, tile=4)
    c = k.cheby_coeffs(15)
    for j, s in enumerate([0, 17, 29000]):
        want, _, _ = Port.cheby_power(off, nb, c, 15, s)
        assert_parity(got[j], want)
        assert_parity(got_b[j], want)
    assert st.mass_err_max <= 1e-9


@pytest.mark.parametrize("self_store", ["0", "1"])
def test_sharded_fused_allgather(cpg, gpu, self_store, monkeypatch):
    """Fused all-gather (CPG_P2P=1): the iterates are NCCL symmetric windows and
    the batched epilogue stores every row into every rank's replica through the
    LSA peer pointers, with a one-element all-reduce per iteration as the
    barrier.  One rank: with CPG_P2P_SELF=1 the epilogue also stores through its
    own LSA alias (the peer-store code path and the window mapping), with 0 it
    runs the barrier path only.  Single-source queries on the same handle keep
    the NCCL all-gather."""
    import ctypes

    import torch  # loads the torch-bundled NCCL (device API) into the process

    from oracle import Port

    assert torch.cuda.is_available()
    monkeypatch.setenv("CPG_P2P", "1")
    monkeypatch.setenv("CPG_P2P_SELF", self_store)
    off, nb = cpg.gen_rmat(13, 16 << 13, seed=9)
    offs = np.ascontiguousarray(off, np.uint64)
    nbs = np.ascontiguousarray(nb, np.uint32)
    dg = cpg.DeviceGraph.sharded(offs.ctypes.data_as(ctypes.c_void_p), nbs.ctypes.data_as(ctypes.c_void_p),
                                 len(off) - 1, len(nb), False, 0, 0, 1, cpg.nccl_unique_id())
    assert dg.info.fused_allgather == 1 and dg.info.chunks == 1
    n = len(off) - 1
    k = cpg.Kernel.ppr(0.2)
    c = k.cheby_coeffs(26)
    src = [0, 7, n // 3, n - 1, 11]
    for tile in (4, 16):
        got_b, st = cpg.cheby_power_many(dg, k, src, 26, batched=True, tile=tile)
        for j, s in enumerate(src):
            want, _, _ = Port.cheby_power(off, nb, c, 26, s)
            assert_parity(got_b[j], want)
    got, _ = cpg.cheby_power_many(dg, k, src[:2], 26)
    for j, s in enumerate(src[:2]):
        want, _, _ = Port.cheby_power(off, nb, c, 26, s)
        assert_parity(got[j], want)


@pytest.mark.parametrize("chunks", ["1", "3"])
def test_sharded_single_rank_chunked(cpg, gpu, chunks, monkeypatch):
    """Chunked layout (CPG_CHUNKS) with per-chunk NCCL in-place all-gathers on the
    comm stream (one rank), single-source and batched, against the oracle."""
    import ctypes

    from oracle import Port

    monkeypatch.setenv("CPG_CHUNKS", chunks)
    off, nb = cpg.gen_rmat(13, 16 << 13, seed=4)
    offs = np.ascontiguousarray(off, np.uint64)
    nbs = np.ascontiguousarray(nb, np.uint32)
    dg = cpg.DeviceGraph.sharded(offs.ctypes.data_as(ctypes.c_void_p), nbs.ctypes.data_as(ctypes.c_void_p),
                                 len(off) - 1, len(nb), False, 0, 0, 1, cpg.nccl_unique_id())
    n = len(off) - 1
    assert dg.info.n_padded >= n
    k = cpg.Kernel.ppr(0.2)
    c = k.cheby_coeffs(26)
    src = [0, 5, n // 2, n - 1]
    got, st = cpg.cheby_power_many(dg, k, src, 26)
    got_b, _ = cpg.cheby_power_many(dg, k, src, 26, batched=True, tile=4)
    for j, s in enumerate(src):
        want, _, _ = Port.cheby_power(off, nb, c, 26, s)
        assert_parity(got[j], want)
        assert_parity(got_b[j], want)
    assert st.mass_err_max <= 1e-9


@pytest.mark.parametrize("chunks", ["2", "5"])
def test_single_gpu_chunked_layout(cpg, gpu, chunks, monkeypatch):
    """Chunked item tables / per-chunk launches without NCCL (one GPU)."""
    from oracle import Port

    monkeypatch.setenv("CPG_CHUNKS", chunks)
    off, nb = cpg.gen_chunglu(40000, 400000, 2.1, 20.0, 9000, seed=6)
    dg = cpg.DeviceGraph.from_host(off, nb, 0)
    k = cpg.Kernel.hkpr(5.0)
    c = k.cheby_coeffs(15)
    src = [0, 3, 20000]
    got, st = cpg.cheby_power_many(dg, k, src, 15)
    got_b, _ = cpg.cheby_power_many(dg, k, src, 15, batched=True, tile=16)
    for j, s in enumerate(src):
        want, _, _ = Port.cheby_power(off, nb, c, 15, s)
        assert_parity(got[j], want)
        assert_parity(got_b[j], want)
    est = cpg.cheby_power(dg, k, 7, 15, observer=lambda kk, r, e: None)
    want, _, _ = Port.cheby_power(off, nb, c, 15, 7)
    assert_parity(est.values, want)
