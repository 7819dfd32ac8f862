"""GPU: the row-partitioned multi-GPU path with R > 1 ranks on ONE device.

The shards are real libcpg handles (cpg_graph_create_loopback): the device
relabel and row partition (graph_build.cu k_assign / k_local), chunk_row0,
the per-chunk in-place all-gathers (gather_chunk), the mass all-reduce, the
result gather (gather_result) and the unpermute all run the product's code;
only the data plane is the test-only loopback (peer-buffer copies between the
handles instead of NCCL over NVLink).  One host thread per rank makes the
same call, as one process per GPU would (solvers.cpp:217-224 is the loop
being sharded).  Every rank's output is checked against the
oracle (the reference library), single-source and batched.
"""
import os
import threading

import numpy as np
import pytest

from conftest import assert_parity

pytestmark = pytest.mark.gpu

PPR, HKPR = 0, 1


@pytest.fixture(scope="module")
def graph(gpu):
    import paper_2412_10789_b200 as P

    # hubs above every piece threshold (max degree ~3000), n not a multiple of any R*C below
    return P.gen_chunglu(20011, 220000, 2.1, 20.0, 3000, seed=11)


def _run_ranks(fn, R):
    out, errs = [None] * R, []

    def work(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # surfaced below
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.mark.parametrize("R,C,sparse", [(2, 1, None), (3, 1, None), (8, 1, None), (2, 4, None), (3, 4, None),
                                        (8, 4, None), (3, 1, "2"), (2, 4, "2"), (8, 4, "1")])
def test_loopback_sharded_matches_reference(cpg, graph, R, C, sparse, monkeypatch):
    from oracle import RefGraph

    off, nb = graph
    monkeypatch.setenv("CPG_CHUNKS", str(C))
    # sparse early steps: a sharded rank masks step 1 only (the sources'
    # bitmap); this graph is below the default's edge threshold, so force it too
    if sparse is not None:
        monkeypatch.setenv("CPG_SPARSE_STEPS", sparse)
    grp = cpg.LoopbackGroup(R)
    shards = [cpg.DeviceGraph.loopback(off, nb, r, grp) for r in range(R)]
    n = len(off) - 1
    for r, dg in enumerate(shards):
        assert (dg.info.rank, dg.info.nranks, dg.info.chunks) == (r, R, C)
        if sparse is not None:
            assert dg.sparse_early_steps(8, 26) == 1 and dg.sparse_early_steps(1, 26) == 1
        assert dg.info.n_padded % (R * C) == 0
    # the shards partition the rows and the edges
    assert sum(d.info.n_local for d in shards) == shards[0].info.n_padded
    assert sum(d.info.nnz_local for d in shards) == len(nb)
    ref = RefGraph.from_csr(off, nb)
    sources = [0, 7, n // 2, n - 1, 12345]
    for fam, param, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15)):
        k = cpg.Kernel.ppr(param) if fam == PPR else cpg.Kernel.hkpr(param)
        single = _run_ranks(lambda r: cpg.cheby_power_many(shards[r], k, sources, K), R)
        batched = _run_ranks(lambda r: cpg.cheby_power_many(shards[r], k, sources, K, batched=True, tile=8), R)
        for j, s in enumerate(sources):
            want, _, _ = ref.cheby_power(fam, param, s, K)
            for r in range(R):
                assert_parity(single[r][0][j], want)
                assert_parity(batched[r][0][j], want)
        for r in range(R):
            assert single[r][1].mass_err_max <= 1e-9, single[r][1].mass_err_max  # C13, all-reduced
            assert batched[r][1].mass_err_max <= 1e-9, batched[r][1].mass_err_max
            # every rank holds the same gathered result
            assert np.array_equal(single[r][0], single[0][0])
            assert np.array_equal(batched[r][0], batched[0][0])
    for dg in shards:
        dg.close()


def test_concurrent_queries_on_one_handle(cpg, graph):
    """The reference allows concurrent queries on a shared Graph (
    its bench drives them from a worker pool, tools/chebyprop.cpp:305-334).  Eight
    host threads x 16 queries on ONE handle, mixing single-source, batched and
    pipelined calls, must return exactly what the same calls return serially."""
    off, nb = graph
    g = cpg.Graph.from_csr(off, nb)
    dg = g.device(0)
    n = g.node_count()
    k = cpg.Kernel.ppr(0.2)
    K = 26
    rng = np.random.default_rng(5)
    work = [sorted(rng.choice(n, 16, replace=False).tolist()) for _ in range(8)]

    def call(t, srcs):
        if t % 3 == 0:
            return cpg.cheby_power_many(dg, k, srcs, K)[0]
        if t % 3 == 1:
            return cpg.cheby_power_many(dg, k, srcs, K, batched=True, tile=16)[0]
        return np.stack([cpg.cheby_power(dg, k, s, K).values for s in srcs])

    serial = [call(t, work[t]) for t in range(8)]
    for _ in range(2):
        conc = _run_ranks(lambda t: call(t, work[t]), 8)
        for t in range(8):
            assert np.array_equal(conc[t], serial[t]), t


def test_pipelined_slot_layout_change(cpg, graph):
    """an async batched call leaves its last copy in flight; a following call
    with another slot size must not overwrite the staging bytes that copy still reads."""
    off, nb = graph
    dg = cpg.Graph.from_csr(off, nb).device(0)
    k = cpg.Kernel.ppr(0.2)
    n = dg.n
    try:
        import torch

        pinned = [torch.empty((16, n), dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
    except Exception:
        pinned = [np.empty((16, n)) for _ in range(2)]
    want4 = cpg.cheby_power_many(dg, k, [1, 2, 3, 4], 26, batched=True, tile=4)[0]
    want16 = cpg.cheby_power_many(dg, k, list(range(16)), 26, batched=True, tile=16)[0]
    out4 = pinned[0][:4]
    cpg.cheby_power_many_pipelined(dg, k, [1, 2, 3, 4], 26, out4, tile=4)
    cpg.cheby_power_many_pipelined(dg, k, list(range(16)), 26, pinned[1], tile=16)
    cpg.sync(dg)
    assert np.array_equal(out4, want4)
    assert np.array_equal(pinned[1], want16)


@pytest.mark.parametrize("R", [1, 3])
def test_multi_device_facade(cpg, graph, R):
    """cpg_graph_create_multi's facade (one handle over a device list): one
    host call fans out to every shard's thread; rank 0's output equals the reference.  On
    one GPU the shards use the loopback plane; a one-device list is a plain handle."""
    from oracle import Port, RefGraph

    off, nb = graph
    n = len(off) - 1
    dg = cpg.DeviceGraph.multi_loopback(off, nb, R) if R > 1 else cpg.DeviceGraph.multi(off, nb, [0])
    assert dg.info.nranks == R and dg.info.n == n
    ref = RefGraph.from_csr(off, nb)
    k = cpg.Kernel.ppr(0.2)
    src = [0, 9, n // 3, n - 1]
    single, st = cpg.cheby_power_many(dg, k, src, 26)
    batched, bst = cpg.cheby_power_many(dg, k, src, 26, batched=True, tile=4)
    for j, s in enumerate(src):
        want, _, _ = ref.cheby_power(PPR, 0.2, s, 26)
        assert_parity(single[j], want)
        assert_parity(batched[j], want)
    assert st.mass_err_max <= 1e-9 and bst.mass_err_max <= 1e-9
    x = Port.random_vector(n, 3, 0.0, 1.0)
    got = cpg.cheby_power_vec(dg, cpg.Kernel.hkpr(5.0), x, 15).values
    want = ref.cheby_power_vec(HKPR, 5.0, x, 15)
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
    if R > 1:
        with pytest.raises(cpg.ParameterError):
            cpg.cheby_power_topk(dg, k, src, 26, k=5)
    dg.close()
