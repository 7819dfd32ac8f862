"""GPU parity: the sm_100a path (through the C ABI) against the reference library.

The checker is the UNMODIFIED reference (oracle/_ref/libchebyprop_ref.so, built
from /root/reference sources), whose restatement oracle/cheby_oracle.c is
pinned bit-for-bit in tests/test_oracle_pin.py.  Tolerance (north star):
per score vector max-abs <= 1e-12, L1 <= 1e-10, identical top-100 set.
"""
import numpy as np
import pytest

from conftest import assert_parity

pytestmark = pytest.mark.gpu

PPR, HKPR = 0, 1


def _ref_graph(off, nb):
    from oracle import RefGraph

    return RefGraph.from_csr(off, nb)


def _graphs():
    from oracle import Port

    gs = {
        "star": Port.edges_to_csr([[0, 1], [0, 2], [0, 3]]),          # tests/oracles.hpp:181-184
        "path3": Port.edges_to_csr([[0, 1], [1, 2]]),                 # oracles.hpp:186-189
        "ring_chord_200": Port.make_graph(200, 300, 1),               # acceptance.cpp:139-157 (C4)
        "ring_chord_1000": Port.make_graph(1000, 1500, 5),
        "big_star": Port.edges_to_csr([[0, i] for i in range(1, 9001)] + [[i, i + 1] for i in range(1, 9000)]),
    }
    return gs


@pytest.fixture(scope="module")
def graphs(gpu):
    import paper_2412_10789_b200 as P

    gs = _graphs()
    gs["rmat12"] = P.gen_rmat(12, 8 * 4096, seed=3)
    gs["chunglu"] = P.gen_chunglu(20000, 200000, 2.1, 20.0, 12000, seed=4)  # hubs split in pieces
    return gs


@pytest.mark.parametrize("name", ["star", "path3", "ring_chord_200", "ring_chord_1000", "big_star", "rmat12",
                                  "chunglu"])
@pytest.mark.parametrize("family,param", [(PPR, 0.2), (HKPR, 5.0)])
def test_cheby_power_matches_reference(graphs, cpg, name, family, param):
    off, nb = graphs[name]
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    kernel = cpg.Kernel.ppr(param) if family == PPR else cpg.Kernel.hkpr(param)
    K = cpg.plan_truncation(kernel, 1e-8).cheby_steps
    n = g.node_count()
    sources = sorted({0, n // 2, n - 1, min(n - 1, 7)})
    for s in sources:
        est = cpg.cheby_power(g, kernel, s, K)
        want, mass, rst = ref.cheby_power(family, param, s, K)
        assert_parity(est.values, want)
        assert est.stats.iterations == rst["iterations"] == K
        assert est.stats.push_work == rst["push_work"]
        assert est.stats.mass_err_max <= 1e-9  # acceptance.cpp:349-360 (C13)


def test_k1_two_term(graphs, cpg):
    """test_solvers.cpp:89-100: K = 1 is c0 e_s + c1 P e_s."""
    off, nb = graphs["star"]
    g = cpg.Graph.from_csr(off, nb)
    k = cpg.Kernel.ppr(0.2)
    c = k.cheby_coeffs(1)
    est = cpg.cheby_power(g, k, 1, 1)
    e = np.zeros(4)
    e[1] = 1
    pe = cpg.apply_walk(g, e)
    np.testing.assert_allclose(est.values, c[0] * e + c[1] * pe, rtol=1e-14, atol=0)


def test_star_r3_lands_on_hub(graphs, cpg):
    """test_solvers.cpp:101-113 through the observer slow path."""
    off, nb = graphs["star"]
    g = cpg.Graph.from_csr(off, nb)
    seen = {}
    cpg.cheby_power(g, cpg.Kernel.ppr(0.2), 1, 3, observer=lambda k, r, e: seen.__setitem__(k, r.copy()))
    r3 = seen[3]
    assert abs(r3[0] - 1.0) <= 1e-14
    assert np.all(np.abs(r3[1:]) < 1e-14)


def test_observer_trace_matches_reference(graphs, cpg):
    off, nb = graphs["ring_chord_200"]
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    K = 12
    rs, es = [], []
    est = cpg.cheby_power(g, cpg.Kernel.hkpr(5.0), 17, K, observer=lambda k, r, e: (rs.append(r.copy()),
                                                                                    es.append(e.copy())))
    want, rt, et = ref.cheby_power_trace(HKPR, 5.0, 17, K)
    assert len(rs) == K + 1
    for k in range(K + 1):
        assert np.abs(rs[k] - rt[k]).max() <= 1e-12
        assert np.abs(es[k] - et[k]).max() <= 1e-12
    assert_parity(est.values, want)


def test_vec_observer_trace_matches_oracle(graphs, cpg):
    """cheby_power_vec with an observer (solvers.hpp:62-64): the per-step T_k x and
    partial estimates equal the pinned C restatement's trace."""
    from oracle import Port

    off, nb = graphs["ring_chord_200"]
    g = cpg.Graph.from_csr(off, nb)
    x = Port.random_vector(g.node_count(), 5, -1.0, 1.0)
    K = 11
    k5 = cpg.Kernel.hkpr(5.0)
    rs, es = [], []
    est = cpg.cheby_power_vec(g, k5, x, K, observer=lambda k, r, e: (rs.append(r.copy()), es.append(e.copy())))
    want, _, rt, et = Port.cheby_power_vec(off, nb, k5.cheby_coeffs(K), K, x, trace=True)
    assert len(rs) == K + 1
    for k in range(K + 1):
        assert np.abs(rs[k] - rt[k]).max() <= 1e-12
        assert np.abs(es[k] - et[k]).max() <= 1e-12
    assert np.abs(est.values - want).max() <= 1e-12
    with pytest.raises(cpg.ParameterError):
        cpg.cheby_power_vec(g, k5, np.stack([x, x]), K, observer=lambda *a: None)


def test_mass_conservation_every_step(graphs, cpg):
    """test_solvers.cpp:122-128 / acceptance C13: |sum r_k - 1| <= 1e-9."""
    from oracle import Port

    off, nb = Port.make_graph(50, 80, 17)
    g = cpg.Graph.from_csr(off, nb)
    sums = []
    cpg.cheby_power(g, cpg.Kernel.ppr(0.2), 7, 30, observer=lambda k, r, e: sums.append(r.sum()))
    assert len(sums) == 31
    assert max(abs(s - 1.0) for s in sums) <= 1e-9


def test_cheby_power_vec_matches_reference(graphs, cpg):
    from oracle import Port

    for name in ("ring_chord_1000", "rmat12", "chunglu"):
        off, nb = graphs[name]
        g = cpg.Graph.from_csr(off, nb)
        ref = _ref_graph(off, nb)
        x = Port.random_vector(g.node_count(), 92, 0.0, 1.0)
        est = cpg.cheby_power_vec(g, cpg.Kernel.ppr(0.2), x, 40)
        want = ref.cheby_power_vec(PPR, 0.2, x, 40)
        assert np.abs(est.values - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
        assert np.abs(est.values - want).sum() <= 1e-10 * max(1.0, np.abs(want).sum())


def test_apply_walk_matches_reference(graphs, cpg):
    from oracle import Port

    for name in ("star", "path3", "rmat12", "big_star"):
        off, nb = graphs[name]
        g = cpg.Graph.from_csr(off, nb)
        ref = _ref_graph(off, nb)
        x = Port.random_vector(g.node_count(), 5, 0.0, 1.0)
        np.testing.assert_allclose(cpg.apply_walk(g, x), ref.apply_walk(x), rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("nsrc,tile", [(1, 64), (10, 64), (64, 64), (70, 64), (3, 3), (9, 8), (20, 16),
                                       (40, 32)])
def test_batched_matches_single_source(graphs, cpg, nsrc, tile):
    off, nb = graphs["chunglu"]
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    kernel = cpg.Kernel.hkpr(5.0)
    K = cpg.plan_truncation(kernel, 1e-8).cheby_steps
    src = ref.select_sources_uniform(nsrc, 11)
    got, st = cpg.cheby_power_many(g, kernel, src, K, batched=True, tile=tile)
    assert got.shape == (nsrc, g.node_count())
    for j in range(0, nsrc, max(1, nsrc // 5)):
        want, _, _ = ref.cheby_power(HKPR, 5.0, int(src[j]), K)
        assert_parity(got[j], want)
    assert st.push_work == K * g.volume() * nsrc


def test_many_single_source_pinned_output(graphs, cpg):
    import torch

    off, nb = graphs["rmat12"]
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    kernel = cpg.Kernel.ppr(0.2)
    K = 26
    src = ref.select_sources_uniform(9, 1)
    pinned = torch.empty((len(src), g.node_count()), dtype=torch.float64, pin_memory=True)
    got, st = cpg.cheby_power_many(g, kernel, src, K, out=pinned.numpy())
    for j, s in enumerate(src):
        want, _, _ = ref.cheby_power(PPR, 0.2, int(s), K)
        assert_parity(got[j], want)
    assert st.mass_err_max <= 1e-9


def test_sum_property(graphs, cpg):
    """Property 1: sum yhat = sum_k c_k."""
    off, nb = graphs["chunglu"]
    g = cpg.Graph.from_csr(off, nb)
    k = cpg.Kernel.ppr(0.2)
    est = cpg.cheby_power(g, k, 3, 26)
    assert abs(est.values.sum() - k.cheby_coeffs(26).sum()) <= 1e-12


def test_bit_reproducible(graphs, cpg):
    off, nb = graphs["chunglu"]
    g = cpg.Graph.from_csr(off, nb)
    k = cpg.Kernel.ppr(0.2)
    a = cpg.cheby_power(g, k, 5, 26).values
    b = cpg.cheby_power(g, k, 5, 26).values
    assert np.array_equal(a, b)


def test_errors(graphs, cpg):
    off, nb = graphs["path3"]
    g = cpg.Graph.from_csr(off, nb)
    with pytest.raises(cpg.ParameterError):
        cpg.cheby_power(g, cpg.Kernel.ppr(0.2), 99, 5)  # solvers.cpp:28-29
    with pytest.raises(cpg.ParameterError):
        cpg.cheby_power(g, cpg.Kernel.ppr(0.2), 0, 0)  # solvers.cpp:201
    with pytest.raises(cpg.ParameterError):
        cpg.cheby_power_vec(g, cpg.Kernel.ppr(0.2), np.zeros(2), 5)  # solvers.cpp:36-37


@pytest.mark.parametrize("a", [0.0, 0.5, 1.0, -0.3])
@pytest.mark.parametrize("tile", [1, 4, 16, 64])
def test_general_gp_matrix_matches_reference(graphs, cpg, a, tile):
    """general_gp_matrix (solvers.cpp:405-414) with fused D^{+-a} scalings, in column tiles."""
    from oracle import Port

    off, nb = graphs["chunglu"]
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    cols = [Port.random_vector(g.node_count(), 100 + j, 0.0, 1.0) for j in range(7)]
    kern = cpg.Kernel.hkpr(5.0)
    got = cpg.general_gp_matrix(g, kern, a, cols, 15, tile=tile)
    for j, x in enumerate(cols):
        want = ref.general_gp_vector(HKPR, 5.0, a, x, 15)
        scale = max(1.0, np.abs(want).max())
        assert np.abs(got[j] - want).max() <= 1e-12 * scale
        assert np.abs(got[j] - want).sum() <= 1e-10 * max(1.0, np.abs(want).sum())


def test_general_gp_vector_a_half(graphs, cpg):
    """acceptance.cpp:317-347 (C12) style: a = 1/2 against the reference wrapper."""
    from oracle import Port

    off, nb = Port.make_graph(10, 12, 63)
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    x = Port.random_vector(g.node_count(), 64, 0.0, 1.0)
    steps = cpg.plan_truncation(cpg.Kernel.ppr(0.2), 1e-13).cheby_steps
    z = cpg.general_gp_vector(g, cpg.Kernel.ppr(0.2), 0.5, x, steps)
    want = ref.general_gp_vector(PPR, 0.2, 0.5, x, steps)
    assert np.abs(z - want).max() <= 1e-12


def test_device_generator_matches_host(cpg, gpu):
    dev = cpg.gen_rmat(14, 8 << 14, seed=9, device=0)
    off, nb = dev.to_host()
    hoff, hnb = cpg.gen_rmat(14, 8 << 14, seed=9)
    assert np.array_equal(off, hoff) and np.array_equal(nb, hnb)
    dev.close()
    dev = cpg.gen_chunglu(30000, 150000, 2.3, 10.0, 2000, seed=5, device=0)
    off, nb = dev.to_host()
    hoff, hnb = cpg.gen_chunglu(30000, 150000, 2.3, 10.0, 2000, seed=5)
    assert np.array_equal(off, hoff) and np.array_equal(nb, hnb)


def test_graph_from_device_csr(cpg, gpu):
    dev = cpg.gen_rmat(13, 8 << 13, seed=21, device=0)
    off, nb = dev.to_host()
    dg = cpg.DeviceGraph.from_device(dev)
    ref = _ref_graph(off, nb)
    est = cpg.cheby_power(dg, cpg.Kernel.ppr(0.2), 11, 26)
    want, _, _ = ref.cheby_power(PPR, 0.2, 11, 26)
    assert_parity(est.values, want)


@pytest.mark.parametrize("tile", ["1024", "4096"])
def test_both_tile_widths(cpg, gpu, tile, monkeypatch):
    """Force each tile width (CPG_TILE) on a graph with hubs split into pieces."""
    monkeypatch.setenv("CPG_TILE", tile)
    off, nb = cpg.gen_chunglu(60000, 900000, 2.1, 30.0, 20000, seed=8)
    dg = cpg.DeviceGraph.from_host(off, nb, 0)
    ref = _ref_graph(off, nb)
    assert dg.info.n_hubs > 0
    for fam, par, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15)):
        kern = cpg.Kernel.ppr(par) if fam == PPR else cpg.Kernel.hkpr(par)
        for s in (0, 1, 12345, dg.n - 1):
            est = cpg.cheby_power(dg, kern, s, K)
            want, _, _ = ref.cheby_power(fam, par, s, K)
            assert_parity(est.values, want)


@pytest.mark.parametrize("graph", ["chunglu_hubs", "rmat", "ring"])
def test_warp_tile_step(cpg, gpu, graph, monkeypatch):
    """The barrier-free warp-tile single-source step (CPG_WARP_TILES=1): CTA hub pieces for
    rows above 4096 edges, single-row warp sweeps for 256 < degree <= 4096, 512-edge
    multi-row warp tiles below; against the reference, bit-reproducible, C13 mass."""
    from oracle import Port

    monkeypatch.setenv("CPG_WARP_TILES", "1")
    if graph == "chunglu_hubs":
        off, nb = cpg.gen_chunglu(60000, 900000, 2.1, 30.0, 20000, seed=8)  # rows of every class
    elif graph == "rmat":
        off, nb = cpg.gen_rmat(15, 16 << 15, seed=5)
    else:
        off, nb = Port.make_graph(3000, 5000, 3)
    dg = cpg.DeviceGraph.from_host(off, nb, 0)
    ref = _ref_graph(off, nb)
    for fam, par, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15)):
        kern = cpg.Kernel.ppr(par) if fam == PPR else cpg.Kernel.hkpr(par)
        for s in (0, 1, dg.n // 2, dg.n - 1):
            est = cpg.cheby_power(dg, kern, s, K)
            want, _, _ = ref.cheby_power(fam, par, s, K)
            assert_parity(est.values, want)
            assert est.stats.mass_err_max <= 1e-9
    again = cpg.cheby_power(dg, cpg.Kernel.ppr(0.2), 1, 26).values
    assert np.array_equal(again, cpg.cheby_power(dg, cpg.Kernel.ppr(0.2), 1, 26).values)
    monkeypatch.setenv("CPG_WARP_TILES", "0")
    assert np.abs(again - cpg.cheby_power(dg, cpg.Kernel.ppr(0.2), 1, 26).values).max() <= 1e-14


def test_large_graph_default_tiles(cpg, gpu):
    """A graph big enough for the large-tile table (>= 4096*148*8 edges)."""
    off, nb = cpg.gen_rmat(18, 16 << 18, seed=12)
    assert len(nb) >= 4096 * 148 * 8
    dg = cpg.DeviceGraph.from_host(off, nb, 0)
    ref = _ref_graph(off, nb)
    src = ref.select_sources_uniform(3, 1)
    got, st = cpg.cheby_power_many(dg, cpg.Kernel.ppr(0.2), src, 26)
    for j, s in enumerate(src):
        want, _, _ = ref.cheby_power(PPR, 0.2, int(s), 26)
        assert_parity(got[j], want)
    assert st.mass_err_max <= 1e-9


@pytest.mark.parametrize("family,param", [(PPR, 0.2), (HKPR, 5.0)])
def test_ground_truth_power_method_matches_reference(graphs, cpg, family, param):
    """GPU PwMethod with the reference's ground-truth N (eval.cpp:39-59) vs the reference."""
    kern = cpg.Kernel.ppr(param) if family == PPR else cpg.Kernel.hkpr(param)
    assert cpg.ground_truth_steps(kern) == (231 if family == PPR else 461)
    for name in ("ring_chord_1000", "chunglu", "rmat12"):
        off, nb = graphs[name]
        g = cpg.Graph.from_csr(off, nb)
        ref = _ref_graph(off, nb)
        for s in (0, g.node_count() // 3):
            assert_parity(cpg.ground_truth(g, kern, s), ref.ground_truth(family, param, s))


def test_power_method_small_n(graphs, cpg):
    """test_solvers.cpp:29-35 (N = 1 is zeta_0 e_s) and the Taylor tail bound (:42-51)."""
    from oracle import Port

    off, nb = Port.make_graph(12, 10, 5)
    g = cpg.Graph.from_csr(off, nb)
    est = cpg.power_method(g, cpg.Kernel.ppr(0.3), 4, 1)
    assert est.values[4] == 0.3 and np.count_nonzero(est.values) == 1 and est.stats.iterations == 1
    off, nb = Port.make_graph(40, 60, 9)
    g = cpg.Graph.from_csr(off, nb)
    P = np.zeros((g.node_count(), g.node_count()))
    for u in range(g.node_count()):
        for v in nb[off[u]:off[u + 1]]:
            P[v, u] = 1.0 / (off[u + 1] - off[u])
    exact = np.linalg.solve(np.eye(g.node_count()) - 0.8 * P, 0.2 * np.eye(g.node_count())[3])
    for n_steps in (5, 10, 25):
        est = cpg.power_method(g, cpg.Kernel.ppr(0.2), 3, n_steps)
        assert np.abs(est.values - exact).sum() <= 0.8 ** n_steps * (1 + 1e-12)
        want = Port.power_method(off, nb, Port.taylor_coeffs(PPR, 0.2, n_steps - 1), n_steps, 3)
        assert np.abs(est.values - want).max() <= 1e-12


def test_edge_cases(cpg, gpu):
    """Empty source list, duplicate sources, repeated calls, large K and extreme parameters."""
    from oracle import Port

    off, nb = Port.make_graph(300, 500, 13)
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    k = cpg.Kernel.ppr(0.2)
    out, st = cpg.cheby_power_many(g, k, [], 26)
    assert out.shape == (0, g.node_count()) and st.push_work == 0
    out_b, _ = cpg.cheby_power_many(g, k, [], 26, batched=True)
    assert out_b.shape == (0, g.node_count())
    got, _ = cpg.cheby_power_many(g, k, [5, 5, 5], 26)
    want, _, _ = ref.cheby_power(PPR, 0.2, 5, 26)
    for j in range(3):
        assert_parity(got[j], want)
    got_b, _ = cpg.cheby_power_many(g, k, [5, 5, 7], 26, batched=True, tile=3)
    assert_parity(got_b[0], want) and assert_parity(got_b[1], want)
    for fam, p, eps in ((PPR, 0.02, 1e-10), (HKPR, 40.0, 1e-12), (PPR, 0.9, 1e-3), (HKPR, 0.3, 1e-6)):
        kern = cpg.Kernel.ppr(p) if fam == PPR else cpg.Kernel.hkpr(p)
        K = cpg.plan_truncation(kern, eps).cheby_steps
        est = cpg.cheby_power(g, kern, 11, K)
        want, _, _ = ref.cheby_power(fam, p, 11, K)
        assert_parity(est.values, want)
    est = cpg.cheby_power(g, k, 0, 200)  # far past convergence
    want, _, _ = ref.cheby_power(PPR, 0.2, 0, 200)
    assert_parity(est.values, want)


def _cheby_power_longdouble(off, nb, coeffs, K, s):
    """The reference recurrence (solvers.cpp:197-234) in x87 extended precision (numpy longdouble)."""
    n = len(off) - 1
    deg = np.diff(off).astype(np.longdouble)
    rows = np.repeat(np.arange(n), np.diff(off).astype(np.int64))

    def walk(x):  # graph.cpp:257-267
        out = np.zeros(n, dtype=np.longdouble)
        np.add.at(out, nb, (x / deg)[rows])
        return out

    c = np.asarray(coeffs, dtype=np.longdouble)
    seed = np.zeros(n, dtype=np.longdouble)
    seed[s] = 1
    y = c[0] * seed
    r_prev, r_cur = seed, walk(seed)
    for k in range(1, K):
        y = y + c[k] * r_cur
        r_prev, r_cur = r_cur, 2 * walk(r_cur) - r_prev
    return y + c[K] * r_cur


def test_giant_hub_star(cpg, gpu):
    """A 200k-leaf star (+ path among leaves): hub pieces P > 1 in every kernel.

    The hub's score sums 200k terms; the reference adds them sequentially
    (error up to ~n*eps relative), the GPU in pieces and trees.  Both are
    compared against an extended-precision evaluation: the GPU must be at
    least as accurate as the reference, and within 5e-12 of it."""
    from oracle import Port

    m = 200_000
    pairs = [[0, i] for i in range(1, m + 1)] + [[i, i + 1] for i in range(1, m, 7)]
    off, nb = Port.edges_to_csr(pairs)
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    k = cpg.Kernel.hkpr(5.0)
    c = k.cheby_coeffs(15)
    src = [0, 1, 12345]
    got, _ = cpg.cheby_power_many(g, k, src, 15)
    for tile in (3, 16, 64):
        got_b, _ = cpg.cheby_power_many(g, k, src, 15, batched=True, tile=tile)
        for j, s in enumerate(src):
            want, _, _ = ref.cheby_power(HKPR, 5.0, s, 15)
            truth = _cheby_power_longdouble(off, nb, c, 15, s)
            for v in (got[j], got_b[j]):
                assert_parity(v, want, max_abs=5e-12)
                err_gpu = float(np.abs(v.astype(np.longdouble) - truth).max())
                err_ref = float(np.abs(want.astype(np.longdouble) - truth).max())
                assert err_gpu <= err_ref + 1e-13, (err_gpu, err_ref)


@pytest.mark.parametrize("k", [1, 50, 100, 1000])
def test_device_topk_matches_reference_ranking(graphs, cpg, k):
    """Device top-k equals ranking the reference's vector by (value desc, id asc)."""
    off, nb = graphs["chunglu"]
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    src = [0, 3, 999]
    ids, vals, _ = cpg.cheby_power_topk(g, cpg.Kernel.ppr(0.2), src, 26, k)
    full, _ = cpg.cheby_power_many(g, cpg.Kernel.ppr(0.2), src, 26)
    for j, s in enumerate(src):
        order = np.lexsort((np.arange(g.node_count()), -full[j]))[:k]
        assert np.array_equal(ids[j], order.astype(np.uint32))
        assert np.array_equal(vals[j], full[j][order])
        want, _, _ = ref.cheby_power(PPR, 0.2, s, 26)
        assert np.abs(vals[j] - want[ids[j]]).max() <= 1e-12


def test_device_topk_ties_and_k_over_n(cpg, gpu):
    from oracle import Port

    off, nb = Port.make_graph(64, 0, 1)  # plain ring: massive ties
    g = cpg.Graph.from_csr(off, nb)
    ids, vals, _ = cpg.cheby_power_topk(g, cpg.Kernel.ppr(0.5), [0], 1, 1000)
    assert ids.shape == (1, 64)
    full, _ = cpg.cheby_power_many(g, cpg.Kernel.ppr(0.5), [0], 1)
    order = np.lexsort((np.arange(64), -full[0]))
    assert np.array_equal(ids[0], order.astype(np.uint32))


def test_gpu_ingest_matches_reference_loader(cpg, gpu, tmp_path):
    """GPU edge-list ingest == the reference's load_edge_list (graph.cpp:113-171):
    self-loops, duplicates, both directions, negative / sparse int64 labels."""
    from oracle import RefGraph, edge_text

    rng = np.random.default_rng(7)
    for trial in range(3):
        m = 5000
        labels = rng.choice(np.arange(-10**12, 10**12, 10**7), size=800, replace=False)
        pairs = labels[rng.integers(0, 800, size=(m, 2))]
        pairs[::97, 1] = pairs[::97, 0]          # self-loops
        pairs = np.concatenate([pairs, pairs[:300, ::-1], pairs[:200]])  # reversed and exact duplicates
        ref = RefGraph.from_edge_text(edge_text(pairs))
        csr, ids = cpg.ingest_edges(pairs, 0)
        off, nb = csr.to_host()
        roff, rnb = ref.csr()
        assert np.array_equal(off, roff) and np.array_equal(nb, rnb)
        assert np.array_equal(ids, ref.original_ids())
        csr.close()
    path = tmp_path / "g.txt"
    path.write_text("# comment\n\n1 2\n2 3 0.5\n  # indented comment\n3 1\n3 3\n4 1\n")
    g = cpg.load_edge_list_file(str(path))
    ref = RefGraph.from_edge_text("1 2\n2 3\n3 1\n3 3\n4 1\n")
    roff, rnb = ref.csr()
    assert np.array_equal(g.offsets(), roff) and np.array_equal(g.neighbor_array(), rnb)
    assert list(g.original_ids) == [1, 2, 3, 4]
    with pytest.raises(cpg.StructuralError):  # graph.cpp:156: StructuralError, like the reference
        cpg.ingest_edges([[5, 5]], 0)  # empty after cleaning


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("tile", [4, 16, 64])
def test_batched_split_and_fused_paths(cpg, gpu, split, tile, monkeypatch):
    """Both batched code paths (hub-piece + plain-row kernels, and the fused kernel)
    on a graph with many hub pieces, against the reference."""
    monkeypatch.setenv("CPG_BATCH_SPLIT", split)
    off, nb = cpg.gen_chunglu(50000, 600000, 2.0, 24.0, 15000, seed=11)
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    src = ref.select_sources_uniform(min(tile, 9), 5)
    kern = cpg.Kernel.ppr(0.2)
    got, _ = cpg.cheby_power_many(g, kern, src, 26, batched=True, tile=tile)
    for j, s in enumerate(src):
        want, _, _ = ref.cheby_power(PPR, 0.2, int(s), 26)
        assert_parity(got[j], want)


def test_pipelined_batched_output(cpg, gpu):
    """cpg_chebypower_batched_async: back-to-back calls whose result copies stay in
    flight (alternating staging slots across calls, pinned and pageable outputs,
    one and several tiles per call) give the synchronous call's results exactly."""
    import torch

    off, nb = cpg.gen_chunglu(20000, 200000, 2.2, 12.0, 4000, seed=31)
    g = cpg.Graph.from_csr(off, nb)
    n = g.node_count()
    kern = cpg.Kernel.ppr(0.2)
    calls = [([3, 5, 7, 11], 4), ([13, 17, 19], 16), (list(range(40, 50)), 4), ([23], 1)]
    want = [cpg.cheby_power_many(g, kern, s, 26, batched=True, tile=t)[0] for s, t in calls]
    outs = []
    for j, (s, t) in enumerate(calls):
        if j % 2 == 0:
            o = torch.empty((len(s), n), dtype=torch.float64, pin_memory=True).numpy()
        else:
            o = np.empty((len(s), n))
        o.fill(np.nan)
        cpg.cheby_power_many_pipelined(g, kern, s, 26, o, tile=t)
        outs.append(o)
    cpg.sync(g)
    for o, w in zip(outs, want):
        assert np.array_equal(o, w)
    # a synchronous call after pipelined ones waits for nothing stale
    again, _ = cpg.cheby_power_many(g, kern, calls[0][0], 26, batched=True, tile=4)
    assert np.array_equal(again, want[0])


@pytest.mark.parametrize("tile", ["1024", "2048", "4096"])
def test_single_source_split_step(cpg, gpu, tile, monkeypatch):
    """The split single-source step (hub-piece kernel + tile kernel at higher
    occupancy; default when the iterate exceeds L2) at every tile width, on a
    graph with multi-piece hubs: PPR and HKPR against the reference, the mass
    check, and bit-identical to the combined kernel (same reduction order)."""
    monkeypatch.setenv("CPG_TILE", tile)
    monkeypatch.setenv("CPG_GROUP_Q", "1")  # the split step runs one query per launch
    off, nb = cpg.gen_chunglu(30000, 500000, 2.0, 30.0, 12000, seed=21)
    assert np.diff(off).max() > 4096  # hubs split into several pieces
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    src = ref.select_sources_uniform(5, 3)
    for fam, param, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15)):
        kern = cpg.Kernel.ppr(param) if fam == PPR else cpg.Kernel.hkpr(param)
        monkeypatch.setenv("CPG_STEP_SPLIT", "1")
        got, st = cpg.cheby_power_many(g, kern, src, K)
        monkeypatch.setenv("CPG_STEP_SPLIT", "0")
        combined, _ = cpg.cheby_power_many(g, kern, src, K)
        assert np.array_equal(got, combined)
        assert st.mass_err_max <= 1e-9
        for j, s in enumerate(src):
            want, _, _ = ref.cheby_power(fam, param, int(s), K)
            assert_parity(got[j], want)


@pytest.mark.gpu
@pytest.mark.parametrize("group", ["1", "3", "16"])
def test_single_source_query_groups(cpg, gpu, group, monkeypatch):
    """Query groups of the single-source step (several queries per launch, each
    with its own iterate slices, hub partial slots and tickets, and mass
    partials), on a graph with multi-piece hubs: PPR and HKPR against the
    reference, and the mass check."""
    monkeypatch.setenv("CPG_GROUP_Q", group)
    off, nb = cpg.gen_chunglu(30000, 500000, 2.0, 30.0, 12000, seed=21)
    assert np.diff(off).max() > 4096  # hubs split into several pieces
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref_graph(off, nb)
    src = ref.select_sources_uniform(19, 3)  # 19 = groups of 16 + 3 (ragged tail)
    for fam, param, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15)):
        kern = cpg.Kernel.ppr(param) if fam == PPR else cpg.Kernel.hkpr(param)
        got, st = cpg.cheby_power_many(g, kern, src, K)
        assert st.mass_err_max <= 1e-9
        for j, s in enumerate(src):
            want, _, _ = ref.cheby_power(fam, param, int(s), K)
            assert_parity(got[j], want)


def test_batched_mass_check(cpg, gpu):
    """North star item (3) for the batched step: the epilogue's per-column mass
    sum_v d_v w_{k+1}(v) = sum_v T_{k+1}(v) (acceptance.cpp:349-360, C13) is reduced
    on the device for every column and step, in both batched paths; dense seed
    columns (general_gp_matrix, a = 0) conserve their own sums; a != 0 has no
    conserved mass and reports NaN."""
    import os

    off, nb = cpg.gen_chunglu(20000, 200000, 2.1, 20.0, 3000, seed=12)
    g = cpg.Graph.from_csr(off, nb)
    k = cpg.Kernel.ppr(0.2)
    for split in ("0", "1"):
        os.environ["CPG_BATCH_SPLIT"] = split
        try:
            for tile in (4, 16, 64):
                _, st = cpg.cheby_power_many(g, k, list(range(tile)), 26, batched=True, tile=tile)
                assert 0.0 <= st.mass_err_max <= 1e-9, (split, tile, st.mass_err_max)
        finally:
            del os.environ["CPG_BATCH_SPLIT"]
    from oracle import Port

    n = g.node_count()
    X = np.stack([Port.random_vector(n, 3 + j, 0.0, 1.0) for j in range(5)])
    cols = cpg.general_gp_matrix(g, k, 0.0, X, 26, tile=8)
    assert len(cols) == 5
    # stats through the C ABI: conserved mass = column sums
    import ctypes

    from paper_2412_10789_b200 import _lib

    c = k.cheby_coeffs(26)
    out = np.empty_like(X)
    s = _lib.cpg_stats()
    rc = _lib.lib().cpg_general_gp(g.device(0).handle, c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 26, 0.0,
                                   X.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 5, 8, out.ctypes.data,
                                   ctypes.byref(s))
    assert rc == 0 and s.mass_err_max <= 1e-9 * X.sum(axis=1).max()
    rc = _lib.lib().cpg_general_gp(g.device(0).handle, c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 26, 0.5,
                                   X.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 5, 8, out.ctypes.data,
                                   ctypes.byref(s))
    assert rc == 0 and np.isnan(s.mass_err_max)
