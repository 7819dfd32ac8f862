"""Pin the oracle: the C restatement (oracle/cheby_oracle.c) against the reference
itself and against the reference tests' known answers.  CPU only."""
import math
import os

import numpy as np
import pytest

from oracle import HKPR, PPR, Port, Ref, RefGraph, edge_text

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden(oracle_mod):
    return np.load(GOLDEN)


# ---- known answers from the reference's own tests --------------------------------------
def test_ppr_first_terms(oracle_mod):
    """test_kernels.cpp:14-21: alpha = 0.2 -> [1/3, 1/3, 1/6]."""
    c = Port.ppr_cheby_coeffs(0.2, 2)
    assert c == pytest.approx([1 / 3, 1 / 3, 1 / 6], rel=1e-14)


def test_appendix_a_values(oracle_mod):
    """SURVEY.md Appendix A (measured from the reference)."""
    c = Port.ppr_cheby_coeffs(0.2, 26)
    assert c[0] == c[1] == 0.33333333333333337
    assert c[26] == 9.9341074625651053e-09
    assert sum(c.tolist()) == pytest.approx(0.99999999006589269, rel=1e-15)
    h = Port.hkpr_cheby_coeffs(5.0, 15)
    assert h[0] == 0.18354081260932834
    assert h[1] == 0.32794453388908473
    assert h[15] == 1.412243606638146e-08
    assert sum(h.tolist()) == pytest.approx(0.99999999748215751, rel=1e-15)
    p = Port.plan_truncation(PPR, 0.2, 1e-8)
    assert (p.cheby_steps, p.taylor_steps) == (26, 83)
    assert p.tail_bound == pytest.approx(9.934e-9, rel=1e-3)
    p = Port.plan_truncation(HKPR, 5.0, 1e-8)
    assert (p.cheby_steps, p.taylor_steps) == (15, 23)
    assert p.tail_bound == pytest.approx(2.518e-9, rel=1e-3)


def test_hkpr_sum_and_ratio(oracle_mod):
    """test_kernels.cpp:47-58: sum 1 at t = 5, K = 40; c1/c0 = 2 I1/I0 (quadrature)."""
    c = Port.hkpr_cheby_coeffs(5.0, 40)
    assert abs(c.sum() - 1.0) <= 1e-12

    def bessel(k, t, panels=1 << 15):  # tests/oracles.hpp:125-135
        h = math.pi / (2 * panels)
        th = np.arange(2 * panels + 1) * h
        f = np.exp(t * np.cos(th)) * np.cos(k * th)
        w = np.where(np.arange(2 * panels + 1) % 2 == 1, 4.0, 2.0)
        w[0] = w[-1] = 1.0
        return (f * w).sum() * h / 3.0 / math.pi

    assert abs(c[1] / c[0] - 2 * bessel(1, 5.0) / bessel(0, 5.0)) <= 1e-10


def test_c1_coefficient_identities(oracle_mod):
    """acceptance.cpp:74-90 (C1)."""
    for fam, params in ((PPR, (0.2, 0.1, 0.02)), (HKPR, (5.0, 20.0, 40.0))):
        for p in params:
            K = Port.plan_truncation(fam, p, 5e-13).cheby_steps
            assert abs(Port.cheby_coeffs(fam, p, K).sum() - 1.0) <= 1e-12


def test_plan_monotone_and_domain(oracle_mod):
    """test_kernels.cpp:142-182."""
    for fam, p in ((PPR, 0.2), (HKPR, 5.0)):
        prev_k = prev_n = 0
        for eps in (1e-2, 1e-4, 1e-6, 1e-8):
            pl = Port.plan_truncation(fam, p, eps)
            assert pl.cheby_steps >= prev_k and pl.taylor_steps >= prev_n
            prev_k, prev_n = pl.cheby_steps, pl.taylor_steps
    pl = Port.plan_truncation(PPR, 0.2, 0.999)
    assert pl.cheby_steps == 1 and pl.taylor_steps == 1
    for bad in (0.0, 1.0):
        with pytest.raises(Exception):
            Port.plan_truncation(PPR, 0.2, bad)


def test_star_and_path(oracle_mod):
    """test_solvers.cpp:89-121 on the restatement."""
    off, nb = Port.edges_to_csr([[0, 1], [0, 2], [0, 3]])
    c = Port.ppr_cheby_coeffs(0.2, 3)
    _, _, rt, _ = Port.cheby_power_vec(off, nb, c, 3, np.eye(4)[1], trace=True)
    assert rt[3][0] == pytest.approx(1.0, rel=1e-14) and np.all(np.abs(rt[3][1:]) < 1e-14)
    off, nb = Port.edges_to_csr([[0, 1], [1, 2]])
    K = Port.plan_truncation(PPR, 0.2, 1e-8).cheby_steps
    y, _, _ = Port.cheby_power(off, nb, Port.ppr_cheby_coeffs(0.2, K), K, 1)
    P = np.array([[0, 0.5, 0], [1, 0, 1], [0, 0.5, 0]])
    exact = np.linalg.solve(np.eye(3) - 0.8 * P, 0.2 * np.eye(3)[1])
    assert np.linalg.norm(y - exact) < 1e-8


# ---- bit-exact against the reference library ------------------------------------------
needs_ref = pytest.mark.skipif(not Ref.available(), reason="reference library not built")


@needs_ref
def test_port_matches_reference_bit_exact(oracle_mod):
    for fam, params in ((PPR, (0.2, 0.1, 0.02, 0.5)), (HKPR, (5.0, 20.0, 40.0, 0.3))):
        for p in params:
            assert np.array_equal(Port.cheby_coeffs(fam, p, 120), Ref.cheby_coeffs(fam, p, 120))
            assert np.array_equal(Port.taylor_coeffs(fam, p, 60), Ref.taylor_coeffs(fam, p, 60))
            for eps in (1e-3, 1e-6, 1e-8, 1e-12):
                a, b = Port.plan_truncation(fam, p, eps), Ref.plan_truncation(fam, p, eps)
                assert a.__dict__ == b.__dict__
    for args in ((25, 35, 31), (200, 300, 1), (500, 900, 7)):
        pairs = Port.ring_chord_pairs(*args)
        g = RefGraph.from_edge_text(edge_text(pairs))
        off, nb = Port.edges_to_csr(pairs)
        roff, rnb = g.csr()
        assert np.array_equal(off, roff) and np.array_equal(nb, rnb)  # loader restatement
        for fam, p, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15), (PPR, 0.02, 40)):
            c = Port.cheby_coeffs(fam, p, K)
            for s in (0, g.n // 2, g.n - 1):
                v, m, w = Port.cheby_power(off, nb, c, K, s)
                rv, rm, st = g.cheby_power(fam, p, s, K)
                assert np.array_equal(v, rv) and np.array_equal(m, rm)
                assert w == st["push_work"]
        x = Port.random_vector(g.n, 3, -1.0, 1.0)
        assert np.array_equal(Port.apply_walk(off, nb, x), g.apply_walk(x))
        assert np.array_equal(Port.select_sources_uniform(g.n, 10, 4), g.select_sources_uniform(10, 4))


@needs_ref
def test_adopted_reference_graph_equals_from_csr(oracle_mod):
    """bench.py's huge-graph CPU baseline builds the reference Graph without from_csr's
    symmetry check; it must compute exactly what the validated Graph computes."""
    pairs = Port.ring_chord_pairs(500, 900, 7)
    off, nb = Port.edges_to_csr(pairs)
    g, a = RefGraph.from_csr(off, nb), RefGraph.adopt_csr(off, nb)
    assert (a.n, a.nnz) == (g.n, g.nnz)
    roff, rnb = a.csr()
    assert np.array_equal(off, roff) and np.array_equal(nb, rnb)
    x = Port.random_vector(g.n, 5, -1.0, 1.0)
    assert np.array_equal(a.apply_walk(x), g.apply_walk(x))
    assert np.array_equal(a.cheby_power(PPR, 0.2, 3, 26)[0], g.cheby_power(PPR, 0.2, 3, 26)[0])
    for threads, per in ((1, 0), (1, len(nb)), (4, 1000)):
        wall, edges = a.apply_walk_subset_pool(threads, per)
        assert wall >= 0.0
        if per == 0:
            assert edges == 0
        elif threads == 1:
            assert edges == len(nb)  # one run over every row is one full apply_walk
        else:
            assert 4 * 1000 <= edges <= 4 * (1000 + int(np.diff(off).max()))
    with pytest.raises(oracle_mod.OracleError):
        RefGraph.adopt_csr(np.array([0, 1, 1], dtype=np.uint64), np.array([1], dtype=np.uint32))


@needs_ref
def test_port_power_method_matches_ground_truth(oracle_mod):
    """eval.cpp:39-59: ground truth = PwMethod with N = 231 (PPR .2)."""
    off, nb = Port.make_graph(100, 150, 3)
    g = RefGraph.from_csr(off, nb)
    assert Ref.ground_truth_steps(PPR, 0.2) == 231 and Ref.ground_truth_steps(HKPR, 5.0) == 461
    z = Port.taylor_coeffs(PPR, 0.2, 230)
    assert np.array_equal(Port.power_method(off, nb, z, 231, 5), g.ground_truth(PPR, 0.2, 5))


@needs_ref
def test_pull_oracle_matches_reference_bit_exact(oracle_mod):
    """The row-parallel pull restatement (the checker for configs 3-5 in
    tests/test_gpu_fullsize.py) equals the reference's scatter-order cheby_power
    bit for bit: ring+chord graphs, a star (one hub row), a path, and a seeded
    R-MAT / Chung-Lu graph from the generator restatement; 1, 2, 3 and 17
    interleaved columns; 1 and 5 threads; dense seeds with zeros and signs."""
    graphs = {f"ring{a}": Port.make_graph(*a) for a in ((25, 35, 31), (200, 300, 1), (1000, 1500, 5))}
    graphs["star"] = Port.edges_to_csr([[0, i] for i in range(1, 300)] + [[i, i + 1] for i in range(1, 299, 3)])
    graphs["path3"] = Port.edges_to_csr([[0, 1], [1, 2]])
    graphs["rmat"] = Port.gen_rmat(11, 8 << 11, seed=9, n_threads=3)
    graphs["chunglu"] = Port.gen_chunglu(5000, 40000, 2.1, 12.0, 800, seed=4, n_threads=2)
    for name, (off, nb) in graphs.items():
        g = RefGraph.from_csr(off, nb)
        for fam, p, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15), (PPR, 0.02, 3), (HKPR, 1.0, 1)):
            c = Port.cheby_coeffs(fam, p, K)
            src = [0, g.n - 1, g.n // 2][: min(3, g.n)]
            for cols, threads in ((src[:1], 1), (src[:2], 5), (src, 5)):
                got = Port.cheby_power_pull(off, nb, c, K, cols, n_threads=threads)
                for j, s in enumerate(cols):
                    want, _, _ = g.cheby_power(fam, p, s, K)
                    assert np.array_equal(got[j], want), (name, fam, p, s, cols, threads)
        seeds = np.stack([Port.random_vector(g.n, 11 + j, -1.0, 1.0) for j in range(17)])
        seeds[:, ::3] = 0.0
        got = Port.cheby_power_vec_pull(off, nb, Port.cheby_coeffs(PPR, 0.2, 26), 26, seeds, n_threads=4)
        for j in (0, 7, 16):
            assert np.array_equal(got[j], g.cheby_power_vec(PPR, 0.2, seeds[j], 26)), (name, j)
    with pytest.raises(oracle_mod.OracleError):
        Port.cheby_power_pull(*graphs["path3"], Port.cheby_coeffs(PPR, 0.2, 3), 3, [3])


def test_generator_restatement_equals_product_generator(oracle_mod, cpg):
    """oracle/graphgen_port.c (the reference arm's and the checkers' graph builder, no
    product library loaded) builds the same CSR as the product's host generator
    (csrc/graphgen.cu, whose device build tests/test_gpu_parity.py pins to the host
    build), for any thread count, on both models."""
    cases = [("rmat", (12, 8 << 12), dict(seed=3)), ("rmat", (16, 8 << 16), dict(seed=1)),
             ("rmat", (10, 3000), dict(a=0.45, b=0.15, c=0.15, seed=7)),
             ("chunglu", (20000, 200000, 2.1, 20.0, 12000), dict(seed=4)),
             ("chunglu", (317_080, 1_050_000, 2.5, 6.6, 0), dict(seed=2))]
    for kind, args, kw in cases:
        want = getattr(cpg, f"gen_{kind}")(*args, **kw)
        for threads in (1, 3, 8):
            got = getattr(Port, f"gen_{kind}")(*args, n_threads=threads, **kw)
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), (kind, args, threads)


# ---- golden vectors (committed; made by tests/golden/make_golden.py) -------------------
def test_port_matches_golden(golden):
    for fam, params in ((PPR, (0.2, 0.1, 0.02)), (HKPR, (5.0, 20.0, 40.0))):
        for p in params:
            tag = f"{'ppr' if fam == PPR else 'hkpr'}_{p:g}"
            assert np.array_equal(Port.cheby_coeffs(fam, p, 200), golden[f"coeffs/{tag}"])
            for row in golden[f"plans/{tag}"]:
                pl = Port.plan_truncation(fam, p, row[2])
                assert [pl.cheby_steps, pl.taylor_steps, pl.epsilon, pl.tail_bound] == list(row)
    names = sorted({k.split("/")[1] for k in golden.files if k.startswith("graph/")})
    assert len(names) >= 5
    for name in names:
        off, nb = golden[f"graph/{name}/offsets"], golden[f"graph/{name}/neighbors"]
        for tag, fam, p in (("ppr", PPR, 0.2), ("hkpr", HKPR, 5.0)):
            K = int(golden[f"graph/{name}/{tag}/K"])
            c = Port.cheby_coeffs(fam, p, K)
            for j, s in enumerate(golden[f"graph/{name}/sources"]):
                v, m, _ = Port.cheby_power(off, nb, c, K, int(s))
                assert np.array_equal(v, golden[f"graph/{name}/{tag}/values"][j])
                assert np.array_equal(m, golden[f"graph/{name}/{tag}/mass"][j])
        x = golden[f"graph/{name}/walk_x"]
        assert np.array_equal(Port.apply_walk(off, nb, x), golden[f"graph/{name}/walk_y"])
