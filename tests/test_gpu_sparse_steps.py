"""Sparse early steps: the first M steps of a one-hot query gather
only the rows of w_{k-1} whose support bit is set, as the reference's scatter skips
every zero entry (graph.cpp:262, `if (xu == 0.0) continue;`).

The masked steps must give the unmasked steps' results bit for bit (a skipped
gather is an exact zero), on every kernel path that takes a mask -- the combined
and split single-source steps, the fused and split batched steps at several tile
widths, the power method's Taylor steps -- for any M (including M > the steps
where the support is small, and M = K), with sources that are hubs, leaves and
isolated-ish nodes; and they must match the reference.
"""
import numpy as np
import pytest

from conftest import assert_parity

pytestmark = pytest.mark.gpu

PPR, HKPR = 0, 1


@pytest.fixture(scope="module")
def hub_graph(cpg):
    off, nb = cpg.gen_chunglu(30000, 500000, 2.0, 30.0, 12000, seed=21)
    assert np.diff(off).max() > 4096  # hubs split into several pieces
    return off, nb


def _ref(off, nb):
    from oracle import RefGraph

    return RefGraph.from_csr(off, nb)


def _sources(off, ref):
    deg = np.diff(off)
    hub = int(np.argmax(deg))              # the biggest hub: its 1-hop ball is most of the graph
    leaf = int(np.argmin(deg))             # a degree-1-ish node
    return [hub, leaf] + [int(s) for s in ref.select_sources_uniform(3, 9)]


@pytest.mark.parametrize("split", ["0", "1"])
def test_single_source_masked_equals_unmasked(cpg, gpu, hub_graph, split, monkeypatch):
    off, nb = hub_graph
    monkeypatch.setenv("CPG_STEP_SPLIT", split)
    monkeypatch.setenv("CPG_GROUP_Q", "1")
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref(off, nb)
    src = _sources(off, ref)
    for fam, param, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15)):
        kern = cpg.Kernel.ppr(param) if fam == PPR else cpg.Kernel.hkpr(param)
        monkeypatch.setenv("CPG_SPARSE_STEPS", "0")
        base, _ = cpg.cheby_power_many(g, kern, src, K)
        for M in ("1", "2", "3", "5", str(K)):
            monkeypatch.setenv("CPG_SPARSE_STEPS", M)
            got, st = cpg.cheby_power_many(g, kern, src, K)
            assert np.array_equal(got, base), (fam, M)
            assert st.mass_err_max <= 1e-9
        monkeypatch.delenv("CPG_SPARSE_STEPS")
        got, _ = cpg.cheby_power_many(g, kern, src, K)  # default M
        assert np.array_equal(got, base)
        for j, s in enumerate(src):
            want, _, _ = ref.cheby_power(fam, param, s, K)
            assert_parity(got[j], want)


@pytest.mark.parametrize("kern", ["1", "0"])  # scan + fill kernels / masked full-step kernels
@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("tile", [4, 16, 64])
def test_batched_masked_equals_unmasked(cpg, gpu, hub_graph, split, tile, kern, monkeypatch):
    off, nb = hub_graph
    monkeypatch.setenv("CPG_BATCH_SPLIT", split)
    monkeypatch.setenv("CPG_SPARSE_KERNEL", kern)
    g = cpg.Graph.from_csr(off, nb)
    ref = _ref(off, nb)
    src = _sources(off, ref)
    kern = cpg.Kernel.ppr(0.2)
    monkeypatch.setenv("CPG_SPARSE_STEPS", "0")
    base, _ = cpg.cheby_power_many(g, kern, src, 26, batched=True, tile=tile)
    for M in ("1", "2", "3", "26"):
        monkeypatch.setenv("CPG_SPARSE_STEPS", M)
        got, st = cpg.cheby_power_many(g, kern, src, 26, batched=True, tile=tile)
        assert np.array_equal(got, base), M
        assert 0.0 <= st.mass_err_max <= 1e-9
    monkeypatch.delenv("CPG_SPARSE_STEPS")
    got, _ = cpg.cheby_power_many(g, kern, src, 26, batched=True, tile=tile)
    assert np.array_equal(got, base)
    for j, s in enumerate(src):
        want, _, _ = ref.cheby_power(PPR, 0.2, s, 26)
        assert_parity(got[j], want)


def test_power_method_masked_equals_unmasked(cpg, gpu, hub_graph, monkeypatch):
    off, nb = hub_graph
    g = cpg.Graph.from_csr(off, nb)
    kern = cpg.Kernel.ppr(0.2)
    monkeypatch.setenv("CPG_SPARSE_STEPS", "0")
    base = cpg.power_method(g, kern, 7, 40).values
    monkeypatch.setenv("CPG_SPARSE_STEPS", "3")
    assert np.array_equal(cpg.power_method(g, kern, 7, 40).values, base)


def test_small_graphs_and_star_sources(cpg, gpu, monkeypatch):
    """Tiny graphs where the support fills the graph in one hop (star centre,
    path), and K = 1, 2 (M capped at K)."""
    from oracle import Port

    monkeypatch.setenv("CPG_GROUP_Q", "1")  # query groups take no mask
    for off, nb in (Port.edges_to_csr([[0, 1], [0, 2], [0, 3]]), Port.edges_to_csr([[0, 1], [1, 2]]),
                    Port.make_graph(200, 300, 1)):
        g = cpg.Graph.from_csr(off, nb)
        ref = _ref(off, nb)
        n = g.node_count()
        for K in (1, 2, 26):
            kern = cpg.Kernel.ppr(0.2)
            monkeypatch.setenv("CPG_SPARSE_STEPS", "0")
            base, _ = cpg.cheby_power_many(g, kern, list(range(n))[:8], K)
            baseb, _ = cpg.cheby_power_many(g, kern, list(range(n))[:8], K, batched=True, tile=8)
            monkeypatch.setenv("CPG_SPARSE_STEPS", "3")
            got, _ = cpg.cheby_power_many(g, kern, list(range(n))[:8], K)
            gotb, _ = cpg.cheby_power_many(g, kern, list(range(n))[:8], K, batched=True, tile=8)
            assert np.array_equal(got, base) and np.array_equal(gotb, baseb)
            for j in range(min(n, 8)):
                want, _, _ = ref.cheby_power(PPR, 0.2, j, K)
                assert_parity(gotb[j], want)


def test_default_rule_and_override(cpg, gpu, hub_graph, monkeypatch):
    """cpg_sparse_early_steps reports the library's rule (api.cu sparse_steps): batched tiles
    mask 2 steps from 1.5 M directed edges, one source only where the iterate exceeds the L2;
    CPG_SPARSE_STEPS overrides; never more than K."""
    off, nb = hub_graph
    monkeypatch.delenv("CPG_SPARSE_STEPS", raising=False)
    small = cpg.Graph.from_csr(off, nb).device(0)          # ~1 M directed edges
    assert len(nb) < 1500000
    assert small.sparse_early_steps(16, 26) == 0 and small.sparse_early_steps(1, 26) == 0
    boff, bnb = cpg.gen_chunglu(60000, 1200000, 2.0, 40.0, 12000, seed=5)
    assert len(bnb) >= 1500000
    big = cpg.Graph.from_csr(boff, bnb).device(0)
    assert big.sparse_early_steps(16, 26) == 2 and big.sparse_early_steps(16, 1) == 1
    assert big.sparse_early_steps(1, 26) == 0               # iterate fits the L2
    monkeypatch.setenv("CPG_SPARSE_STEPS", "5")
    assert small.sparse_early_steps(16, 26) == 5 and small.sparse_early_steps(1, 3) == 3
    # the default batched path on the bigger graph (masks on) against the reference
    monkeypatch.delenv("CPG_SPARSE_STEPS")
    ref = _ref(boff, bnb)
    src = _sources(boff, ref)
    got, st = cpg.cheby_power_many(big, cpg.Kernel.ppr(0.2), src, 26, batched=True, tile=8)
    for j, s in enumerate(src):
        want, _, _ = ref.cheby_power(PPR, 0.2, s, 26)
        assert_parity(got[j], want)
    assert st.mass_err_max <= 1e-9
