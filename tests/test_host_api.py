"""Host side of the product (no GPU): C-ABI exports, coefficients / truncation /
spec parsing / CSR validation restated in C++ (host_math.cpp) against the
reference and the golden vectors, generators, source selection, shard plan."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import HKPR, PPR, Port, Ref, RefGraph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")
needs_ref = pytest.mark.skipif(not Ref.available(), reason="reference library not built")


def test_library_exports_every_declared_symbol(cpg):
    """libcpg.so loads without a GPU and exports every function include/cpg.h declares."""
    with open(os.path.join(ROOT, "include", "cpg.h")) as f:
        text = f.read()
    declared = set(re.findall(r"\b(cpg_[a-z0-9_]+)\s*\(", text))
    assert len(declared) >= 25
    lib = ctypes.CDLL(cpg._lib.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(cpg._lib.SIGNATURES) >= declared, sorted(declared - set(cpg._lib.SIGNATURES))
    assert cpg._lib.lib().cpg_version().decode().startswith("cpg")


def test_coefficients_and_plans_match_golden(cpg):
    g = np.load(GOLDEN)
    for fam, params in ((PPR, (0.2, 0.1, 0.02)), (HKPR, (5.0, 20.0, 40.0))):
        for p in params:
            tag = f"{'ppr' if fam == PPR else 'hkpr'}_{p:g}"
            k = cpg.Kernel.ppr(p) if fam == PPR else cpg.Kernel.hkpr(p)
            assert np.array_equal(k.cheby_coeffs(200), g[f"coeffs/{tag}"])
            for row in g[f"plans/{tag}"]:
                pl = cpg.plan_truncation(k, row[2])
                assert [pl.cheby_steps, pl.taylor_steps, pl.epsilon, pl.tail_bound] == list(row)


@needs_ref
def test_taylor_coefficients_and_truth_steps_vs_reference(cpg):
    for fam, p in ((PPR, 0.2), (PPR, 0.02), (HKPR, 5.0), (HKPR, 40.0)):
        assert np.array_equal(cpg.Kernel(fam, p).taylor_coeffs(300), Ref.taylor_coeffs(fam, p, 300))
        assert cpg.ground_truth_steps(cpg.Kernel(fam, p)) == Ref.ground_truth_steps(fam, p)


@needs_ref
def test_coefficients_bit_exact_vs_reference(cpg):
    for a in (0.2, 0.1, 0.02, 0.5, 0.999):
        assert np.array_equal(cpg.ppr_cheby_coeffs(a, 300), Ref.ppr_cheby_coeffs(a, 300))
    for t in (5.0, 20.0, 40.0, 0.3, 1e-12, 300.0):
        assert np.array_equal(cpg.hkpr_cheby_coeffs(t, 300), Ref.hkpr_cheby_coeffs(t, 300))
    for eps in (1e-3, 1e-6, 1e-8, 1e-12, 0.999):
        for fam, p in ((PPR, 0.2), (PPR, 0.02), (HKPR, 5.0), (HKPR, 40.0)):
            k = cpg.Kernel(fam, p)
            a, b = cpg.plan_truncation(k, eps), Ref.plan_truncation(fam, p, eps)
            assert (a.cheby_steps, a.taylor_steps, a.epsilon, a.tail_bound) == (
                b.cheby_steps, b.taylor_steps, b.epsilon, b.tail_bound)


def test_parameter_errors(cpg):
    """kernels.cpp:26-33, 254-255, 343-383."""
    for bad in (0.0, 1.0, -0.1, 1.5):
        with pytest.raises(cpg.ParameterError):
            cpg.Kernel.ppr(bad)
        with pytest.raises(cpg.ParameterError):
            cpg.ppr_cheby_coeffs(bad, 3)
    with pytest.raises(cpg.ParameterError):
        cpg.Kernel.hkpr(0.0)
    with pytest.raises(cpg.ParameterError):
        cpg.hkpr_cheby_coeffs(-1.0, 3)
    for eps in (0.0, 1.0, -1e-3):
        with pytest.raises(cpg.ParameterError):
            cpg.plan_truncation(cpg.Kernel.ppr(0.2), eps)
    assert cpg.parse_kernel_spec("ppr:alpha=0.2").alpha() == 0.2
    assert cpg.parse_kernel_spec("hkpr:t=5").t() == 5.0
    for bad in ("ppr:alpha=", "ppr:beta=0.2", "ppr:alpha=0.2x", "foo:t=1", "hkpr:t=-1", "ppr"):
        with pytest.raises(cpg.ParameterError):
            cpg.parse_kernel_spec(bad)
    assert cpg.Kernel.ppr(0.2).descriptor() == "ppr:alpha=0.2"
    assert cpg.Kernel.hkpr(5).descriptor() == "hkpr:t=5"


def test_validate_csr_rejects_what_from_csr_rejects(cpg):
    """graph.cpp:51-95: every structural check raises StructuralError."""
    off, nb = Port.edges_to_csr([[0, 1], [1, 2], [2, 0], [2, 3]])
    g = cpg.Graph.from_csr(off, nb)
    assert g.node_count() == 4 and g.edge_count() == 4 and g.volume() == 8
    cases = []
    cases.append((np.array([1, 2], np.uint64), np.array([0, 0], np.uint32)))           # offsets not from 0
    cases.append((off, nb[:-1]))                                                         # coverage
    b = nb.copy(); b[0], b[1] = b[1], b[0]; cases.append((off, b))                       # unsorted
    b = nb.copy(); b[0] = 0; cases.append((off, b))                                      # self loop
    b = nb.copy(); b[-1] = 9; cases.append((off, b))                                     # out of range
    o = off.copy(); o[1] = o[0]; cases.append((o, nb))                                   # degree 0 / monotone
    a_off, a_nb = np.array([0, 1, 2, 3], np.uint64), np.array([1, 2, 0], np.uint32)     # asymmetric, odd
    cases.append((a_off, a_nb))
    a_off, a_nb = np.array([0, 1, 3, 4], np.uint64), np.array([1, 0, 2, 0], np.uint32)  # asymmetric
    cases.append((a_off, a_nb))
    for o, b in cases:
        with pytest.raises(cpg.StructuralError):
            cpg.Graph.from_csr(o, b)


@needs_ref
def test_structure_hash_matches_reference(cpg):
    off, nb = Port.make_graph(300, 500, 2)
    assert cpg.Graph.from_csr(off, nb).structure_hash() == RefGraph.from_csr(off, nb).structure_hash()


@needs_ref
@pytest.mark.parametrize("gen", ["rmat", "chunglu"])
def test_host_generators_satisfy_from_csr(cpg, gen):
    if gen == "rmat":
        off, nb = cpg.gen_rmat(12, 8 << 12, seed=3)
    else:
        off, nb = cpg.gen_chunglu(20000, 120000, 2.3, 10.0, 3000, seed=4)
    g = RefGraph.from_csr(off, nb)  # the reference's own validation accepts it
    assert g.n == len(off) - 1 and g.nnz == len(nb)
    off2, nb2 = (cpg.gen_rmat(12, 8 << 12, seed=3) if gen == "rmat"
                 else cpg.gen_chunglu(20000, 120000, 2.3, 10.0, 3000, seed=4))
    assert np.array_equal(off, off2) and np.array_equal(nb, nb2)  # deterministic


@needs_ref
def test_select_sources_matches_reference(cpg):
    off, nb = Port.make_graph(500, 800, 5)
    g = RefGraph.from_csr(off, nb)
    for seed in (1, 2, 99):
        assert np.array_equal(cpg.select_sources_uniform(g.n, 16, seed), g.select_sources_uniform(16, seed))
    with pytest.raises(cpg.ParameterError):
        cpg.select_sources_uniform(10, 11, 1)


@pytest.mark.parametrize("chunks", [1, 3])
def test_shard_plan_is_a_balanced_permutation(cpg, chunks):
    off, nb = cpg.gen_rmat(12, 8 << 12, seed=6)
    n = len(off) - 1
    deg = np.diff(off)
    for R in (1, 2, 3, 8):
        no, cr = cpg.shard_plan(off, R, chunks)
        assert cr == -(-n // (R * chunks))
        assert len(np.unique(no)) == n and no.max() < cr * R * chunks
        chunk = no // (R * cr)
        owner = (no % (R * cr)) // cr
        counts = np.bincount(owner * chunks + chunk, minlength=R * chunks)
        assert counts.max() - counts.min() <= 1
        vol = np.bincount(owner, weights=deg, minlength=R)
        assert vol.max() <= 1.1 * vol.mean() + deg.max()
        # within a (rank, chunk), rows are degree-descending
        for r in range(R):
            for c in range(chunks):
                sel = (owner == r) & (chunk == c)
                d = deg[sel][np.argsort(no[sel])]
                assert np.all(np.diff(d.astype(np.int64)) <= 0)
