"""SURVEY.md 8f rows 3-4 on the GPU: device measure (eval.cpp:18-37) and the device
estimate+measure query against the reference; the truth cache round trip through
load_or_compute_truth (eval.cpp:158-192, the reference's test_eval.cpp:110-160 cases);
text / CPGR loading into a GPU graph with the loader's semantics."""
import numpy as np
import pytest

from oracle import Port, Ref, RefGraph

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not Ref.available(), reason="reference library not built")
PPR, HKPR = 0, 1


def _check_report(got, want):
    l1, l2, dn, arg = want
    assert abs(got.l1 - l1) <= 1e-14 * max(1.0, l1)  # the reference's own tolerance, test_eval.cpp:66
    assert abs(got.l2 - l2) <= 1e-14 * max(1.0, l2)
    assert got.deg_norm_inf == dn  # exact
    assert got.argmax_node == arg  # exact, ties keep the first id


@needs_ref
def test_measure_matches_reference(cpg):
    path3 = Port.edges_to_csr([[0, 1], [1, 2]])
    g = cpg.Graph.from_csr(*path3)
    ref = RefGraph.from_csr(*path3)
    v = np.array([0.1, 0.5, 0.4])
    r = cpg.measure(v, v, g)  # test_eval.cpp:39-45: identical vectors give zeros
    assert (r.l1, r.l2, r.deg_norm_inf, r.argmax_node) == (0.0, 0.0, 0.0, 0)
    pair = cpg.load_edge_list("0 1\n")  # test_eval.cpp:46-54: hand computation on a swap
    r = cpg.measure(np.array([1.0, 0.0]), np.array([0.0, 1.0]), pair)
    assert r.l1 == 2.0 and r.l2 == np.sqrt(2.0) and r.deg_norm_inf == 1.0 and r.argmax_node == 0
    for n, extra, seed in ((100, 150, 9), (30, 40, 4), (5000, 9000, 2)):
        off, nb = Port.make_graph(n, extra, seed)
        g = cpg.Graph.from_csr(off, nb)
        ref = RefGraph.from_csr(off, nb)
        a = Port.random_vector(g.node_count(), 1, 0.0, 1.0)
        b = Port.random_vector(g.node_count(), 2, 0.0, 1.0)
        _check_report(cpg.measure(a, b, g), ref.measure(a, b))
        ab, ba = cpg.measure(a, b, g), cpg.measure(b, a, g)  # test_eval.cpp:70-80: symmetry
        assert (ab.l1, ab.l2, ab.deg_norm_inf) == (ba.l1, ba.l2, ba.deg_norm_inf)
        # ties in d/deg: the first id wins, like the reference's strict '>'
        t = np.zeros(g.node_count())
        e = np.zeros(g.node_count())
        deg = np.diff(off).astype(float)
        for u in (n - 1, 7, 3 * n // 4):
            e[u] = 0.25 * deg[u]
        _check_report(cpg.measure(t, e, g), ref.measure(t, e))
        assert cpg.measure(t, e, g).argmax_node == 7


@needs_ref
def test_measure_stacks_and_large_graph(cpg):
    off, nb = cpg.gen_chunglu(200_000, 1_000_000, 2.3, 10.0, 2000, seed=5)
    g = cpg.Graph.from_csr(off, nb)
    ref = RefGraph.from_csr(off, nb)
    n = g.node_count()
    T = np.stack([Port.random_vector(n, s, 0.0, 1e-3) for s in (1, 2, 3)])
    E = np.stack([Port.random_vector(n, s, 0.0, 1e-3) for s in (4, 5, 6)])
    reps = cpg.measure(T, E, g)
    for i in range(3):
        l1, l2, dn, arg = ref.measure(T[i], E[i])
        assert abs(reps[i].l1 - l1) <= 1e-13 * l1 and abs(reps[i].l2 - l2) <= 1e-13 * l2
        assert reps[i].deg_norm_inf == dn and reps[i].argmax_node == arg
    with pytest.raises(cpg.ParameterError):
        cpg.measure(T[0], E[0][:-1], g)


@needs_ref
def test_cheby_power_measure_matches_reference_eval(cpg):
    """Device estimate + device measure == the reference's cheby_power, ground_truth and measure."""
    off, nb = cpg.gen_rmat(12, 8 * 4096, seed=3)
    g = cpg.Graph.from_csr(off, nb)
    ref = RefGraph.from_csr(off, nb)
    srcs = [0, 5, 17, 100, 1000]
    for fam, par, kern in ((PPR, 0.2, cpg.Kernel.ppr(0.2)), (HKPR, 5.0, cpg.Kernel.hkpr(5.0))):
        K = cpg.plan_truncation(kern, 1e-6).cheby_steps
        truths = np.stack([ref.ground_truth(fam, par, s) for s in srcs])
        reps, st = cpg.cheby_power_measure(g, kern, srcs, K, truths)
        assert st.iterations == K and st.push_work == K * len(nb) * len(srcs)
        for s, t, r in zip(srcs, truths, reps):
            est, _, _ = ref.cheby_power(fam, par, s, K)
            l1, l2, dn, arg = ref.measure(t, est)
            # the estimate differs from the reference's by <= 1e-15; the metrics by that much
            assert abs(r.l1 - l1) <= 1e-12 and abs(r.l2 - l2) <= 1e-12 and abs(r.deg_norm_inf - dn) <= 1e-12


def test_truth_cache_round_trip_and_regeneration(cpg, tmp_path):
    """test_eval.cpp:110-160 restated: round trip, no-op rerun, corrupt magic regenerates."""
    off, nb = Port.make_graph(20, 25, 12)
    g = cpg.Graph.from_csr(off, nb)
    k = cpg.Kernel.ppr(0.2)
    first, cached = cpg.load_or_compute_truth(g, k, 3, str(tmp_path))
    assert not cached
    second, cached = cpg.load_or_compute_truth(g, k, 3, str(tmp_path))
    assert cached and np.array_equal(first.values, second.values)
    assert second.kernel_descriptor == k.descriptor() and second.source == 3
    assert second.truncation == cpg.ground_truth_steps(k)
    cpg.load_or_compute_truth(g, k, 4, str(tmp_path))
    path = tmp_path / cpg.truth_cache_filename(g, k, 4)
    raw = bytearray(path.read_bytes())
    raw[:4] = b"XXXX"
    path.write_bytes(bytes(raw))
    redo, cached = cpg.load_or_compute_truth(g, k, 4, str(tmp_path))
    assert not cached
    assert np.array_equal(redo.values, cpg.ground_truth(g, k, 4))
    cpg.read_truth_cache(path)  # healthy again
    with pytest.raises(cpg.ParameterError):
        cpg.load_or_compute_truth(g, k, 99, str(tmp_path))


@needs_ref
def test_truth_cache_interoperates_with_reference_ground_truth(cpg, tmp_path):
    off, nb = Port.make_graph(300, 500, 7)
    g = cpg.Graph.from_csr(off, nb)
    ref = RefGraph.from_csr(off, nb)
    k = cpg.Kernel.hkpr(5.0)
    # a file written from the reference's ground truth is picked up as cached
    want = ref.ground_truth(HKPR, 5.0, 11)
    name = ref.truth_cache_filename(HKPR, 5.0, 11)
    (tmp_path / name).write_bytes(Ref.write_truth_cache(k.descriptor(), 11, want))
    t, cached = cpg.load_or_compute_truth(g, k, 11, str(tmp_path))
    assert cached and np.array_equal(t.values, want)
    # a truth computed here matches the reference's to 1e-13
    t2, cached = cpg.load_or_compute_truth(g, k, 12, str(tmp_path))
    assert not cached and np.abs(t2.values - ref.ground_truth(HKPR, 5.0, 12)).max() <= 1e-13


@needs_ref
def test_text_and_csr_cache_load_onto_gpu(cpg, tmp_path):
    text = "# header\n7\t9\n9 3 0.5\n3 7\n3 3\n12 7\n"
    p = tmp_path / "g.txt"
    p.write_text(text)
    g = cpg.load_edge_list_file(str(p))
    ref = RefGraph.from_edge_text(text)
    woff, wnb = ref.csr()
    assert np.array_equal(g.offsets(), woff) and np.array_equal(g.neighbor_array(), wnb)
    assert np.array_equal(g.original_ids, ref.original_ids())
    with pytest.raises(cpg.StructuralError):  # test_graph.cpp:57-60
        cpg.load_edge_list("# nothing\n4 4\n")
    with pytest.raises(cpg.ParseError):
        cpg.load_edge_list("0 1\n2 x\n")
    with pytest.raises(cpg.IoError):
        cpg.load_edge_list_file(str(tmp_path / "missing.txt"))
    # CPGR round trip through the GPU path
    off, nb = cpg.gen_chunglu(50_000, 300_000, 2.3, 10.0, 1000, seed=9)
    g = cpg.Graph.from_csr(off, nb)
    c = tmp_path / "g.cpgr"
    cpg.write_csr_cache(g, c)
    h = cpg.read_csr_cache(c)
    k = cpg.Kernel.ppr(0.2)
    a = cpg.cheby_power(g, k, 17, 26).values
    b = cpg.cheby_power(h, k, 17, 26).values
    assert np.array_equal(a, b)
    want, _, _ = RefGraph.from_csr(off, nb).cheby_power(PPR, 0.2, 17, 26)
    assert np.abs(b - want).max() <= 1e-12
