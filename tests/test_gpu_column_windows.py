"""Column-window hub pieces: the biggest hub rows are cut at the window
boundaries of the warm tier of the iterate and their pieces run window-major, claimed in
list order.  The cuts change only how a hub row's sum is associated (pieces are still added
left to right by the ordered last-arriver combine), so the results stay within the parity
bar of the reference, are bit-reproducible, and the sparse early steps on a column-window
table still equal its full steps bit for bit.
"""
import numpy as np
import pytest

from conftest import assert_parity

pytestmark = pytest.mark.gpu

PPR, HKPR = 0, 1


@pytest.fixture(scope="module")
def hub_graph(cpg):
    off, nb = cpg.gen_chunglu(30000, 500000, 2.0, 30.0, 12000, seed=21)
    assert np.diff(off).max() > 4096
    return off, nb


def _env(monkeypatch, deg, spread="1"):
    monkeypatch.setenv("CPG_BATCH_SPLIT", "1")   # the piece + row kernels on a small graph
    monkeypatch.setenv("CPG_HOT_MB", "1")        # hot prefix: 8192 rows at B = 16, 2048 at B = 64
    monkeypatch.setenv("CPG_CW_HOT_MB", "1")     # the piece kernel's own (the first window starts there)
    monkeypatch.setenv("CPG_CW_MB", "1")
    monkeypatch.setenv("CPG_CW_WARM_MB", "3")
    monkeypatch.setenv("CPG_CW_SPREAD", spread)
    monkeypatch.setenv("CPG_CW_DEG", str(deg))  # 0 = uniform pieces
    monkeypatch.setenv("CPG_CW_MIN_ROWS", "1")  # the test graph has a few dozen hub rows


@pytest.mark.parametrize("tile", [16, 64])
@pytest.mark.parametrize("spread", ["0", "1"])
def test_column_window_pieces_match_reference(cpg, gpu, hub_graph, tile, spread, monkeypatch):
    from oracle import RefGraph

    off, nb = hub_graph
    ref = RefGraph.from_csr(off, nb)
    deg = np.diff(off)
    src = [int(np.argmax(deg)), int(np.argmin(deg))] + [int(s) for s in ref.select_sources_uniform(tile - 2, 3)]
    monkeypatch.setenv("CPG_SPARSE_STEPS", "0")
    _env(monkeypatch, 0)
    plain = cpg.Graph.from_csr(off, nb).device(0)
    base, _ = cpg.cheby_power_many(plain, cpg.Kernel.ppr(0.2), src, 26, batched=True, tile=tile)
    plain.close()
    _env(monkeypatch, 2048, spread)
    dg = cpg.Graph.from_csr(off, nb).device(0)
    for fam, param, K in ((PPR, 0.2, 26), (HKPR, 5.0, 15)):
        kern = cpg.Kernel.ppr(param) if fam == PPR else cpg.Kernel.hkpr(param)
        got, st = cpg.cheby_power_many(dg, kern, src, K, batched=True, tile=tile)
        again, _ = cpg.cheby_power_many(dg, kern, src, K, batched=True, tile=tile)
        assert np.array_equal(got, again)                       # fixed reduction order
        assert st.mass_err_max <= 1e-9
        for j in (0, 1, 2, len(src) - 1):
            want, _, _ = ref.cheby_power(fam, param, src[j], K)
            assert_parity(got[j], want)
        if fam == PPR:
            assert np.abs(got - base).max() <= 1e-14            # only the association of hub sums differs
        # sparse early steps on the column-window table: bit-identical to its full steps
        for M in ("1", "2", "3"):
            monkeypatch.setenv("CPG_SPARSE_STEPS", M)
            masked, _ = cpg.cheby_power_many(dg, kern, src, K, batched=True, tile=tile)
            assert np.array_equal(masked, got), (fam, M)
        monkeypatch.setenv("CPG_SPARSE_STEPS", "0")
    # a ragged tile (fewer sources than the tile) and the power method share the table
    few, _ = cpg.cheby_power_many(dg, cpg.Kernel.ppr(0.2), src[:3], 26, batched=True, tile=tile)
    for j in range(3):
        want, _, _ = ref.cheby_power(PPR, 0.2, src[j], 26)
        assert_parity(few[j], want)
    dg.close()


@pytest.mark.parametrize("R,C", [(2, 1), (3, 2)])
def test_column_window_pieces_on_sharded_ranks(cpg, gpu, hub_graph, R, C, monkeypatch):
    """A row-sharded rank cuts its own hub rows at the same (global) column windows: R ranks on one
    GPU through the loopback data plane, every rank's gathered result against the reference."""
    import threading

    from oracle import RefGraph

    off, nb = hub_graph
    _env(monkeypatch, 512)
    monkeypatch.setenv("CPG_CHUNKS", str(C))
    ref = RefGraph.from_csr(off, nb)
    deg = np.diff(off)
    src = [int(np.argmax(deg)), 5, 77, len(off) - 2] + [int(s) for s in ref.select_sources_uniform(12, 4)]
    grp = cpg.LoopbackGroup(R)
    shards = [cpg.DeviceGraph.loopback(off, nb, r, grp) for r in range(R)]
    out, errs = [None] * R, []

    def work(r):
        try:
            out[r] = cpg.cheby_power_many(shards[r], cpg.Kernel.ppr(0.2), src, 26, batched=True, tile=16)
        except BaseException as e:
            errs.append((r, e))

    for sparse in ("0", "1"):
        monkeypatch.setenv("CPG_SPARSE_STEPS", sparse)
        th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        assert not errs, errs
        for j in (0, 1, 5, len(src) - 1):
            want, _, _ = ref.cheby_power(PPR, 0.2, src[j], 26)
            for r in range(R):
                assert_parity(out[r][0][j], want)
        for r in range(R):
            assert out[r][1].mass_err_max <= 1e-9
            assert np.array_equal(out[r][0], out[0][0])
    for dg in shards:
        dg.close()
