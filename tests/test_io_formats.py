"""The formats either side of the path, CPU only: the native
edge-list parser against the reference loader's line rules (graph.cpp:126-151),
the CPGR CSR cache (graph.cpp:217-255) and the CPGT truth cache (eval.cpp:92-156)
against the unmodified reference (oracle/_ref) -- bytes, values, error types and
messages."""
import os

import numpy as np
import pytest

from oracle import OracleError, Port, Ref, RefGraph

needs_ref = pytest.mark.skipif(not Ref.available(), reason="reference library not built")

VALID = [
    "0 1\n1 2\n",
    "0 1\n1 0\n0 0\n",
    "# snap header\n\n7\t9\n9 3\n3 7\n",  # test_graph.cpp:32-41
    "  # indented comment\n1 2\r\n2 3\r\n",
    "1 2 0.5\n2 3 1e-3\n3 1 -7\n",  # a weight column is accepted
    "1 2 inf\n2 3 nan\n3 4 0x1p3\n",  # strtod accepts these
    "-5 3\n+3 -5\n3 4",  # signs, no trailing newline
    "1-2\n2 3\n",  # istream stops at '-', b = -2
    "10 20 30 abc\n20 30\n",  # only the first extra token is checked
    "9223372036854775807 -9223372036854775808\n1 2\n",
    "\t\t\n \n1\t2\t\n",
]
INVALID = [
    "0 1\n2 x\n",  # test_graph.cpp:44-47
    "0 1\n\nbad line\n",  # :48-56
    "1 2 abc\n",
    "1 2abc\n",
    "1 2 # inline comment\n",
    "1\n",
    "1 2\n3\n",
    "1,2\n",
    "99999999999999999999 1\n",
    "1 2 3e5x\n",
    "\v\n",
    "%1 2\n1 2\n",
    "1 2\n" * 5 + "x y\n" + "1 2\n" * 5,
]


def _parse(cpg, text, comment="#", threads=0):
    return cpg.parse_edge_text(text, comment, threads)


@needs_ref
@pytest.mark.parametrize("text", VALID)
def test_parser_accepts_what_the_reference_accepts(cpg, text):
    pairs = _parse(cpg, text)
    want = RefGraph.from_edge_text(text)
    off, nb = Port.edges_to_csr(pairs)  # the loader's CSR build (pinned to the reference)
    woff, wnb = want.csr()
    assert np.array_equal(off, woff) and np.array_equal(nb, wnb)


@needs_ref
@pytest.mark.parametrize("text", INVALID)
def test_parser_rejects_with_the_reference_message(cpg, text):
    with pytest.raises(OracleError) as ref_err:
        RefGraph.from_edge_text(text)
    assert ref_err.value.status == Ref.PARSE
    with pytest.raises(cpg.ParseError) as err:
        _parse(cpg, text)
    assert str(err.value) == ref_err.value.detail


@needs_ref
def test_parser_comment_char_and_empty_graph(cpg):
    assert len(_parse(cpg, "% c\n1 2\n", comment="%")) == 1
    with pytest.raises(cpg.ParseError):
        _parse(cpg, "% c\n1 2\n", comment="#")
    # no edges left: the reference raises StructuralError (test_graph.cpp:57-60); here the
    # parser returns the self-loop and the ingest drops it (tested on the GPU)
    assert _parse(cpg, "# nothing\n4 4\n").tolist() == [[4, 4]]
    assert _parse(cpg, "").shape == (0, 2)


@needs_ref
def test_parser_fuzz_against_reference(cpg):
    rng = np.random.default_rng(7)
    toks = ["0", "1", "2", "17", "-3", "+4", "x", "1.5", "nan", "#", "", "  ", "\t", "5e", "0x10", "2-", "--1"]
    agree = 0
    for trial in range(300):
        lines = []
        for _ in range(rng.integers(1, 6)):
            k = rng.integers(0, 5)
            lines.append(" ".join(toks[i] for i in rng.integers(0, len(toks), k)))
        text = "\n".join(lines) + ("\n" if rng.random() < 0.5 else "")
        try:
            want = RefGraph.from_edge_text(text)
            ref_err = None
        except OracleError as e:
            want, ref_err = None, e
        try:
            pairs = _parse(cpg, text)
            err = None
        except cpg.ParseError as e:
            pairs, err = None, e
        if ref_err is not None and ref_err.status == Ref.PARSE:
            assert err is not None and str(err) == ref_err.detail, text
        else:
            assert err is None, (text, str(err))
            if want is not None:
                off, nb = Port.edges_to_csr(pairs)
                woff, wnb = want.csr()
                assert np.array_equal(off, woff) and np.array_equal(nb, wnb), text
            else:  # the reference's StructuralError: nothing but self-loops survives
                assert ref_err.status == Ref.STRUCTURAL
                assert all(a == b for a, b in pairs), text
        agree += 1
    assert agree == 300


@needs_ref
def test_parser_threads_agree_and_first_error_wins(cpg):
    rng = np.random.default_rng(3)
    pairs = rng.integers(-1000, 1000, size=(400_000, 2))
    text = "".join(f"{a} {b}\n" for a, b in pairs)
    for t in (1, 2, 8):
        assert np.array_equal(_parse(cpg, text, threads=t), pairs)
    lines = text.splitlines(keepends=True)
    bad = lines[:123_456] + ["7 oops\n"] + lines[123_456:300_000] + ["q\n"] + lines[300_000:]
    for t in (1, 8):
        with pytest.raises(cpg.ParseError, match=r'^line 123457: expected two integers, got "7 oops"$'):
            _parse(cpg, "".join(bad), threads=t)


@needs_ref
def test_csr_cache_bytes_and_round_trip_match_reference(cpg, tmp_path):
    for off, nb in (Port.make_graph(40, 60, 3), Port.edges_to_csr([[0, 1]])):
        g = cpg.Graph.from_csr(off, nb)
        p = tmp_path / "g.cpgr"
        cpg.write_csr_cache(g, p)
        ref = RefGraph.from_csr(off, nb)
        assert p.read_bytes() == ref.csr_cache_bytes()  # graph.cpp:217-232, bit-exact
        h = cpg.read_csr_cache(p)
        assert np.array_equal(h.offsets(), off) and np.array_equal(h.neighbor_array(), nb)
        assert h.structure_hash() == ref.structure_hash()
        # a file the reference wrote reads back here
        p2 = tmp_path / "ref.cpgr"
        p2.write_bytes(ref.csr_cache_bytes())
        assert np.array_equal(cpg.read_csr_cache(p2).neighbor_array(), nb)


@needs_ref
def test_csr_cache_errors_match_reference(cpg, tmp_path):
    off, nb = Port.make_graph(20, 30, 5)
    good = RefGraph.from_csr(off, nb).csr_cache_bytes()
    bad_sym = bytearray(good)
    bad_sym[-4:] = (0).to_bytes(4, "little")  # breaks symmetry -> from_csr's StructuralError
    cases = {
        "magic": b"XPGR" + good[4:],
        "version": good[:4] + (2).to_bytes(4, "little") + good[8:],
        "short header": good[:12],
        "truncated": good[:-3],
        "n zero": good[:8] + (0).to_bytes(8, "little") + good[16:],
        "empty": b"",
        "asymmetric": bytes(bad_sym),
    }
    kinds = {Ref.PARSE: cpg.ParseError, Ref.STRUCTURAL: cpg.StructuralError}
    for name, data in cases.items():
        p = tmp_path / f"{name}.cpgr"
        p.write_bytes(data)
        with pytest.raises(OracleError) as ref_err:
            RefGraph.from_csr_cache_bytes(data)
        with pytest.raises(kinds[ref_err.value.status]) as err:
            cpg.read_csr_cache(p)
        if name != "asymmetric":  # from_csr's messages are pinned in test_host_api
            assert str(err.value) == ref_err.value.detail, name
    with pytest.raises(cpg.IoError):
        cpg.read_csr_cache(tmp_path / "missing.cpgr")


@needs_ref
def test_truth_cache_bytes_names_and_errors_match_reference(cpg, tmp_path):
    vals = Port.random_vector(37, 4, 0.0, 1.0)
    t = cpg.GroundTruth(vals, "ppr:alpha=0.2", 5, 231)
    p = tmp_path / "t.bin"
    cpg.write_truth_cache(t, p)
    data = p.read_bytes()
    assert data == Ref.write_truth_cache("ppr:alpha=0.2", 5, vals)  # eval.cpp:113-124
    r = cpg.read_truth_cache(p)
    assert r.kernel_descriptor == "ppr:alpha=0.2" and r.source == 5 and np.array_equal(r.values, vals)
    assert Ref.read_truth_cache(data) == ("ppr:alpha=0.2", 5, pytest.approx(vals, abs=0))
    cases = {
        "magic": b"XXXX" + data[4:],
        "version": data[:4] + (9).to_bytes(4, "little") + data[8:],
        "short": data[:10],
        "desc": data[:14],
        "values": data[:-1],
    }
    for name, bad in cases.items():
        q = tmp_path / f"{name}.bin"
        q.write_bytes(bad)
        with pytest.raises(OracleError) as ref_err:
            Ref.read_truth_cache(bad)
        assert ref_err.value.status == Ref.PARSE
        with pytest.raises(cpg.ParseError) as err:
            cpg.read_truth_cache(q)
        assert str(err.value) == ref_err.value.detail, name
    # truth_cache_filename (eval.cpp:147-156)
    off, nb = Port.make_graph(20, 25, 12)
    g = cpg.Graph.from_csr(off, nb)
    ref = RefGraph.from_csr(off, nb)
    for k, fam, par in ((cpg.Kernel.ppr(0.2), 0, 0.2), (cpg.Kernel.hkpr(5.0), 1, 5.0), (cpg.Kernel.ppr(0.1), 0, 0.1)):
        for s in (1, 2, 19):
            assert cpg.truth_cache_filename(g, k, s) == ref.truth_cache_filename(fam, par, s)
    other = cpg.Graph.from_csr(*Port.make_graph(20, 25, 13))
    assert cpg.truth_cache_filename(g, cpg.Kernel.ppr(0.2), 1) != cpg.truth_cache_filename(other, cpg.Kernel.ppr(0.2), 1)
