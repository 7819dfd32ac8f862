"""oracle -- CPU checkers for the ChebyPower hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package, and only as the checker or the timed CPU baseline -- never as the
thing measured or shipped.  The product package ``paper_2412_10789_b200``
does not import it.

Two checkers, both ctypes over shared objects built by ``oracle/Makefile``:

* ``Port``  -- ``oracle/_ref/libcheby_oracle.so``, the C restatement in
  ``oracle/cheby_oracle.c`` (each function cites the reference file:line it
  restates).
* ``Ref``   -- ``oracle/_ref/libchebyprop_ref.so``, the UNMODIFIED reference
  library compiled from ``/root/reference/proj/src`` plus ``ref_shim.cpp``.

The Port is pinned against the Ref bit-for-bit (``tests/test_oracle_pin.py``)
and against the reference tests' known answers and the committed golden
vectors (``tests/golden/``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
PORT_SO = os.path.join(REF_DIR, "libcheby_oracle.so")
REF_SO = os.path.join(REF_DIR, "libchebyprop_ref.so")

PPR, HKPR = 0, 1

_u64p = POINTER(c_uint64)
_u32p = POINTER(c_uint32)
_f64p = POINTER(c_double)
_i64p = POINTER(c_int64)


def build() -> None:
    """Compile the checkers (the reference part only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _csr(offsets, nbrs):
    return (np.ascontiguousarray(offsets, dtype=np.uint64),
            np.ascontiguousarray(nbrs, dtype=np.uint32))


class OracleError(RuntimeError):
    def __init__(self, msg, status=0, detail=""):
        super().__init__(msg)
        self.status = status  # Ref: the reference exception's code (Ref.PARSE, ...)
        self.detail = detail  # Ref: the reference exception's what()


class _Plan:
    def __init__(self, cheby_steps, taylor_steps, epsilon, tail_bound):
        self.cheby_steps = int(cheby_steps)
        self.taylor_steps = int(taylor_steps)
        self.epsilon = float(epsilon)
        self.tail_bound = float(tail_bound)


class _CpoPlan(ctypes.Structure):
    _fields_ = [("cheby_steps", c_uint64), ("taylor_steps", c_uint64),
                ("epsilon", c_double), ("tail_bound", c_double)]


class Port:
    """The C restatement (oracle/cheby_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(PORT_SO):
                build()
            L = ctypes.CDLL(PORT_SO)
            L.cpo_ppr_cheby_coeffs.argtypes = [c_double, c_uint64, _f64p]
            L.cpo_hkpr_cheby_coeffs.argtypes = [c_double, c_uint64, _f64p]
            L.cpo_taylor_coeffs.argtypes = [c_int, c_double, c_uint64, _f64p]
            L.cpo_plan_truncation.argtypes = [c_int, c_double, c_double, POINTER(_CpoPlan)]
            L.cpo_apply_walk.argtypes = [c_uint32, _u64p, _u32p, _f64p, _f64p]
            L.cpo_apply_walk.restype = None
            L.cpo_cheby_power_vec.argtypes = [c_uint32, _u64p, _u32p, _f64p, c_uint64, _f64p,
                                              _f64p, _f64p, _f64p, _f64p, _u64p]
            L.cpo_cheby_power.argtypes = [c_uint32, _u64p, _u32p, _f64p, c_uint64, c_uint32,
                                          _f64p, _f64p, _u64p]
            L.cpo_power_method.argtypes = [c_uint32, _u64p, _u32p, _f64p, c_uint64, c_uint32, _f64p]
            L.cpo_select_sources_uniform.argtypes = [c_uint32, c_uint64, c_uint64, _u32p]
            L.cpo_ring_chord_edges.argtypes = [c_uint64, c_uint64, c_uint64, _i64p]
            L.cpo_ring_chord_edges.restype = c_uint64
            L.cpo_random_vector.argtypes = [c_uint64, c_uint64, c_double, c_double, _f64p]
            L.cpo_random_vector.restype = None
            L.cpo_edges_to_csr.argtypes = [_i64p, c_uint64, _u32p, _u64p, _u64p, _u32p]
            L.cpo_cheby_power_pool.argtypes = [c_uint32, _u64p, _u32p, _f64p, c_uint64, _u32p,
                                               c_uint64, _f64p, c_int]
            L.cpo_apply_walk_pool.argtypes = [c_uint32, _u64p, _u32p, c_int, c_uint64, _u64p]
            L.cpo_apply_walk_pool.restype = c_double
            L.cpo_cheby_power_pull.argtypes = [c_uint32, _u64p, _u32p, _f64p, c_uint64, _u32p, c_uint32,
                                               _f64p, c_int]
            L.cpo_cheby_power_vec_pull.argtypes = [c_uint32, _u64p, _u32p, _f64p, c_uint64, _f64p, c_uint32,
                                                   _f64p, c_int]
            _pp = POINTER(c_void_p)
            L.cpo_gen_rmat.argtypes = [c_uint32, c_uint64, c_double, c_double, c_double, c_uint64, c_int, _pp,
                                       _pp, _u32p, _u64p]
            L.cpo_gen_chunglu.argtypes = [c_uint32, c_uint64, c_double, c_double, c_uint32, c_uint64, c_int,
                                          _pp, _pp, _u32p, _u64p]
            L.cpo_gen_free.argtypes = [c_void_p, c_void_p]
            L.cpo_gen_free.restype = None
            cls._lib = L
        return cls._lib

    @staticmethod
    def _check(rc, what):
        if rc != 0:
            raise OracleError(f"{what}: status {rc}")

    # -- coefficients / truncation ------------------------------------------------
    @classmethod
    def ppr_cheby_coeffs(cls, alpha, max_index):
        out = np.empty(max_index + 1)
        cls._check(cls.lib().cpo_ppr_cheby_coeffs(alpha, max_index, _p(out, _f64p)), "ppr coeffs")
        return out

    @classmethod
    def hkpr_cheby_coeffs(cls, t, max_index):
        out = np.empty(max_index + 1)
        cls._check(cls.lib().cpo_hkpr_cheby_coeffs(t, max_index, _p(out, _f64p)), "hkpr coeffs")
        return out

    @classmethod
    def cheby_coeffs(cls, family, param, max_index):
        return (cls.ppr_cheby_coeffs if family == PPR else cls.hkpr_cheby_coeffs)(param, max_index)

    @classmethod
    def taylor_coeffs(cls, family, param, max_index):
        out = np.empty(max_index + 1)
        cls._check(cls.lib().cpo_taylor_coeffs(family, param, max_index, _p(out, _f64p)), "taylor")
        return out

    @classmethod
    def plan_truncation(cls, family, param, eps):
        p = _CpoPlan()
        cls._check(cls.lib().cpo_plan_truncation(family, param, eps, ctypes.byref(p)), "plan")
        return _Plan(p.cheby_steps, p.taylor_steps, p.epsilon, p.tail_bound)

    # -- graph fixtures -------------------------------------------------------------
    @classmethod
    def edges_to_csr(cls, pairs):
        """Reference load_edge_list semantics (graph.cpp:113-171) on label pairs."""
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
        n, nnz = c_uint32(), c_uint64()
        L = cls.lib()
        cls._check(L.cpo_edges_to_csr(_p(pairs, _i64p), len(pairs), ctypes.byref(n),
                                      ctypes.byref(nnz), None, None), "edges_to_csr")
        off = np.empty(n.value + 1, dtype=np.uint64)
        nb = np.empty(nnz.value, dtype=np.uint32)
        cls._check(L.cpo_edges_to_csr(_p(pairs, _i64p), len(pairs), ctypes.byref(n),
                                      ctypes.byref(nnz), _p(off, _u64p), _p(nb, _u32p)),
                   "edges_to_csr")
        return off, nb

    @classmethod
    def ring_chord_pairs(cls, n, extra, seed):
        buf = np.empty(2 * (n + extra), dtype=np.int64)
        m = cls.lib().cpo_ring_chord_edges(n, extra, seed, _p(buf, _i64p))
        return buf[: 2 * m].reshape(-1, 2)

    @classmethod
    def make_graph(cls, n, extra, seed):
        """tests/oracles.hpp:175-178 -- ring + seeded chords through the loader."""
        return cls.edges_to_csr(cls.ring_chord_pairs(n, extra, seed))

    @classmethod
    def random_vector(cls, n, seed, lo=-1.0, hi=1.0):
        out = np.empty(n)
        cls.lib().cpo_random_vector(n, seed, lo, hi, _p(out, _f64p))
        return out

    # -- the path ---------------------------------------------------------------------
    @classmethod
    def apply_walk(cls, offsets, nbrs, x):
        offsets, nbrs = _csr(offsets, nbrs)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(len(offsets) - 1)
        cls.lib().cpo_apply_walk(len(offsets) - 1, _p(offsets, _u64p), _p(nbrs, _u32p),
                                 _p(x, _f64p), _p(out, _f64p))
        return out

    @classmethod
    def cheby_power_vec(cls, offsets, nbrs, coeffs, K, seed, trace=False):
        offsets, nbrs = _csr(offsets, nbrs)
        n = len(offsets) - 1
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        seed = np.ascontiguousarray(seed, dtype=np.float64)
        out = np.empty(n)
        mass = np.empty(K + 1)
        rt = np.empty((K + 1, n)) if trace else None
        et = np.empty((K + 1, n)) if trace else None
        work = c_uint64()
        cls._check(cls.lib().cpo_cheby_power_vec(n, _p(offsets, _u64p), _p(nbrs, _u32p),
                                                 _p(coeffs, _f64p), K, _p(seed, _f64p),
                                                 _p(out, _f64p), _p(mass, _f64p), _p(rt, _f64p),
                                                 _p(et, _f64p), ctypes.byref(work)), "cheby_power_vec")
        if trace:
            return out, mass, rt, et
        return out, mass, work.value

    @classmethod
    def cheby_power(cls, offsets, nbrs, coeffs, K, source):
        n = len(offsets) - 1
        seed = np.zeros(n)
        seed[source] = 1.0
        out, mass, work = cls.cheby_power_vec(offsets, nbrs, coeffs, K, seed)
        return out, mass, work

    @classmethod
    def power_method(cls, offsets, nbrs, zeta, n_steps, source):
        offsets, nbrs = _csr(offsets, nbrs)
        zeta = np.ascontiguousarray(zeta, dtype=np.float64)
        out = np.empty(len(offsets) - 1)
        cls._check(cls.lib().cpo_power_method(len(offsets) - 1, _p(offsets, _u64p), _p(nbrs, _u32p),
                                               _p(zeta, _f64p), n_steps, source, _p(out, _f64p)),
                   "power_method")
        return out

    @classmethod
    def cheby_power_pool(cls, offsets, nbrs, coeffs, K, sources, n_threads, keep=True):
        offsets, nbrs = _csr(offsets, nbrs)
        n = len(offsets) - 1
        sources = np.ascontiguousarray(sources, dtype=np.uint32)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.empty((len(sources), n)) if keep else None
        cls._check(cls.lib().cpo_cheby_power_pool(n, _p(offsets, _u64p), _p(nbrs, _u32p),
                                                  _p(coeffs, _f64p), K, _p(sources, _u32p),
                                                  len(sources), _p(out, _f64p), n_threads), "pool")
        return out

    @classmethod
    def apply_walk_pool(cls, offsets, nbrs, n_threads, edges_per_thread=0):
        """(wall seconds, edges) for n_threads concurrent dense apply_walk runs, each over
        ~edges_per_thread edges (0 = one full iteration each)."""
        offsets, nbrs = _csr(offsets, nbrs)
        done = c_uint64()
        t = cls.lib().cpo_apply_walk_pool(len(offsets) - 1, _p(offsets, _u64p), _p(nbrs, _u32p), n_threads,
                                          edges_per_thread, ctypes.byref(done))
        if t < 0:
            raise OracleError("apply_walk_pool: out of memory")
        return t, done.value

    @classmethod
    def cheby_power_pull(cls, offsets, nbrs, coeffs, K, sources, n_threads=None):
        """values[S][n] for S unit seeds: the row-parallel pull restatement (bit-exact with
        the reference's scatter loop on a valid CSR), S <= 64 columns interleaved."""
        offsets, nbrs = _csr(offsets, nbrs)
        n = len(offsets) - 1
        src = np.ascontiguousarray(np.atleast_1d(sources), dtype=np.uint32)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.empty((len(src), n))
        nt = n_threads or os.cpu_count() or 1
        cls._check(cls.lib().cpo_cheby_power_pull(n, _p(offsets, _u64p), _p(nbrs, _u32p), _p(coeffs, _f64p), K,
                                                  _p(src, _u32p), len(src), _p(out, _f64p), nt), "cheby_power_pull")
        return out

    @classmethod
    def cheby_power_vec_pull(cls, offsets, nbrs, coeffs, K, seeds, n_threads=None):
        offsets, nbrs = _csr(offsets, nbrs)
        n = len(offsets) - 1
        seeds = np.ascontiguousarray(np.atleast_2d(seeds), dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.empty_like(seeds)
        nt = n_threads or os.cpu_count() or 1
        cls._check(cls.lib().cpo_cheby_power_vec_pull(n, _p(offsets, _u64p), _p(nbrs, _u32p), _p(coeffs, _f64p), K,
                                                      _p(seeds, _f64p), seeds.shape[0], _p(out, _f64p), nt),
                   "cheby_power_vec_pull")
        return out

    @classmethod
    def _gen_result(cls, rc, off, nbr, n, nnz, what):
        cls._check(rc, what)
        o = np.ctypeslib.as_array(ctypes.cast(off, _u64p), shape=(n.value + 1,)).copy()
        b = np.ctypeslib.as_array(ctypes.cast(nbr, _u32p), shape=(nnz.value,)).copy()
        cls.lib().cpo_gen_free(off, nbr)
        return o, b

    @classmethod
    def gen_rmat(cls, scale, n_samples, a=0.57, b=0.19, c=0.19, seed=1, n_threads=None):
        """Host restatement of the repo's R-MAT generator (graphgen_port.c): same CSR."""
        off, nbr, n, nnz = c_void_p(), c_void_p(), c_uint32(), c_uint64()
        rc = cls.lib().cpo_gen_rmat(scale, n_samples, a, b, c, seed, n_threads or os.cpu_count() or 1,
                                    ctypes.byref(off), ctypes.byref(nbr), ctypes.byref(n), ctypes.byref(nnz))
        return cls._gen_result(rc, off, nbr, n, nnz, "gen_rmat")

    @classmethod
    def gen_chunglu(cls, n_ids, n_samples, exponent, mean_degree, max_degree=0, seed=1, n_threads=None):
        """Host restatement of the repo's Chung-Lu generator (graphgen_port.c): same CSR."""
        off, nbr, n, nnz = c_void_p(), c_void_p(), c_uint32(), c_uint64()
        rc = cls.lib().cpo_gen_chunglu(n_ids, n_samples, exponent, mean_degree, max_degree, seed,
                                       n_threads or os.cpu_count() or 1, ctypes.byref(off), ctypes.byref(nbr),
                                       ctypes.byref(n), ctypes.byref(nnz))
        return cls._gen_result(rc, off, nbr, n, nnz, "gen_chunglu")

    @classmethod
    def select_sources_uniform(cls, n, count, seed):
        out = np.empty(count, dtype=np.uint32)
        cls._check(cls.lib().cpo_select_sources_uniform(n, count, seed, _p(out, _u32p)), "sources")
        return out


class Ref:
    """The unmodified reference library (oracle/_ref/libchebyprop_ref.so)."""

    _lib = None

    @classmethod
    def available(cls):
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise OracleError(f"{REF_SO} not built (reference sources absent?)")
            L = ctypes.CDLL(REF_SO)
            L.ref_last_error.restype = c_char_p
            L.ref_ppr_cheby_coeffs.argtypes = [c_double, c_uint64, _f64p]
            L.ref_hkpr_cheby_coeffs.argtypes = [c_double, c_uint64, _f64p]
            L.ref_taylor_coeffs.argtypes = [c_int, c_double, c_uint64, _f64p]
            L.ref_plan_truncation.argtypes = [c_int, c_double, c_double, _u64p, _f64p]
            L.ref_ground_truth_steps.argtypes = [c_int, c_double]
            L.ref_ground_truth_steps.restype = c_uint64
            L.ref_graph_from_csr.argtypes = [_u64p, _u32p, c_uint64, c_uint64, POINTER(c_void_p)]
            L.ref_graph_adopt_csr.argtypes = [_u64p, _u32p, c_uint64, c_uint64, POINTER(c_void_p)]
            L.ref_apply_walk_subset_pool.argtypes = [c_void_p, c_int, c_uint64, _u64p, _f64p]
            L.ref_graph_from_edge_text.argtypes = [c_char_p, POINTER(c_void_p)]
            L.ref_graph_free.argtypes = [c_void_p]
            L.ref_graph_free.restype = None
            for f in ("ref_graph_n", "ref_graph_nnz", "ref_graph_hash"):
                getattr(L, f).argtypes = [c_void_p]
                getattr(L, f).restype = c_uint64
            L.ref_graph_csr.argtypes = [c_void_p, _u64p, _u32p]
            L.ref_graph_original_ids.argtypes = [c_void_p, _i64p]
            L.ref_graph_original_ids.restype = c_uint64
            L.ref_apply_walk.argtypes = [c_void_p, _f64p, _f64p]
            L.ref_cheby_power.argtypes = [c_void_p, c_int, c_double, c_uint32, c_uint64, _f64p,
                                          _f64p, _u64p, _f64p]
            L.ref_cheby_power_trace.argtypes = [c_void_p, c_int, c_double, c_uint32, c_uint64,
                                                _f64p, _f64p, _f64p]
            L.ref_cheby_power_vec.argtypes = [c_void_p, c_int, c_double, _f64p, c_uint64, _f64p]
            L.ref_general_gp_vector.argtypes = [c_void_p, c_int, c_double, c_double, _f64p,
                                                c_uint64, _f64p]
            L.ref_ground_truth.argtypes = [c_void_p, c_int, c_double, c_uint32, _f64p]
            L.ref_select_sources_uniform.argtypes = [c_void_p, c_uint64, c_uint64, _u32p]
            L.ref_cheby_power_pool.argtypes = [c_void_p, c_int, c_double, _u32p, c_uint64,
                                               c_uint64, c_int, _f64p, _f64p]
            L.ref_measure.argtypes = [c_void_p, _f64p, _f64p, _f64p, _u32p]
            L.ref_write_csr_cache.argtypes = [c_void_p, c_void_p, c_uint64, _u64p]
            L.ref_read_csr_cache.argtypes = [c_void_p, c_uint64, POINTER(c_void_p)]
            L.ref_write_truth_cache.argtypes = [c_char_p, c_uint64, _f64p, c_uint64, c_void_p, c_uint64, _u64p]
            L.ref_read_truth_cache.argtypes = [c_void_p, c_uint64, c_char_p, c_uint64, _u64p, _f64p, c_uint64,
                                               _u64p]
            L.ref_truth_cache_filename.argtypes = [c_void_p, c_int, c_double, c_uint32, c_char_p, c_uint64]
            cls._lib = L
        return cls._lib

    @classmethod
    def _check(cls, rc, what):
        if rc != 0:
            raise OracleError(f"{what}: status {rc}: {cls.lib().ref_last_error().decode()}", rc,
                              cls.lib().ref_last_error().decode())

    # status codes of ref_shim.cpp's guarded(): the reference's exception types
    PARAMETER, STRUCTURAL, OTHER, PARSE, IO = 1, 5, 6, 7, 8

    @classmethod
    def write_truth_cache(cls, desc, source, values):
        """write_truth_cache (eval.cpp:113-124) -> bytes."""
        values = np.ascontiguousarray(values, dtype=np.float64)
        n = np.zeros(1, dtype=np.uint64)
        cls._check(cls.lib().ref_write_truth_cache(desc.encode(), source, _p(values, _f64p), len(values), None, 0,
                                                   _p(n, _u64p)), "write_truth_cache")
        buf = ctypes.create_string_buffer(int(n[0]))
        cls._check(cls.lib().ref_write_truth_cache(desc.encode(), source, _p(values, _f64p), len(values), buf,
                                                   int(n[0]), _p(n, _u64p)), "write_truth_cache")
        return buf.raw

    @classmethod
    def read_truth_cache(cls, data):
        """read_truth_cache (eval.cpp:126-145) of bytes -> (descriptor, source, values)."""
        desc = ctypes.create_string_buffer(4096)
        src = np.zeros(1, dtype=np.uint64)
        n = np.zeros(1, dtype=np.uint64)
        vals = np.empty(max(1, len(data) // 8))
        cls._check(cls.lib().ref_read_truth_cache(data, len(data), desc, len(desc), _p(src, _u64p), _p(vals, _f64p),
                                                  len(vals), _p(n, _u64p)), "read_truth_cache")
        return desc.value.decode(), int(src[0]), vals[: int(n[0])].copy()

    @classmethod
    def ppr_cheby_coeffs(cls, alpha, max_index):
        out = np.empty(max_index + 1)
        cls._check(cls.lib().ref_ppr_cheby_coeffs(alpha, max_index, _p(out, _f64p)), "ppr")
        return out

    @classmethod
    def hkpr_cheby_coeffs(cls, t, max_index):
        out = np.empty(max_index + 1)
        cls._check(cls.lib().ref_hkpr_cheby_coeffs(t, max_index, _p(out, _f64p)), "hkpr")
        return out

    @classmethod
    def cheby_coeffs(cls, family, param, max_index):
        return (cls.ppr_cheby_coeffs if family == PPR else cls.hkpr_cheby_coeffs)(param, max_index)

    @classmethod
    def taylor_coeffs(cls, family, param, max_index):
        out = np.empty(max_index + 1)
        cls._check(cls.lib().ref_taylor_coeffs(family, param, max_index, _p(out, _f64p)), "taylor")
        return out

    @classmethod
    def plan_truncation(cls, family, param, eps):
        s = np.zeros(2, dtype=np.uint64)
        d = np.zeros(2)
        cls._check(cls.lib().ref_plan_truncation(family, param, eps, _p(s, _u64p), _p(d, _f64p)),
                   "plan")
        return _Plan(s[0], s[1], d[1], d[0])

    @classmethod
    def ground_truth_steps(cls, family, param):
        return int(cls.lib().ref_ground_truth_steps(family, param))


class RefGraph:
    """A reference ``chebyprop::Graph`` (built by ``Graph::from_csr`` / ``load_edge_list``)."""

    def __init__(self, handle):
        self.h = c_void_p(handle) if not isinstance(handle, c_void_p) else handle
        L = Ref.lib()
        self.n = int(L.ref_graph_n(self.h))
        self.nnz = int(L.ref_graph_nnz(self.h))

    @classmethod
    def from_csr(cls, offsets, nbrs):
        offsets, nbrs = _csr(offsets, nbrs)
        h = c_void_p()
        Ref._check(Ref.lib().ref_graph_from_csr(_p(offsets, _u64p), _p(nbrs, _u32p),
                                                len(offsets) - 1, len(nbrs), ctypes.byref(h)),
                   "from_csr")
        return cls(h)

    @classmethod
    def adopt_csr(cls, offsets, nbrs):
        """A reference Graph over an already-validated CSR without from_csr's O(nnz log d)
        symmetry check (ref_shim.cpp: ref_graph_adopt_csr).  structure_hash() reads 0."""
        offsets, nbrs = _csr(offsets, nbrs)
        h = c_void_p()
        Ref._check(Ref.lib().ref_graph_adopt_csr(_p(offsets, _u64p), _p(nbrs, _u32p),
                                                 len(offsets) - 1, len(nbrs), ctypes.byref(h)),
                   "adopt_csr")
        return cls(h)

    def apply_walk_subset_pool(self, n_threads, edges_per_thread):
        """(wall seconds, edges) for n_threads concurrent reference apply_walk_from_subset
        calls (graph.cpp:275-288), each over a contiguous run of ~edges_per_thread slots."""
        done = np.zeros(1, dtype=np.uint64)
        wall = np.zeros(1)
        Ref._check(Ref.lib().ref_apply_walk_subset_pool(self.h, n_threads, edges_per_thread,
                                                        _p(done, _u64p), _p(wall, _f64p)), "subset_pool")
        return float(wall[0]), int(done[0])

    @classmethod
    def from_edge_text(cls, text):
        h = c_void_p()
        Ref._check(Ref.lib().ref_graph_from_edge_text(text.encode(), ctypes.byref(h)), "load")
        return cls(h)

    def __del__(self):
        try:
            if self.h:
                Ref.lib().ref_graph_free(self.h)
                self.h = None
        except Exception:
            pass

    def csr(self):
        off = np.empty(self.n + 1, dtype=np.uint64)
        nb = np.empty(self.nnz, dtype=np.uint32)
        Ref.lib().ref_graph_csr(self.h, _p(off, _u64p), _p(nb, _u32p))
        return off, nb

    def measure(self, truth, est):
        """measure (eval.cpp:18-37) -> (l1, l2, deg_norm_inf, argmax_node)."""
        truth = np.ascontiguousarray(truth, dtype=np.float64)
        est = np.ascontiguousarray(est, dtype=np.float64)
        out = np.empty(3)
        arg = np.zeros(1, dtype=np.uint32)
        Ref._check(Ref.lib().ref_measure(self.h, _p(truth, _f64p), _p(est, _f64p), _p(out, _f64p), _p(arg, _u32p)),
                   "measure")
        return float(out[0]), float(out[1]), float(out[2]), int(arg[0])

    def csr_cache_bytes(self):
        """write_csr_cache (graph.cpp:217-232) -> bytes."""
        n = np.zeros(1, dtype=np.uint64)
        Ref._check(Ref.lib().ref_write_csr_cache(self.h, None, 0, _p(n, _u64p)), "write_csr_cache")
        buf = ctypes.create_string_buffer(int(n[0]))
        Ref._check(Ref.lib().ref_write_csr_cache(self.h, buf, int(n[0]), _p(n, _u64p)), "write_csr_cache")
        return buf.raw

    @classmethod
    def from_csr_cache_bytes(cls, data):
        """read_csr_cache (graph.cpp:234-255) of bytes."""
        h = c_void_p()
        Ref._check(Ref.lib().ref_read_csr_cache(data, len(data), ctypes.byref(h)), "read_csr_cache")
        return cls(h)

    def truth_cache_filename(self, family, param, source):
        out = ctypes.create_string_buffer(4096)
        Ref._check(Ref.lib().ref_truth_cache_filename(self.h, family, param, source, out, len(out)),
                   "truth_cache_filename")
        return out.value.decode()

    def original_ids(self):
        k = int(Ref.lib().ref_graph_original_ids(self.h, None))
        out = np.empty(k, dtype=np.int64)
        Ref.lib().ref_graph_original_ids(self.h, _p(out, _i64p))
        return out

    def structure_hash(self):
        return int(Ref.lib().ref_graph_hash(self.h))

    def apply_walk(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.n)
        Ref._check(Ref.lib().ref_apply_walk(self.h, _p(x, _f64p), _p(out, _f64p)), "apply_walk")
        return out

    def cheby_power(self, family, param, source, K, with_mass=True):
        out = np.empty(self.n)
        mass = np.empty(K + 1) if with_mass else None
        st = np.zeros(2, dtype=np.uint64)
        wall = c_double()
        Ref._check(Ref.lib().ref_cheby_power(self.h, family, param, source, K, _p(out, _f64p),
                                             _p(mass, _f64p), _p(st, _u64p), ctypes.byref(wall)),
                   "cheby_power")
        return out, mass, {"iterations": int(st[0]), "push_work": int(st[1]),
                           "wall_seconds": wall.value}

    def cheby_power_trace(self, family, param, source, K):
        out = np.empty(self.n)
        rt = np.empty((K + 1, self.n))
        et = np.empty((K + 1, self.n))
        Ref._check(Ref.lib().ref_cheby_power_trace(self.h, family, param, source, K, _p(out, _f64p),
                                                   _p(rt, _f64p), _p(et, _f64p)), "trace")
        return out, rt, et

    def cheby_power_vec(self, family, param, seed, K):
        seed = np.ascontiguousarray(seed, dtype=np.float64)
        out = np.empty(self.n)
        Ref._check(Ref.lib().ref_cheby_power_vec(self.h, family, param, _p(seed, _f64p), K,
                                                 _p(out, _f64p)), "cheby_power_vec")
        return out

    def general_gp_vector(self, family, param, a, x, steps):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.n)
        Ref._check(Ref.lib().ref_general_gp_vector(self.h, family, param, a, _p(x, _f64p), steps,
                                                   _p(out, _f64p)), "gp")
        return out

    def ground_truth(self, family, param, source):
        out = np.empty(self.n)
        Ref._check(Ref.lib().ref_ground_truth(self.h, family, param, source, _p(out, _f64p)), "truth")
        return out

    def select_sources_uniform(self, count, seed):
        out = np.empty(count, dtype=np.uint32)
        Ref._check(Ref.lib().ref_select_sources_uniform(self.h, count, seed, _p(out, _u32p)),
                   "select_sources")
        return out

    def cheby_power_pool(self, family, param, sources, K, n_threads, keep=False):
        sources = np.ascontiguousarray(sources, dtype=np.uint32)
        out = np.empty((len(sources), self.n)) if keep else None
        wall = c_double()
        Ref._check(Ref.lib().ref_cheby_power_pool(self.h, family, param, _p(sources, _u32p),
                                                  len(sources), K, n_threads, _p(out, _f64p),
                                                  ctypes.byref(wall)), "pool")
        return out, wall.value


def edge_text(pairs) -> str:
    return "".join(f"{int(a)} {int(b)}\n" for a, b in np.asarray(pairs).reshape(-1, 2))


def parity(gpu, ref, topk=100, tie_tol=1e-12):
    """max-abs, L1 and top-k set agreement (value desc, id asc: tools/chebyprop.cpp:151-156).

    ``topk_equal`` is exact set equality.  ``topk_equal_mod_ties`` allows the
    sets to differ only in nodes whose scores lie within ``tie_tol`` of the k-th
    score in both vectors (structural ties broken by last-bit rounding)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.abs(gpu - ref)
    k = min(topk, len(ref))

    def top(v):
        order = np.lexsort((np.arange(len(v)), -v))
        return order[:k]

    tg, tr = top(gpu), top(ref)
    sg, sr = set(tg.tolist()), set(tr.tolist())
    eq = sg == sr
    mod_ties = eq
    if not eq and k > 0:
        kth = ref[tr[-1]]
        diff = np.array(sorted(sg ^ sr))
        mod_ties = bool(np.all(np.abs(ref[diff] - kth) <= tie_tol) and np.all(np.abs(gpu[diff] - kth) <= tie_tol))
    return {"max_abs": float(d.max()) if len(d) else 0.0, "l1": float(d.sum()), "topk_equal": eq,
            "topk_equal_mod_ties": mod_ties}
