"""paper_2412_10789_b200 -- B200-native ChebyPower (arXiv 2412.10789) behind the
reference's own API.

Python mirror of the reference C++ surface for the hot path
(reference paths relative to /root/reference/proj):

=============================  ==================================================
this package                   reference
=============================  ==================================================
``Graph.from_csr``             ``Graph::from_csr``            graph.hpp:51-53, graph.cpp:48-104
``Kernel.ppr / Kernel.hkpr``   ``Kernel::ppr / Kernel::hkpr``  kernels.hpp:15-42, kernels.cpp:37-51
``ppr_cheby_coeffs``           ``ppr_cheby_coeffs``            kernels.cpp:157-170
``hkpr_cheby_coeffs``          ``hkpr_cheby_coeffs``           kernels.cpp:172-194
``plan_truncation``            ``plan_truncation``             kernels.cpp:253-341
``parse_kernel_spec``          ``parse_kernel_spec``           kernels.cpp:343-383 (ppr/hkpr)
``cheby_power``                ``cheby_power``                 solvers.cpp:236-239
``cheby_power_vec``            ``cheby_power_vec``             solvers.cpp:197-234
``apply_walk``                 ``apply_walk``                  graph.cpp:269-273
``general_gp_vector/matrix``   same (ChebyPower only)          solvers.cpp:390-414
``cheby_power_many``           bench worker pool of cheby_power (tools/chebyprop.cpp:305-334),
                               single-source or batched 64-column SpMM tiles
=============================  ==================================================

Errors follow error.hpp: ``ParameterError`` (a ``ValueError``) for bad sources,
K < 1, alpha/t/epsilon out of domain, length mismatches; ``StructuralError`` for
invalid CSR.  All compute runs in ``libcpg.so`` (sm_100a); there is no CPU path.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import cpg_graph_info, cpg_plan, cpg_stats

__all__ = [
    "ParameterError", "StructuralError", "DeviceError", "Graph", "DeviceGraph", "Kernel", "KernelFamily",
    "TruncationPlan", "SolveStats", "Estimate", "ppr_cheby_coeffs", "hkpr_cheby_coeffs", "plan_truncation",
    "parse_kernel_spec", "cheby_power", "cheby_power_vec", "cheby_power_many", "apply_walk",
    "general_gp_vector", "general_gp_matrix", "gen_rmat", "gen_chunglu", "DeviceCSR", "power_method",
    "ground_truth", "ground_truth_steps", "select_sources_uniform", "shard_plan", "cheby_power_topk",
    "ingest_edges", "load_edge_list_file", "cheby_power_many_pipelined", "sync", "LoopbackGroup",
    "ParseError", "IoError", "parse_edge_text", "load_edge_list", "write_csr_cache", "read_csr_cache",
    "ErrorReport", "measure", "cheby_power_measure", "GroundTruth", "write_truth_cache", "read_truth_cache",
    "truth_cache_filename", "load_or_compute_truth",
]


# ---- errors (error.hpp:7-30) -------------------------------------------------------------
class ParameterError(ValueError):
    pass


class StructuralError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    pass


class ParseError(RuntimeError):
    """Malformed edge-list text or binary cache header (error.hpp:8-10)."""


class IoError(RuntimeError):
    """Cannot open / read / write a file (error.hpp:28-30)."""


def _check(rc: int, what: str = "") -> None:
    if rc == L.CPG_OK:
        return
    msg = L.last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == L.CPG_EINVAL:
        raise ParameterError(msg)
    if rc == L.CPG_ESTRUCT:
        raise StructuralError(msg)
    if rc == L.CPG_EPARSE:
        raise ParseError(msg)
    if rc == L.CPG_EIO:
        raise IoError(msg)
    raise DeviceError(f"[status {rc}] {msg}")


def _f64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _u32p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _u64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


# ---- kernels (kernels.hpp) ---------------------------------------------------------------
class KernelFamily:
    Ppr = 0
    Hkpr = 1


def ppr_cheby_coeffs(alpha: float, max_index: int) -> np.ndarray:
    out = np.empty(max_index + 1)
    _check(L.lib().cpg_ppr_cheby_coeffs(float(alpha), int(max_index), _f64p(out)))
    return out


def hkpr_cheby_coeffs(t: float, max_index: int) -> np.ndarray:
    out = np.empty(max_index + 1)
    _check(L.lib().cpg_hkpr_cheby_coeffs(float(t), int(max_index), _f64p(out)))
    return out


def _fmt(v: float) -> str:
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") else r


class Kernel:
    """Propagation kernel f (PPR or HKPR), validated like kernels.cpp:26-51."""

    def __init__(self, family: int, param: float):
        self._family = family
        self._param = float(param)

    @staticmethod
    def ppr(alpha: float) -> "Kernel":
        if not (0.0 < alpha < 1.0):
            raise ParameterError(f"ppr: alpha must lie in (0,1), got {alpha}")
        return Kernel(KernelFamily.Ppr, alpha)

    @staticmethod
    def hkpr(t: float) -> "Kernel":
        if not (t > 0.0):
            raise ParameterError(f"hkpr: t must be positive, got {t}")
        return Kernel(KernelFamily.Hkpr, t)

    def family(self) -> int:
        return self._family

    def alpha(self) -> float:
        if self._family != KernelFamily.Ppr:
            raise ParameterError("kernel is not ppr")
        return self._param

    def t(self) -> float:
        if self._family != KernelFamily.Hkpr:
            raise ParameterError("kernel is not hkpr")
        return self._param

    @property
    def param(self) -> float:
        return self._param

    def cheby_coeffs(self, max_index: int) -> np.ndarray:
        out = np.empty(max_index + 1)
        _check(L.lib().cpg_cheby_coeffs(self._family, self._param, int(max_index), _f64p(out)))
        return out

    def taylor_coeffs(self, max_index: int) -> np.ndarray:
        """zeta_0 .. zeta_max_index (kernels.cpp:78-96)."""
        out = np.empty(max_index + 1)
        _check(L.lib().cpg_taylor_coeffs(self._family, self._param, int(max_index), _f64p(out)))
        return out

    def descriptor(self) -> str:  # kernels.cpp:132-137
        if self._family == KernelFamily.Ppr:
            return "ppr:alpha=" + _fmt(self._param)
        return "hkpr:t=" + _fmt(self._param)

    def __repr__(self) -> str:
        return f"Kernel({self.descriptor()})"


def parse_kernel_spec(spec: str) -> Kernel:
    fam, par = ctypes.c_int(), ctypes.c_double()
    _check(L.lib().cpg_parse_kernel_spec(spec.encode(), ctypes.byref(fam), ctypes.byref(par)))
    return Kernel(fam.value, par.value)


@dataclass
class TruncationPlan:  # kernels.hpp:48-53
    cheby_steps: int
    taylor_steps: int
    epsilon: float
    tail_bound: float


def plan_truncation(kernel: Kernel, epsilon: float) -> TruncationPlan:
    p = cpg_plan()
    _check(L.lib().cpg_plan_truncation(kernel.family(), kernel.param, float(epsilon), ctypes.byref(p)))
    return TruncationPlan(int(p.cheby_steps), int(p.taylor_steps), p.epsilon, p.tail_bound)


# ---- graph (graph.hpp) -------------------------------------------------------------------
class Graph:
    """Immutable CSR of a simple undirected graph (graph.hpp:26-66).

    ``offsets`` uint64[n+1] and ``neighbors`` uint32[2m] in the reference's own
    layout; device copies are created lazily per GPU (``device(i)``) and cached.
    """

    def __init__(self, offsets: np.ndarray, neighbors: np.ndarray, structure_hash: int = 0):
        self._off = offsets
        self._nbr = neighbors
        self._hash = structure_hash
        self._dev: dict[int, DeviceGraph] = {}

    @staticmethod
    def from_csr(offsets, neighbors, validate: bool = True) -> "Graph":
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        h = ctypes.c_uint64(0)
        if validate:
            if len(off) == 0:
                raise StructuralError("CSR offsets must start at 0")
            _check(L.lib().cpg_validate_csr(_u64p(off), _u32p(nbr), len(off) - 1, len(nbr), ctypes.byref(h)))
        return Graph(off, nbr, h.value)

    def node_count(self) -> int:
        return len(self._off) - 1

    def edge_count(self) -> int:
        return len(self._nbr) // 2

    def volume(self) -> int:
        return len(self._nbr)

    def degree(self, u: int) -> int:
        return int(self._off[u + 1] - self._off[u])

    def degrees(self) -> np.ndarray:
        return np.diff(self._off).astype(np.int64)

    def offsets(self) -> np.ndarray:
        return self._off

    def neighbor_array(self) -> np.ndarray:
        return self._nbr

    def structure_hash(self) -> int:
        return self._hash

    def device(self, dev: int = 0) -> "DeviceGraph":
        if dev not in self._dev:
            self._dev[dev] = DeviceGraph.from_host(self._off, self._nbr, dev)
        return self._dev[dev]


class DeviceGraph:
    """A ``cpg_graph*`` handle: the relabelled CSR resident on one GPU (or one row shard)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        self._pending = []  # host outputs of pipelined calls whose copies may be in flight
        self.info = cpg_graph_info()
        _check(L.lib().cpg_graph_info_get(self._h, ctypes.byref(self.info)))

    @classmethod
    def from_host(cls, offsets, neighbors, device: int = 0, validate: bool = False) -> "DeviceGraph":
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        h = ctypes.c_void_p()
        _check(L.lib().cpg_graph_create(_u64p(off), _u32p(nbr), len(off) - 1, len(nbr), device, int(validate),
                                        ctypes.byref(h)), "cpg_graph_create")
        return cls(h)

    @classmethod
    def from_device(cls, csr: "DeviceCSR") -> "DeviceGraph":
        h = ctypes.c_void_p()
        _check(L.lib().cpg_graph_create_device(csr.offsets_ptr, csr.neighbors_ptr, csr.n, csr.nnz, csr.device,
                                               ctypes.byref(h)), "cpg_graph_create_device")
        return cls(h)

    @classmethod
    def sharded(cls, offsets_ptr, neighbors_ptr, n: int, nnz: int, on_device: bool, device: int, rank: int,
                nranks: int, nccl_id: Optional[bytes]) -> "DeviceGraph":
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(L.lib().cpg_graph_create_sharded(offsets_ptr, neighbors_ptr, n, nnz, int(on_device), device, rank,
                                                nranks, idbuf, ctypes.byref(h)), "cpg_graph_create_sharded")
        return cls(h)

    @classmethod
    def loopback(cls, offsets, neighbors, rank: int, group: "LoopbackGroup", device: int = 0) -> "DeviceGraph":
        """Rank ``rank``'s shard of a row-partitioned graph whose data plane is the test-only
        loopback group (every rank on ``device`` in this process; see include/cpg.h)."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        h = ctypes.c_void_p()
        _check(L.lib().cpg_graph_create_loopback(off.ctypes.data, nbr.ctypes.data, len(off) - 1, len(nbr), 0, device,
                                                 rank, group.handle, ctypes.byref(h)), "cpg_graph_create_loopback")
        g = cls(h)
        g._group = group  # the group outlives its handles
        return g

    @classmethod
    def multi(cls, offsets, neighbors, devices) -> "DeviceGraph":
        """One handle over several GPUs of this process (cpg_graph_create_multi): the CSR is
        row-partitioned across ``devices``; queries run every shard from its own host thread."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        devs = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        _check(L.lib().cpg_graph_create_multi(_u64p(off), _u32p(nbr), len(off) - 1, len(nbr), devs, len(devices),
                                              ctypes.byref(h)), "cpg_graph_create_multi")
        return cls(h)

    @classmethod
    def multi_loopback(cls, offsets, neighbors, n_ranks: int, device: int = 0) -> "DeviceGraph":
        """Test hook: the multi-device facade over ``n_ranks`` shards on one GPU (loopback plane)."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        h = ctypes.c_void_p()
        _check(L.lib().cpg_graph_create_multi_loopback(_u64p(off), _u32p(nbr), len(off) - 1, len(nbr), device,
                                                       n_ranks, ctypes.byref(h)), "cpg_graph_create_multi_loopback")
        return cls(h)

    @property
    def handle(self):
        return self._h

    @property
    def n(self) -> int:
        return self.info.n

    def bytes_per_step(self, tile: int = 1) -> float:
        return float(L.lib().cpg_bytes_per_step(self._h, tile))

    def sparse_early_steps(self, tile: int, K: int) -> int:
        """Steps at the head of a one-hot query that gather only nonzero rows."""
        return int(L.lib().cpg_sparse_early_steps(self._h, tile, K))

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().cpg_graph_destroy(self._h)  # synchronises the device first
            self._h = None
            self._pending = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """Test-only data plane joining ``nranks`` shard handles of one process on one GPU."""

    def __init__(self, nranks: int):
        self._h = ctypes.c_void_p()
        _check(L.lib().cpg_loopback_group_create(int(nranks), ctypes.byref(self._h)), "loopback group")
        self.nranks = int(nranks)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                L.lib().cpg_loopback_group_destroy(self._h)
                self._h = None
        except Exception:
            pass


def shard_plan(offsets, nranks: int, chunks: int = 1):
    """Host restatement of the device relabel + row partition: (new_of_old[n], cr).

    Node order (degree desc, id asc); position i -> rank i % R, t = i // R,
    chunk t % C, j = t // C; global id chunk*R*cr + rank*cr + j (cr rows per
    rank and chunk; local row chunk*cr + j)."""
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = len(off) - 1
    out = np.empty(n, dtype=np.uint32)
    cr = ctypes.c_uint32()
    _check(L.lib().cpg_shard_plan(_u64p(off), n, nranks, chunks, _u32p(out), ctypes.byref(cr)))
    return out, int(cr.value)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(L.lib().cpg_nccl_unique_id(buf))
    return buf.raw


# ---- solvers (solvers.hpp) ---------------------------------------------------------------
@dataclass
class SolveStats:  # solvers.hpp:18-25 + device evidence
    iterations: int = 0
    push_work: int = 0
    walks: int = 0
    wall_seconds: float = 0.0
    algorithm: str = "chebypower"
    params: str = ""
    device_ms: float = 0.0
    mass_err_max: float = 0.0
    bytes_model: float = 0.0
    launches: int = 0


@dataclass
class Estimate:  # solvers.hpp:27-30
    values: np.ndarray
    stats: SolveStats = field(default_factory=SolveStats)


StepObserver = Callable[[int, np.ndarray, np.ndarray], None]


def _to_stats(s: cpg_stats, K: int) -> SolveStats:
    return SolveStats(iterations=int(s.iterations), push_work=int(s.push_work), wall_seconds=s.wall_seconds,
                      algorithm="chebypower", params=f"K={K}", device_ms=s.device_ms,
                      mass_err_max=s.mass_err_max, bytes_model=s.bytes_model, launches=int(s.launches))


def _dev(g, device: int) -> DeviceGraph:
    return g if isinstance(g, DeviceGraph) else g.device(device)


def _steps(cheby_steps) -> int:
    K = int(cheby_steps)
    if K < 1:
        raise ParameterError("cheby_power: cheby_steps must be >= 1")  # solvers.cpp:201
    return K


def cheby_power(g, kernel: Kernel, source: int, cheby_steps: int, observer: Optional[StepObserver] = None,
                device: int = 0) -> Estimate:
    """yhat = sum_{k=0..K} c_k T_k(P) e_source (solvers.cpp:236-239) on the GPU.

    wall_seconds covers coefficients + iterations, not the first call's graph
    upload (the reference times queries on a loaded graph, README.md:93-95)."""
    K = _steps(cheby_steps)
    dg = _dev(g, device)
    t0 = time.perf_counter()
    c = kernel.cheby_coeffs(K)  # coefficients inside the call, like solvers.cpp:205
    if source < 0 or source >= dg.n:
        raise ParameterError(f"source node {source} out of range")
    n = dg.n
    out = np.empty(n)
    if observer is not None:  # slow path: per-step T_k and partial estimates (tests only)
        rt = np.empty((K + 1, n))
        et = np.empty((K + 1, n))
        _check(L.lib().cpg_chebypower_trace(dg.handle, _f64p(c), K, int(source), out.ctypes.data,
                                            rt.ctypes.data, et.ctypes.data))
        for k in range(K + 1):
            observer(k, rt[k], et[k])
        st = SolveStats(iterations=K, push_work=K * int(dg.info.nnz), params=f"K={K}")
    else:
        s = cpg_stats()
        src = np.array([source], dtype=np.uint32)
        _check(L.lib().cpg_chebypower(dg.handle, _f64p(c), K, _u32p(src), 1, out.ctypes.data, ctypes.byref(s)))
        st = _to_stats(s, K)
    st.wall_seconds = time.perf_counter() - t0
    return Estimate(out, st)


def cheby_power_vec(g, kernel: Kernel, seed, cheby_steps: int, observer: Optional[StepObserver] = None,
                    device: int = 0) -> Estimate:
    """cheby_power_vec (solvers.cpp:197-234) for a dense seed vector (or an (s, n) stack).

    A non-None observer (one seed vector only) takes the trace slow path and is
    called with (k, T_k(P) x, partial estimate) for k = 0..K (solvers.cpp:215, 219, 226)."""
    K = _steps(cheby_steps)
    dg = _dev(g, device)
    t0 = time.perf_counter()
    seeds = np.ascontiguousarray(seed, dtype=np.float64)
    single = seeds.ndim == 1
    seeds = seeds.reshape(-1, seeds.shape[-1])
    if seeds.shape[1] != dg.n:
        raise ParameterError("seed vector length mismatch")  # solvers.cpp:36-37
    c = kernel.cheby_coeffs(K)
    if observer is not None:
        if not single:
            raise ParameterError("observer takes one seed vector")
        n = dg.n
        out = np.empty(n)
        rt = np.empty((K + 1, n))
        et = np.empty((K + 1, n))
        _check(L.lib().cpg_chebypower_vec_trace(dg.handle, _f64p(c), K, _f64p(seeds), out.ctypes.data,
                                                rt.ctypes.data, et.ctypes.data))
        for k in range(K + 1):
            observer(k, rt[k], et[k])
        st = SolveStats(iterations=K, push_work=K * int(dg.info.nnz), params=f"K={K}")
        st.wall_seconds = time.perf_counter() - t0
        return Estimate(out, st)
    out = np.empty_like(seeds)
    s = cpg_stats()
    _check(L.lib().cpg_chebypower_vec(dg.handle, _f64p(c), K, _f64p(seeds), seeds.shape[0], out.ctypes.data,
                                      ctypes.byref(s)))
    st = _to_stats(s, K)
    st.wall_seconds = time.perf_counter() - t0
    return Estimate(out[0] if single else out, st)


def cheby_power_many(g, kernel: Kernel, sources: Sequence[int], cheby_steps: int, out: Optional[np.ndarray] = None,
                     batched: bool = False, tile: int = 64, device: int = 0):
    """Many single-source queries in one call: returns (values[n_sources, n], SolveStats).

    ``batched=False`` runs each source through the fused SpMV step;
    ``batched=True`` runs tiles of ``tile`` sources through the SpMM step.
    ``out`` may be a pinned host buffer (then D2H overlaps compute).
    """
    K = _steps(cheby_steps)
    dg = _dev(g, device)
    src = np.ascontiguousarray(sources, dtype=np.uint32)
    c = kernel.cheby_coeffs(K)
    if out is None:
        out = np.empty((len(src), dg.n))
    s = cpg_stats()
    ptr = out.ctypes.data if isinstance(out, np.ndarray) else int(out)
    if batched:
        _check(L.lib().cpg_chebypower_batched(dg.handle, _f64p(c), K, _u32p(src), len(src), tile, ptr,
                                              ctypes.byref(s)))
    else:
        _check(L.lib().cpg_chebypower(dg.handle, _f64p(c), K, _u32p(src), len(src), ptr, ctypes.byref(s)))
    return out, _to_stats(s, K)


def cheby_power_many_pipelined(g, kernel: Kernel, sources: Sequence[int], cheby_steps: int, out,
                               tile: int = 64, device: int = 0):
    """Batched queries whose result copy into ``out`` (a pinned host buffer) is left in
    flight: it overlaps the next call's steps.  Call ``sync(g)`` before reading ``out``.
    Returns the SolveStats of the compute."""
    K = _steps(cheby_steps)
    dg = _dev(g, device)
    src = np.ascontiguousarray(sources, dtype=np.uint32)
    c = kernel.cheby_coeffs(K)
    s = cpg_stats()
    ptr = out.ctypes.data if isinstance(out, np.ndarray) else int(out)
    _check(L.lib().cpg_chebypower_batched_async(dg.handle, _f64p(c), K, _u32p(src), len(src), tile, ptr,
                                                ctypes.byref(s)))
    dg._pending.append(out)  # the copy into `out` is in flight: keep it alive until sync()
    return _to_stats(s, K)


def sync(g, device: int = 0):
    """Wait for every result copy in flight on the graph's device handle."""
    dg = _dev(g, device)
    _check(L.lib().cpg_graph_sync(dg.handle))
    dg._pending.clear()


def cheby_power_topk(g, kernel: Kernel, sources: Sequence[int], cheby_steps: int, k: int = 50, device: int = 0):
    """Top-k (ids, scores) per source ranked on the device by (score desc, id asc),
    the order of the reference's query output (tools/chebyprop.cpp:148-156)."""
    K = _steps(cheby_steps)
    dg = _dev(g, device)
    src = np.ascontiguousarray(sources, dtype=np.uint32)
    kk = min(int(k), dg.n)
    ids = np.empty((len(src), kk), dtype=np.uint32)
    vals = np.empty((len(src), kk))
    c = kernel.cheby_coeffs(K)
    s = cpg_stats()
    _check(L.lib().cpg_chebypower_topk(dg.handle, _f64p(c), K, _u32p(src), len(src), int(k), _u32p(ids),
                                       _f64p(vals), ctypes.byref(s)))
    return ids, vals, _to_stats(s, K)


def power_method(g, kernel: Kernel, source: int, n_steps: int, device: int = 0) -> Estimate:
    """PwMethod (solvers.cpp:87-121) on the GPU: sum_{k<N} zeta_k P^k e_source."""
    t0 = time.perf_counter()
    N = int(n_steps)
    if N < 1:
        raise ParameterError("power_method: n_steps must be >= 1")
    dg = _dev(g, device)
    if source < 0 or source >= dg.n:
        raise ParameterError(f"source node {source} out of range")
    zeta = kernel.taylor_coeffs(N - 1)
    out = np.empty(dg.n)
    s = cpg_stats()
    src = np.array([source], dtype=np.uint32)
    _check(L.lib().cpg_power_method(dg.handle, _f64p(zeta), N, _u32p(src), 1, out.ctypes.data, ctypes.byref(s)))
    st = _to_stats(s, N)
    st.iterations, st.algorithm, st.params = N, "pw", f"N={N}"
    st.push_work = (N - 1) * int(dg.info.nnz)
    st.wall_seconds = time.perf_counter() - t0
    return Estimate(out, st)


def ground_truth_steps(kernel: Kernel) -> int:
    """eval.cpp:39-50."""
    return int(L.lib().cpg_ground_truth_steps(kernel.family(), kernel.param))


def ground_truth(g, kernel: Kernel, source: int, device: int = 0) -> np.ndarray:
    """eval.cpp:52-59: PwMethod far past convergence, on the GPU."""
    return power_method(g, kernel, source, ground_truth_steps(kernel), device=device).values


def apply_walk(g, x, device: int = 0) -> np.ndarray:
    """y = A D^-1 x (graph.cpp:257-273) on the GPU."""
    dg = _dev(g, device)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (dg.n,):
        raise ParameterError("apply_walk: vector length mismatch")
    y = np.empty(dg.n)
    _check(L.lib().cpg_apply_walk(dg.handle, _f64p(x), _f64p(y)))
    return y


def general_gp_matrix(g, kernel: Kernel, a: float, columns, steps: int, tile: int = 64, device: int = 0):
    """z_j = D^-a f(P) D^a x_j with ChebyPower for every column (solvers.cpp:390-414).

    The D^{+-a} scalings are fused into the device seed/output kernels; columns
    run in tiles of ``tile`` through the batched step (tile=1: one at a time)."""
    K = _steps(steps)
    dg = _dev(g, device)
    cols = np.ascontiguousarray(np.atleast_2d(np.asarray(columns, dtype=np.float64)))
    if cols.shape[1] != dg.n:
        raise ParameterError("seed vector length mismatch")  # solvers.cpp:36-37
    c = kernel.cheby_coeffs(K)
    out = np.empty_like(cols)
    s = cpg_stats()
    _check(L.lib().cpg_general_gp(dg.handle, _f64p(c), K, float(a), _f64p(cols), cols.shape[0],
                                  max(1, min(int(tile), 64)), out.ctypes.data, ctypes.byref(s)))
    return list(out)


def general_gp_vector(g, kernel: Kernel, a: float, x, steps: int, device: int = 0) -> np.ndarray:
    """z = D^-a f(P) D^a x with ChebyPower (solvers.cpp:390-403)."""
    return general_gp_matrix(g, kernel, a, [x], steps, tile=1, device=device)[0]


# ---- synthetic inputs ----------------------------------------------------------------------
class DeviceCSR:
    """A generator-built CSR resident on one GPU (owned; freed on close)."""

    def __init__(self, off_ptr: int, nbr_ptr: int, n: int, nnz: int, device: int):
        self.offsets_ptr = off_ptr
        self.neighbors_ptr = nbr_ptr
        self.n = n
        self.nnz = nnz
        self.device = device

    def close(self):
        if self.offsets_ptr:
            L.lib().cpg_free_csr(ctypes.c_void_p(self.offsets_ptr), ctypes.c_void_p(self.neighbors_ptr), self.device)
            self.offsets_ptr = self.neighbors_ptr = 0

    def to_host(self):
        off = np.empty(self.n + 1, dtype=np.uint64)
        nbr = np.empty(self.nnz, dtype=np.uint32)
        _check(L.lib().cpg_csr_to_host(ctypes.c_void_p(self.offsets_ptr), ctypes.c_void_p(self.neighbors_ptr),
                                       self.n, self.nnz, self.device, _u64p(off), _u32p(nbr)), "csr_to_host")
        return off, nbr

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _gen_result(rc, off, nbr, n, nnz, device):
    _check(rc, "generator")
    if device < 0:
        o = np.ctypeslib.as_array(ctypes.cast(off, ctypes.POINTER(ctypes.c_uint64)), shape=(n.value + 1,)).copy()
        b = np.ctypeslib.as_array(ctypes.cast(nbr, ctypes.POINTER(ctypes.c_uint32)), shape=(nnz.value,)).copy()
        L.lib().cpg_free_csr(off, nbr, -1)
        return o, b
    return DeviceCSR(off.value, nbr.value, n.value, nnz.value, device)


def ingest_edges(pairs, device: int = 0):
    """Edge list -> CSR on the GPU with the reference loader's semantics (graph.cpp:113-171).

    Returns (DeviceCSR, original_ids) -- original_ids[i] is the label of compact id i."""
    pr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
    off, nbr = ctypes.c_void_p(), ctypes.c_void_p()
    n, nnz = ctypes.c_uint32(), ctypes.c_uint64()
    labels = np.empty(2 * len(pr) + 1, dtype=np.int64)
    i64p = ctypes.POINTER(ctypes.c_int64)
    _check(L.lib().cpg_ingest_edges(pr.ctypes.data_as(i64p), len(pr), device, ctypes.byref(off), ctypes.byref(nbr),
                                    ctypes.byref(n), ctypes.byref(nnz), labels.ctypes.data_as(i64p), len(labels)),
           "ingest")
    return DeviceCSR(off.value, nbr.value, n.value, nnz.value, device), labels[: n.value].copy()


def parse_edge_text(text, comment: str = "#", n_threads: int = 0) -> np.ndarray:
    """Edge-list text -> (m, 2) int64 label pairs with the reference loader's line rules
    (graph.cpp:126-151): natively parsed, multi-threaded; ParseError names the first bad line."""
    buf = text.encode() if isinstance(text, str) else bytes(text)
    cap = buf.count(b"\n") + 1
    pairs = np.empty((cap, 2), dtype=np.int64)
    got = ctypes.c_uint64()
    _check(L.lib().cpg_parse_edge_text(buf, len(buf), comment.encode()[:1] or b"#", pairs.ctypes.data, cap,
                                       ctypes.byref(got), int(n_threads)))
    return pairs[: got.value]


def load_edge_list(text, comment: str = "#", device: int = 0) -> Graph:
    """load_edge_list (graph.cpp:113-171): parse the text natively, intern / symmetrise /
    dedup on the GPU.  The graph carries ``original_ids`` (graph.hpp:45)."""
    pairs = parse_edge_text(text, comment)
    csr, labels = ingest_edges(pairs, device)
    off, nb = csr.to_host()
    csr.close()
    g = Graph(off, nb)
    g.original_ids = labels
    return g


def load_edge_list_file(path: str, device: int = 0, comment: str = "#") -> Graph:
    """load_edge_list_file (graph.cpp:173-177)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open graph file: {path}") from e
    return load_edge_list(data, comment, device)


def write_csr_cache(g: Graph, path: str) -> None:
    """write_csr_cache (graph.cpp:217-232): "CPGR", u32 1, n, m, offsets, neighbors."""
    off, nb = g.offsets(), g.neighbor_array()
    _check(L.lib().cpg_csr_cache_write(str(path).encode(), _u64p(off), _u32p(nb), len(off) - 1, len(nb)))


def read_csr_cache(path: str, validate: bool = True) -> Graph:
    """read_csr_cache (graph.cpp:234-255): header checks, then Graph::from_csr's validation."""
    p = str(path).encode()
    n, m = ctypes.c_uint64(), ctypes.c_uint64()
    _check(L.lib().cpg_csr_cache_info(p, ctypes.byref(n), ctypes.byref(m)))
    off = np.empty(n.value + 1, dtype=np.uint64)
    nb = np.empty(2 * m.value, dtype=np.uint32)
    _check(L.lib().cpg_csr_cache_read(p, _u64p(off), _u32p(nb), n.value, m.value))
    return Graph.from_csr(off, nb, validate=validate)


@dataclass
class ErrorReport:  # eval.hpp:15-20
    l1: float = 0.0
    l2: float = 0.0
    deg_norm_inf: float = 0.0
    argmax_node: int = 0


def _reports(arr) -> list:
    return [ErrorReport(r.l1, r.l2, r.deg_norm_inf, int(r.argmax_node)) for r in arr]


def measure(truth, estimate, g, device: int = 0) -> ErrorReport:
    """measure (eval.cpp:18-37) on the GPU; (s, n) stacks give a list of reports."""
    dg = _dev(g, device)
    t = np.ascontiguousarray(truth, dtype=np.float64)
    e = np.ascontiguousarray(estimate, dtype=np.float64)
    if t.shape != e.shape or t.shape[-1] != dg.n:
        raise ParameterError("measure: vector length mismatch")  # eval.cpp:21-22
    cols = 1 if t.ndim == 1 else t.shape[0]
    reps = (L.cpg_error_report * cols)()
    _check(L.lib().cpg_measure(dg.handle, t.ctypes.data, e.ctypes.data, cols, 0, reps))
    out = _reports(reps)
    return out[0] if t.ndim == 1 else out


def cheby_power_measure(g, kernel: Kernel, sources: Sequence[int], cheby_steps: int, truths, device: int = 0):
    """ChebyPower for every source, measured against truths[i] on the device (the eval
    harness's estimate + measure, tools/chebyprop.cpp:140-160); only the reports return."""
    K = _steps(cheby_steps)
    dg = _dev(g, device)
    src = np.ascontiguousarray(sources, dtype=np.uint32)
    tr = np.ascontiguousarray(truths, dtype=np.float64).reshape(len(src), -1)
    if tr.shape[1] != dg.n:
        raise ParameterError("measure: vector length mismatch")
    c = kernel.cheby_coeffs(K)
    reps = (L.cpg_error_report * max(1, len(src)))()
    s = cpg_stats()
    _check(L.lib().cpg_chebypower_measure(dg.handle, _f64p(c), K, _u32p(src), len(src), tr.ctypes.data, 0, reps,
                                          ctypes.byref(s)))
    return _reports(reps)[: len(src)], _to_stats(s, K)


@dataclass
class GroundTruth:  # eval.hpp:25-30
    values: np.ndarray
    kernel_descriptor: str = ""
    source: int = 0
    truncation: int = 0


def write_truth_cache(truth: GroundTruth, path: str) -> None:
    """write_truth_cache (eval.cpp:113-124)."""
    v = np.ascontiguousarray(truth.values, dtype=np.float64)
    _check(L.lib().cpg_truth_cache_write(str(path).encode(), truth.kernel_descriptor.encode(), int(truth.source),
                                         _f64p(v), len(v)))


def read_truth_cache(path: str) -> GroundTruth:
    """read_truth_cache (eval.cpp:126-145)."""
    p = str(path).encode()
    desc = ctypes.create_string_buffer(4096)
    src, n = ctypes.c_uint64(), ctypes.c_uint64()
    _check(L.lib().cpg_truth_cache_info(p, desc, len(desc), ctypes.byref(src), ctypes.byref(n)))
    v = np.empty(n.value)
    _check(L.lib().cpg_truth_cache_read(p, _f64p(v), n.value))
    return GroundTruth(v, desc.value.decode(), int(src.value), 0)


def _hash_of(g) -> int:
    if isinstance(g, Graph):
        if not g.structure_hash():
            g._hash = Graph.from_csr(g.offsets(), g.neighbor_array()).structure_hash()
        return g.structure_hash()
    return int(g.info.structure_hash)


def truth_cache_filename(g, kernel: Kernel, source: int) -> str:
    """truth_cache_filename (eval.cpp:147-156)."""
    out = ctypes.create_string_buffer(4096)
    _check(L.lib().cpg_truth_cache_filename(_hash_of(g), kernel.descriptor().encode(), int(source), out, len(out)))
    return out.value.decode()


def load_or_compute_truth(g, kernel: Kernel, source: int, cache_dir: str = "", device: int = 0):
    """load_or_compute_truth (eval.cpp:158-192): (GroundTruth, was_cached).  A cached file is
    used when its descriptor, source and length match; corrupt or stale entries (ParseError)
    are recomputed -- on the GPU (PwMethod, eval.cpp:52-59) -- and rewritten."""
    import os as _os

    dg = _dev(g, device)
    if source < 0 or source >= dg.n:
        raise ParameterError("load_or_compute_truth: source out of range")
    path = ""
    if cache_dir:
        path = _os.path.join(cache_dir, truth_cache_filename(g, kernel, source))
        if _os.path.exists(path):
            try:
                t = read_truth_cache(path)
                if t.kernel_descriptor == kernel.descriptor() and t.source == source and len(t.values) == dg.n:
                    t.truncation = ground_truth_steps(kernel)
                    return t, True
            except (ParseError, IoError):
                pass
    t = GroundTruth(ground_truth(g, kernel, source, device), kernel.descriptor(), int(source),
                    ground_truth_steps(kernel))
    if cache_dir:
        _os.makedirs(cache_dir, exist_ok=True)
        try:
            write_truth_cache(t, path)
        except IoError:
            pass  # eval.cpp:186-189: a cache that cannot be written is skipped
    return t, False


def gen_rmat(scale: int, n_samples: int, a=0.57, b=0.19, c=0.19, seed: int = 1, device: int = -1):
    """Seeded R-MAT, symmetrised/deduplicated/compacted.  device=-1: host (offsets, neighbors)."""
    off, nbr = ctypes.c_void_p(), ctypes.c_void_p()
    n, nnz = ctypes.c_uint32(), ctypes.c_uint64()
    rc = L.lib().cpg_gen_rmat(scale, n_samples, a, b, c, seed, device, ctypes.byref(off), ctypes.byref(nbr),
                              ctypes.byref(n), ctypes.byref(nnz))
    return _gen_result(rc, off, nbr, n, nnz, device)


def gen_chunglu(n_ids: int, n_samples: int, exponent: float, mean_degree: float, max_degree: int = 0,
                seed: int = 1, device: int = -1):
    """Seeded Chung-Lu with power-law expected degrees.  device=-1: host (offsets, neighbors)."""
    off, nbr = ctypes.c_void_p(), ctypes.c_void_p()
    n, nnz = ctypes.c_uint32(), ctypes.c_uint64()
    rc = L.lib().cpg_gen_chunglu(n_ids, n_samples, exponent, mean_degree, max_degree, seed, device,
                                 ctypes.byref(off), ctypes.byref(nbr), ctypes.byref(n), ctypes.byref(nnz))
    return _gen_result(rc, off, nbr, n, nnz, device)


def select_sources_uniform(n: int, count: int, seed: int) -> np.ndarray:
    """Seeded uniform sources without replacement: the reference's partial
    Fisher-Yates over SplitMix64 (eval.cpp:67-90, rng.hpp:13-27)."""
    if count > n:
        raise ParameterError("select_sources: count exceeds node count")
    M = (1 << 64) - 1
    state = seed & M
    picked: dict[int, int] = {}
    out = np.empty(count, dtype=np.uint32)
    for i in range(count):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        j = i + ((z * (n - i)) >> 64)
        vi, vj = picked.get(i, i), picked.get(j, j)
        picked[i], picked[j] = vj, vi
        out[i] = vj
    return out
