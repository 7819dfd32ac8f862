#!/usr/bin/env python
"""ChebyPower bench: GTEPS and queries/s on seeded synthetic graphs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

A "step" is one pass of the hot path over one batch of queries: every source
of the config (16 or 64) runs its K Chebyshev iterations.  The default workload
is config 5 (the 1.8B-edge R-MAT graph, 16 SSPPR sources as one 16-column tile
of the batched step; row-partitioned with per-chunk NCCL all-gathers when
launched on N GPUs).

value  = GTEPS = K * nnz * sources / t   (the reference's push_work / wall_seconds,
         solvers.cpp:214,223), device-resident inputs, CUDA events, max over ranks.
e2e    = same metric through the C-ABI call with HOST buffers: sources and
         coefficients H2D, every result vector D2H into pinned memory, inside the
         timed region.
roofline: the step kernel(s), one launch = one step of one source tile (or query
         group); achieved = min(algorithmic bytes per launch (12*nnz +
         8*(n+1) + 32*n single-source, nnz*(4+8B) + 8*(n+1) + 32*n*B batched), the
         ncu-measured DRAM bytes of that launch) / mean CUDA-event launch duration
         measured here; frac_model keeps the model-only fraction.  Where the batched step is
         two kernels (hub-piece kernel + plain-row kernel, graphs of >= 8 M edges) the line is the
         DOMINANT kernel's: its own ncu DRAM bytes over its own live CUDA-event time
         (cpg_last_split_profile); `kernels` holds both, `step` the step-level numbers.  The
         timed call runs with the sparse early steps off, so every launch is a full step.
cpu_baseline: the reference's own cheby_power (oracle/_ref, compiled from
         /root/reference sources) on all host cores (bounded sample; whole queries
         where they fit, else the SpMV of a query, extrapolated), plus one-thread
         latency (threads_1).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PPR, HKPR = 0, 1

# Synthetic stand-ins for the paper's datasets (BASELINE.json configs).
CONFIGS = {
    1: dict(name="rmat-s16-ef8 ppr", gen="rmat", scale=16, samples=8 << 16, seed=1,
            family=PPR, param=0.2, eps=1e-8, sources=16, mode="batched"),
    2: dict(name="chunglu-dblp-size hkpr", gen="chunglu", n_ids=317_080, samples=1_050_000, exponent=2.5,
            mean=6.6, cap=0, seed=2, family=HKPR, param=5.0, eps=1e-8, sources=64, mode="batched"),
    3: dict(name="chunglu-livejournal-size ppr", gen="chunglu", n_ids=4_846_609, samples=43_200_000,
            exponent=2.3, mean=17.8, cap=20_000, seed=3, family=PPR, param=0.2, eps=1e-8, sources=64,
            mode="single"),
    4: dict(name="chunglu-orkut-size hkpr batched", gen="chunglu", n_ids=3_072_626, samples=121_000_000,
            exponent=2.1, mean=76.0, cap=33_000, seed=4, family=HKPR, param=5.0, eps=1e-8, sources=64,
            mode="batched"),
    5: dict(name="rmat-friendster-size ppr", gen="rmat", scale=27, samples=1_840_000_000, seed=5,
            family=PPR, param=0.2, eps=1e-8, sources=16, mode="batched", tile=16),
}
# Configs 1, 2, 4, 5 run their sources through the batched step (one tile of all of them; the
# faster path for a multi-source workload: DESIGN.md 6); config 3 names the single-source SpMV
# path.  --mode overrides either way.
# Headline: config 5, the 1.8B-edge graph the metric is quoted on at 1/2/4/8 B200;
# its 16 sources run as one 16-column tile through the batched step.
DEFAULT_CONFIG = 5


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_device_csr(cfg, device):
    import paper_2412_10789_b200 as P

    if cfg["gen"] == "rmat":
        return P.gen_rmat(cfg["scale"], cfg["samples"], seed=cfg["seed"], device=device)
    return P.gen_chunglu(cfg["n_ids"], cfg["samples"], cfg["exponent"], cfg["mean"], cfg["cap"],
                         seed=cfg["seed"], device=device)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[2:6]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def load_traffic(cfg_index, mode, tile):
    """DRAM bytes per step of this workload's step kernel(s) from a committed ncu capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(f"{cfg_index}:{mode}:{tile}", {}).get("bytes")
    except Exception:
        return None


def load_traffic_kernels(cfg_index, mode, tile):
    """Per-kernel DRAM bytes per step ({name: bytes, l2_hit_pct}) of the committed ncu capture, or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        ks = t.get(f"{cfg_index}:{mode}:{tile}", {}).get("kernels", {})
        return {k: {"bytes": (v["read_GB"] + v["write_GB"]) * 1e9, "l2_hit_pct": v.get("l2_hit_pct"),
                    "ncu_ms": v.get("ms")} for k, v in ks.items()}
    except Exception:
        return {}


def load_gather_ceiling():
    """Measured rate of random 8-B gathers from an L2-resident table (tools/gather_l2.cu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "gather", "gather_l2_c3.json")) as f:
            rows = [json.loads(x) for x in f if x.startswith("{")]
        return max(r["G_gathers_per_s"] for r in rows if r["variant"].startswith("ldg_U")) * 1e9
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _host_threads(n):
    """All host threads, capped so the per-thread iterate buffers fit in free RAM."""
    threads = os.cpu_count() or 1
    try:
        import psutil

        free = psutil.virtual_memory().available
        threads = max(1, min(threads, int(0.5 * free // max(1, 2 * 8 * n))))
    except Exception:
        pass
    return threads


_REF_GRAPHS = {}


def _ref_graph(off, nb, threads):
    """The reference Graph for this CSR (oracle/_ref, built once per array pair), or None when
    the reference library is absent or the host lacks room for its copy of the graph beside
    the per-thread vectors.  Graphs above BIG_NNZ are adopted without from_csr's O(nnz log d)
    symmetry check (~6 min single-threaded at config 5; ref_shim.cpp: ref_graph_adopt_csr,
    pinned equal to from_csr in tests/test_oracle_pin.py); the CSR comes from the generator,
    whose output tests/test_host_api.py checks against from_csr."""
    import oracle

    key = (id(off), id(nb))
    if key in _REF_GRAPHS:
        return _REF_GRAPHS[key]
    g = None
    if oracle.Ref.available():
        n, nnz = len(off) - 1, len(nb)
        need = 4 * nnz + 20 * (n + 1) + threads * 24 * n
        try:
            import psutil

            room = psutil.virtual_memory().available > 1.25 * need
        except Exception:
            room = True
        if room:
            g = oracle.RefGraph.adopt_csr(off, nb) if nnz > BIG_NNZ else oracle.RefGraph.from_csr(off, nb)
    _REF_GRAPHS.clear()
    _REF_GRAPHS[key] = g
    return g


BIG_NNZ = 300_000_000
REF_RATE = 0.2e9  # edge visits/s of one reference thread under full-socket contention (measured 0.1-0.35)


def cpu_sample(cfg, off, nb, sources, K, budget_s=20.0, threads=None):
    """One throughput sample of the reference's CPU ChebyPower on all host threads.

    When a round of `threads` concurrent whole queries fits the budget (configs 1-2
    at the default budgets), whole cheby_power queries (solvers.cpp:236-239) of the
    reference library (oracle/_ref, compiled from /root/reference) run on a worker
    pool like the reference bench (tools/chebyprop.cpp:305-334); GTEPS =
    K*nnz*queries / wall.  Otherwise the sample is the steady-state SpMV of the
    query: every thread runs the reference's apply_walk_from_subset
    (graph.cpp:275-288, apply_walk_into's scatter loop) over a contiguous run of
    rows scattering into a full-length vector, and queries/s is EXTRAPOLATED as
    GTEPS / (K*nnz) (the dense passes are ~2% of a query).  Without
    the reference library the bit-exact restatement in oracle/ runs instead
    ("kind": "port").  The checker libraries are used only here, as the timed CPU
    baseline."""
    import oracle

    n, nnz = len(off) - 1, len(nb)
    threads = threads or _host_threads(n)
    g = _ref_graph(off, nb, threads)
    kind = "reference" if g is not None else "port"
    if K * nnz / REF_RATE > budget_s:  # a whole query per thread does not fit: SpMV sample
        per = int(max(20e6, min(400e6, budget_s * REF_RATE / 2)))  # edges per thread
        if g is not None:
            wall, edges = g.apply_walk_subset_pool(threads, per)
            what = ("the reference's own apply_walk_from_subset (graph.cpp:275-288; apply_walk_into's scatter "
                    "loop) from oracle/_ref")
        else:
            wall, edges = oracle.Port.apply_walk_pool(off, nb, threads, per)
            what = "the reference's dense apply_walk (oracle restatement)"
        gteps = edges / wall / 1e9
        return {"value": gteps, "unit": "GTEPS", "cores": threads, "kind": kind,
                "queries_per_s": gteps * 1e9 / (K * nnz), "whole_queries": False,
                "sample": f"{threads} threads x ~{per / 1e6:.0f}M edges (one contiguous row run each, scattering "
                          f"into a full-length vector) of {what}, in {wall:.2f}s; queries/s EXTRAPOLATED as "
                          f"GTEPS/(K*nnz): a whole query takes ~{K * nnz / REF_RATE / 60:.0f} min per core",
                "cpu_model": _cpu_model()}
    coeffs = oracle.Port.cheby_coeffs(cfg["family"], cfg["param"], K)
    done, wall = 0, 0.0
    while wall < budget_s / 2 and done < len(sources) * 4:
        batch = [int(sources[(done + i) % len(sources)]) for i in range(threads)]
        t = time.perf_counter()
        if g is not None:
            g.cheby_power_pool(cfg["family"], cfg["param"], batch, K, threads, keep=False)
        else:
            oracle.Port.cheby_power_pool(off, nb, coeffs, K, batch, threads, keep=False)
        wall += time.perf_counter() - t
        done += len(batch)
    return {"value": K * nnz * done / wall / 1e9, "unit": "GTEPS", "cores": threads, "kind": kind,
            "queries_per_s": done / wall, "whole_queries": True,
            "sample": f"{done} whole cheby_power queries x K={K} on {threads} threads ({wall:.2f}s; graph setup "
                      f"excluded)", "cpu_model": _cpu_model()}


def cpu_latency_1thread(cfg, off, nb, sources, K, limit_s=60.0):
    """BASELINE.md 4 latency arm: one query at a time on ONE thread.  A whole reference
    cheby_power query (its own wall_seconds) when it is expected to take <= limit_s;
    else one thread's apply_walk_from_subset sample, extrapolated to K*nnz edges."""
    import oracle

    n, nnz = len(off) - 1, len(nb)
    g = _ref_graph(off, nb, 1)
    kind = "reference" if g is not None else "port"
    if K * nnz / (1.5 * REF_RATE) <= limit_s:
        s = int(sources[0])
        if g is not None:
            _, wall = g.cheby_power_pool(cfg["family"], cfg["param"], [s], K, 1, keep=False)  # its wall_seconds
        else:
            coeffs = oracle.Port.cheby_coeffs(cfg["family"], cfg["param"], K)
            t = time.perf_counter()
            oracle.Port.cheby_power_pool(off, nb, coeffs, K, [s], 1, keep=False)
            wall = time.perf_counter() - t
        return {"query_s": wall, "gteps": K * nnz / wall / 1e9, "kind": kind, "cores": 1,
                "sample": f"one whole cheby_power query (source {s}, K={K}) on one thread"}
    per = int(min(400e6, max(20e6, 5 * 1.5 * REF_RATE)))
    if g is not None:
        wall, edges = g.apply_walk_subset_pool(1, per)
    else:
        wall, edges = oracle.Port.apply_walk_pool(off, nb, 1, per)
    rate = edges / wall
    return {"query_s": K * nnz / rate, "gteps": rate / 1e9, "kind": kind, "cores": 1, "extrapolated": True,
            "sample": f"one thread x {edges / 1e6:.0f}M edges of apply_walk_from_subset in {wall:.2f}s; "
                      f"query time EXTRAPOLATED to K*nnz = {K * nnz / 1e9:.1f}G edge visits"}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def make_host_graph_port(cfg):
    """The config's CSR built on the host by the generator restatement in oracle/
    (graphgen_port.c, pinned equal to the product's generator): no product library."""
    import oracle

    if cfg["gen"] == "rmat":
        return oracle.Port.gen_rmat(cfg["scale"], cfg["samples"], seed=cfg["seed"])
    return oracle.Port.gen_chunglu(cfg["n_ids"], cfg["samples"], cfg["exponent"], cfg["mean"], cfg["cap"],
                                   seed=cfg["seed"])


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU ChebyPower on all host threads.

    Same config, metric and unit as our arm; each step is one bounded throughput
    sample (cpu_sample), plus one single-thread latency measurement
    (cpu_latency_1thread).  Only oracle/ libraries are loaded in this process: the
    input graph comes from the generator restatement (oracle/graphgen_port.c),
    K from the reference's plan_truncation and the sources from its
    select_sources (oracle/_ref), all outside the timed samples.  Rank 0 alone
    runs (the CPU baseline does not shard); other ranks exit."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    t0 = time.perf_counter()
    off, nb = make_host_graph_port(cfg)
    t_gen = time.perf_counter() - t0
    n = len(off) - 1
    lib = oracle.Ref if oracle.Ref.available() else oracle.Port
    K = lib.plan_truncation(cfg["family"], cfg["param"], cfg["eps"]).cheby_steps
    sources = oracle.Port.select_sources_uniform(n, cfg["sources"], 1)  # eval.cpp:67-90 restated, pinned
    # per-step budget: the whole --steps/--warmup run stays within a few minutes
    budget = args.cpu_budget if args.cpu_budget_set else max(2.0, 120.0 / max(1, args.steps + args.warmup))
    samples = []
    t0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        r = cpu_sample(cfg, off, nb, sources, K, budget_s=budget)
        if i >= args.warmup:
            samples.append(r)
    t_samples = time.perf_counter() - t0
    lat = cpu_latency_1thread(cfg, off, nb, sources, K)
    gteps = float(np.median([r["value"] for r in samples]))
    qps = float(np.median([r["queries_per_s"] for r in samples]))
    last = samples[-1]
    line = {"metric": METRIC, "value": gteps, "unit": "GTEPS", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generator restatement, oracle/graphgen_port.c)",
            "queries_per_s": qps,
            "config": {"workload": cfg["name"], "config_index": args.config, "n": n, "nnz": len(nb), "K": K,
                       "sources_per_step": len(sources), "mode": cfg["mode"],
                       "tile": int(cfg.get("tile", min(64, len(sources)))) if cfg["mode"] == "batched" else 1},
            "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": last["cores"], "kind": last["kind"],
                             "sample": last["sample"], "whole_queries": last["whole_queries"],
                             "cpu_model": last["cpu_model"], "threads_1": lat},
            "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": {"generate": t_gen, "samples": t_samples},
            # the reference arm maps only oracle/ libraries (checked, not assumed)
            "product_library_loaded": "paper_2412_10789_b200" in sys.modules}
    emit(line)


METRIC = "ChebyPower GTEPS (K*nnz*sources/s) on the config graph; queries/s and % HBM roofline alongside"


# The JSON line is the only thing on stdout: native libraries print to fd 1 on their own
# (NCCL's "NCCL version ..." banner at communicator init), so fd 1 is pointed at stderr for
# the whole run and the line goes to a saved copy of the original stdout.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    print(json.dumps(line), file=out, flush=True)


def main():
    _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default=None, choices=["single", "batched"], help="override the config's path")
    ap.add_argument("--tile", type=int, default=None, help="sources per batched tile (1..64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="N=1: run the row-partitioned multi-GPU path with one rank (NCCL communicator, "
                         "chunked all-gathers) to measure its overhead on one GPU")
    ap.add_argument("--fused-allgather", action="store_true",
                    help="N>1 batched: epilogue stores into every rank's replica (NCCL symmetric windows) "
                         "instead of the chunked NCCL all-gather")
    ap.add_argument("--cpu-budget", type=float, default=None,
                    help="seconds per CPU baseline sample (default: 20 for our arm's cpu_baseline leg; "
                         "the reference arm splits ~2 min over its steps)")
    ap.add_argument("--sync-e2e", action="store_true",
                    help="e2e through the synchronous cpg_chebypower_batched (no cross-step copy overlap)")
    args = ap.parse_args()
    args.cpu_budget_set = args.cpu_budget is not None
    if args.cpu_budget is None:
        args.cpu_budget = 20.0
    cfg = dict(CONFIGS[args.config])
    if args.mode:
        cfg["mode"] = args.mode
    if args.tile:
        cfg["tile"] = args.tile
    if args.impl == "reference":
        return run_reference(args, cfg)
    run_ours(args, cfg)


def run_ours(args, cfg):
    import torch

    import paper_2412_10789_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = local
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    kernel = P.Kernel.ppr(cfg["param"]) if cfg["family"] == PPR else P.Kernel.hkpr(cfg["param"])
    K = P.plan_truncation(kernel, cfg["eps"]).cheby_steps
    coeffs = kernel.cheby_coeffs(K)

    t0 = time.perf_counter()
    csr = make_device_csr(cfg, dev)
    n, nnz = csr.n, csr.nnz
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    if args.fused_allgather:
        os.environ["CPG_P2P"] = "1"
    if world == 1 and not args.sharded:
        dg = P.DeviceGraph.from_device(csr)
    elif world == 1:  # one-rank sharded path (its own NCCL communicator)
        dg = P.DeviceGraph.sharded(csr.offsets_ptr, csr.neighbors_ptr, n, nnz, True, dev, 0, 1, P.nccl_unique_id())
    else:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(P.nccl_unique_id()), dtype=torch.uint8))
        pg.broadcast(uid, 0)
        dg = P.DeviceGraph.sharded(csr.offsets_ptr, csr.neighbors_ptr, n, nnz, True, dev, rank, world,
                                   bytes(uid.cpu().numpy()))
    torch.cuda.synchronize()
    t_up = time.perf_counter() - t0
    log(f"[bench] cfg{args.config} n={n} nnz={nnz} K={K} gen {t_gen:.1f}s upload {t_up:.1f}s "
        f"hubs={dg.info.n_hubs} items={dg.info.n_items} maxdeg={dg.info.max_degree}")

    sources = P.select_sources_uniform(n, cfg["sources"], 1)
    batched = cfg["mode"] == "batched"
    tile = int(cfg.get("tile", min(64, len(sources))))
    L = P._lib.lib()
    import ctypes

    src_np = np.ascontiguousarray(sources, dtype=np.uint32)
    c_np = np.ascontiguousarray(coeffs)
    d_out = torch.empty((len(sources), n), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    stats = P._lib.cpg_stats()

    def step_device():
        if batched:
            rc = L.cpg_chebypower_batched_device(dg.handle, P._f64p(c_np), K, P._u32p(src_np), len(src_np), tile,
                                                 ctypes.c_void_p(d_out.data_ptr()), ctypes.c_void_p(stream.cuda_stream),
                                                 None)
        else:
            rc = L.cpg_chebypower_device(dg.handle, P._f64p(c_np), K, P._u32p(src_np), len(src_np),
                                         ctypes.c_void_p(d_out.data_ptr()), ctypes.c_void_p(stream.cuda_stream), None)
        P._check(rc, "step")

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if pg is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    # ---- value: device-resident, K steps timed with CUDA events -------------------------
    for _ in range(args.warmup):
        step_device()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step_device()
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms / args.steps
    queries = len(sources) * args.steps
    gteps = K * nnz * queries / (ms / 1e3) / 1e9

    # ---- roofline: per-launch step-kernel time (events bracket each launch) ----------------
    # The roofline characterises the full step kernel: the sparse early steps (DESIGN.md
    # 4.7, which gather only the nonzero rows of w_{k-1}) are switched off for this call,
    # so every timed launch is a full-support step.  `value` keeps them on.
    sparse_env = os.environ.get("CPG_SPARSE_STEPS")
    os.environ["CPG_SPARSE_STEPS"] = "0"
    L.cpg_set_profiling(1)
    s = P._lib.cpg_stats()
    if batched:
        P._check(L.cpg_chebypower_batched(dg.handle, P._f64p(c_np), K, P._u32p(src_np), len(src_np), tile, None,
                                          ctypes.byref(s)))
    else:
        P._check(L.cpg_chebypower(dg.handle, P._f64p(c_np), K, P._u32p(src_np), len(src_np), None, ctypes.byref(s)))
    L.cpg_set_profiling(0)
    # split batched step (hub-piece kernel + plain-row kernel): each kernel's own mean time
    sp_pieces, sp_rows, sp_steps = ctypes.c_double(0.0), ctypes.c_double(0.0), ctypes.c_uint32(0)
    P._check(L.cpg_last_split_profile(dg.handle, ctypes.byref(sp_pieces), ctypes.byref(sp_rows), ctypes.byref(sp_steps)))
    if sparse_env is None:
        del os.environ["CPG_SPARSE_STEPS"]
    else:
        os.environ["CPG_SPARSE_STEPS"] = sparse_env
    launches_per_step = int(s.launches)  # kernels the library launched for one step (its own count)
    # one timed launch = one step of a source tile (batched) or of a query group (single-source:
    # several queries per launch on small graphs), so scale the per-step bytes by the steps it ran
    units = (-(-len(sources) // tile) if batched else len(sources)) * K
    steps_per_launch = units / max(1, s.step_launches)
    bytes_launch = dg.bytes_per_step(tile if batched else 1) * steps_per_launch
    per_launch_ms = max_over_ranks(s.step_ms / max(1, s.step_launches))
    peak, peak_kind = load_peaks()
    # Roofline basis: the algorithmic bytes of SURVEY.md 8d, capped at the DRAM bytes the
    # step's kernels actually move (ncu dram__bytes_read+write of this workload, committed in
    # profiles/ncu_traffic.json).  The batched model charges every gathered row to HBM, but
    # 36-40% of them hit L2 (config 5), so the model exceeds DRAM traffic and its "fraction"
    # can pass 1; there the DRAM bytes are the honest numerator.  Single-source moves MORE
    # DRAM bytes than the model (32-B sector over-fetch of 8-B gathers): there the model is
    # the useful-byte numerator.  frac_model keeps the model fraction either way.
    traffic_step = (load_traffic(args.config, cfg["mode"], tile if batched else 1)
                    if world == 1 and not args.sharded else None)
    traffic_launch = traffic_step * steps_per_launch if traffic_step else None
    basis_bytes = min(bytes_launch, traffic_launch) if traffic_launch else bytes_launch
    basis = "dram" if traffic_launch and traffic_launch < bytes_launch else "model"
    achieved = basis_bytes / (per_launch_ms / 1e3) / 1e9
    achieved_model = bytes_launch / (per_launch_ms / 1e3) / 1e9
    step_share = s.step_ms / max(1e-9, s.device_ms)
    # Dominant kernel of a split batched step: the roofline line is that kernel's (its DRAM bytes from
    # the committed ncu capture over its own live CUDA-event time); the step-level numbers stay beside it.
    split_kernels = None
    if batched and sp_steps.value and world == 1 and not args.sharded:
        tk = load_traffic_kernels(args.config, cfg["mode"], tile)
        split_kernels = {}
        for name, live_ms in (("cheby_batch_pieces_kernel", sp_pieces.value), ("cheby_batch_rows_kernel", sp_rows.value)):
            ent = next((v for k, v in tk.items() if k.startswith(name)), None)
            split_kernels[name] = {"launch_ms": live_ms, "share_of_step": live_ms / max(1e-9, sp_pieces.value + sp_rows.value),
                                   "traffic": ent["bytes"] if ent else None,
                                   "achieved": ent["bytes"] / (live_ms / 1e3) / 1e9 if ent and live_ms else None,
                                   "frac": ent["bytes"] / (live_ms / 1e3) / 1e9 / peak if ent and live_ms else None,
                                   "l2_hit_pct": ent["l2_hit_pct"] if ent else None}

    # ---- e2e: host buffers through the C-ABI call -------------------------------------------
    # Two pinned result buffers, alternating: a caller keeps result i while query i+1 runs.
    # Row-partitioned runs gather the result onto every rank; rank 0 alone reads it back.
    host_out = rank == 0
    outs = [torch.empty((len(sources), n) if host_out else (1, 1), dtype=torch.float64, pin_memory=True).numpy()
            for _ in range(2 if batched else 1)]

    def step_host(i, pipelined, last=True):
        st = P._lib.cpg_stats()
        out_np = outs[i % len(outs)]
        if not host_out:  # same steps and result all-gather (a collective), device output
            step_device()
            return st
        if batched and pipelined:  # the result copy overlaps the next step (cpg_graph_sync at the end);
            # without stats the call returns once queued, so the next query is enqueued while this one runs
            P._check(L.cpg_chebypower_batched_async(dg.handle, P._f64p(c_np), K, P._u32p(src_np), len(src_np),
                                                    tile, out_np.ctypes.data, ctypes.byref(st) if last else None))
        elif batched:
            P._check(L.cpg_chebypower_batched(dg.handle, P._f64p(c_np), K, P._u32p(src_np), len(src_np), tile,
                                              out_np.ctypes.data, ctypes.byref(st)))
        else:  # single-source calls overlap their per-group copies internally
            P._check(L.cpg_chebypower(dg.handle, P._f64p(c_np), K, P._u32p(src_np), len(src_np), out_np.ctypes.data,
                                      ctypes.byref(st)))
        return st

    for i in range(2):
        step_host(i, False)
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    t = time.perf_counter()
    for i in range(args.steps):
        st = step_host(i, not args.sync_e2e, last=i == args.steps - 1)
    P._check(L.cpg_graph_sync(dg.handle))  # the last step's result has landed in pinned memory
    wall_e2e = time.perf_counter() - t
    out_np = outs[(args.steps - 1) % len(outs)]
    e3.record(stream)
    barrier()
    wall_e2e = max_over_ranks(wall_e2e)
    e2e_gteps = K * nnz * queries / wall_e2e / 1e9
    mass_err = st.mass_err_max

    # ---- parity spot check of the timed outputs against the device-resident run -----
    same = bool(np.array_equal(out_np[0], d_out[0].cpu().numpy())) if host_out else None

    # ---- CPU baseline (rank 0, N = 1 only) ----------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        off, nb = csr.to_host()
        cpu = cpu_sample(cfg, off, nb, sources, K, budget_s=args.cpu_budget)
        cpu["threads_1"] = cpu_latency_1thread(cfg, off, nb, sources, K)
    csr.close()

    # Single-source: random 8-B gathers bound the step.  Report the step's gather
    # rate beside the measured ceiling of the gather alone (tools/gather_l2.cu, 192-200 G/s).
    gather_ceiling = {}
    if not batched:
        rate = steps_per_launch * (nnz / world) / (per_launch_ms / 1e3)
        ceil = load_gather_ceiling()
        gather_ceiling = {"gathers_per_s": rate, "gather_ceiling_per_s": ceil,
                          "frac_gather_ceiling": rate / ceil if ceil else None,
                          "gather_ceiling_source": "profiles/r02/gather/gather_l2_c3.json (ldg_U16_occ4)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator; stand-in for the paper's SNAP dataset)",
            "queries_per_s": queries / (ms / 1e3),
            "config": {"workload": cfg["name"], "config_index": args.config, "n": n, "nnz": nnz, "K": K,
                       "sources_per_step": len(sources), "mode": cfg["mode"],
                       "tile": tile if batched else 1,
                       "parallelism": (f"row-partition x{world}" if world > 1 or args.sharded else "1 GPU"),
                       "allgather": (("fused NVLink stores" if dg.info.fused_allgather else
                                      f"NCCL, {dg.info.chunks} chunks overlapped")
                                     if world > 1 or args.sharded else None),
                       "l2": "inputs larger than L2 (index stream 4*nnz bytes per step, re-read every step)",
                       "sparse_early_steps": dg.sparse_early_steps(tile if batched else 1, K)},
            "roofline": {"bound": "hbm", "timed": "every step full-support (sparse early steps off for this call)", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "basis": basis,
                         "frac_model": achieved_model / peak, "achieved_model": achieved_model,
                         # the committed ncu capture is of the one-GPU step; a rank's share differs
                         "traffic": traffic_launch,
                         "traffic_source": "profiles/ncu_traffic.json (ncu --set full, DRAM bytes per step x "
                                           "steps per launch)",
                         "kernel": (("cheby_batch_pieces_kernel (hub pieces) + cheby_batch_rows_kernel, timed as one "
                                     "step" if nnz // world >= (8 << 20) else "cheby_batch_kernel")
                                    if batched else "cheby_step_kernel"),
                         "bytes_per_launch": bytes_launch, "launch_ms": per_launch_ms, "steps_per_launch": steps_per_launch,
                         "step_share_of_device_time": step_share, **gather_ceiling},
            "e2e": {"value": e2e_gteps, "unit": "GTEPS",
                    "h2d_bytes_per_step": int(src_np.nbytes + c_np.nbytes),
                    "d2h_bytes_per_step": int(len(sources) * n * 8), "queries_per_s": queries / wall_e2e,
                    "d2h_ranks": "rank 0 (the result is all-gathered onto every rank)" if world > 1 else "rank 0",
                    "api": (("cpg_chebypower_batched" if args.sync_e2e else
                             "cpg_chebypower_batched_async (result D2H of step i overlaps step i+1, step i+1 "
                             "is enqueued while step i runs; cpg_graph_sync before the clock stops)")
                            if batched else "cpg_chebypower"),
                    "host_out": "pinned, two buffers alternating" if batched else "pinned"},
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
            "mass_err_max": mass_err,
            "e2e_matches_device_run": same,
            "setup_s": {"generate": t_gen, "upload_relabel": t_up},
        }
        if split_kernels and all(v["frac"] for v in split_kernels.values()):
            # the longer of the two kernels is the dominant one: its DRAM-byte fraction is `frac`; the
            # step-level fraction (both kernels as one launch) moves to `step`
            r = line["roofline"]
            dom = max(split_kernels, key=lambda k: split_kernels[k]["launch_ms"])
            r["step"] = {"achieved": r["achieved"], "frac": r["frac"], "basis": r["basis"], "traffic": r["traffic"],
                         "launch_ms": r["launch_ms"], "kernel": r["kernel"]}
            r.update({"kernel": dom + " (dominant kernel of the split step: %.0f%% of its time)"
                                % (100 * split_kernels[dom]["share_of_step"]),
                      "achieved": split_kernels[dom]["achieved"], "frac": split_kernels[dom]["frac"], "basis": "dram",
                      "traffic": split_kernels[dom]["traffic"], "launch_ms": split_kernels[dom]["launch_ms"],
                      "kernels": split_kernels})
        if cpu is not None:
            line["cpu_baseline"] = cpu
        emit(line)
    dg.close()
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
