"""Generate golden vectors from the UNMODIFIED reference library.

    python tests/golden/make_golden.py      (needs oracle/_ref/libchebyprop_ref.so,
                                             i.e. /root/reference present at build time)

Writes tests/golden/golden.npz: Chebyshev coefficients, truncation plans and
cheby_power score vectors (+ per-step residual sums) computed by the
reference's own code on small seeded graphs.  Committed; the tests read it on
machines without /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import HKPR, PPR, Port, Ref, RefGraph, edge_text  # noqa: E402


def graphs():
    gs = {
        "star": [[0, 1], [0, 2], [0, 3]],                      # tests/oracles.hpp:181-184
        "path3": [[0, 1], [1, 2]],                             # oracles.hpp:186-189
        "ring_chord_25_35_31": Port.ring_chord_pairs(25, 35, 31),   # test_solvers.cpp:156-165
        "ring_chord_200_300_1": Port.ring_chord_pairs(200, 300, 1),  # acceptance.cpp:139-157 (C4)
        "ring_chord_1000_1500_5": Port.ring_chord_pairs(1000, 1500, 5),
    }
    out = {}
    for name, pairs in gs.items():
        g = RefGraph.from_edge_text(edge_text(pairs))  # the reference loader, graph.cpp:113-171
        out[name] = g
    return out


def main():
    oracle.build()
    assert Ref.available(), "reference library not built"
    data = {}
    for fam, params in ((PPR, (0.2, 0.1, 0.02)), (HKPR, (5.0, 20.0, 40.0))):
        for p in params:
            tag = f"{'ppr' if fam == PPR else 'hkpr'}_{p:g}"
            data[f"coeffs/{tag}"] = Ref.cheby_coeffs(fam, p, 200)
            plans = []
            for eps in (1e-2, 1e-4, 1e-6, 1e-8, 5e-13):
                pl = Ref.plan_truncation(fam, p, eps)
                plans.append([pl.cheby_steps, pl.taylor_steps, pl.epsilon, pl.tail_bound])
            data[f"plans/{tag}"] = np.array(plans)
    for name, g in graphs().items():
        off, nb = g.csr()
        data[f"graph/{name}/offsets"] = off
        data[f"graph/{name}/neighbors"] = nb
        n = g.n
        sources = sorted({0, n // 2, n - 1})
        data[f"graph/{name}/sources"] = np.array(sources, dtype=np.uint32)
        for fam, p in ((PPR, 0.2), (HKPR, 5.0)):
            K = Ref.plan_truncation(fam, p, 1e-8).cheby_steps
            tag = f"{'ppr' if fam == PPR else 'hkpr'}"
            vals, masses = [], []
            for s in sources:
                v, m, st = g.cheby_power(fam, p, s, K)
                vals.append(v)
                masses.append(m)
            data[f"graph/{name}/{tag}/K"] = np.array(K)
            data[f"graph/{name}/{tag}/values"] = np.array(vals)
            data[f"graph/{name}/{tag}/mass"] = np.array(masses)
        x = Port.random_vector(n, 92, 0.0, 1.0)
        data[f"graph/{name}/walk_x"] = x
        data[f"graph/{name}/walk_y"] = g.apply_walk(x)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
