"""Every bench source of the large configs against the pinned pull oracle (GPU box).

tests/test_gpu_fullsize.py checks the first 4 / 2 / 2 sources of configs 3 / 4 / 5 inside the
test budget; this one-off run checks ALL of them on the bench's own paths (config 3:
single-source and 64-column batched; config 4: 64-column batched; config 5: the headline
16-column batched tile and single-source), against oracle.Port.cheby_power_pull, which
tests/test_oracle_pin.py pins bit-for-bit to the unmodified reference library.

    python tools/parity_all_sources.py [configs...]  -> gpurun_out/parity_all_sources.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2412_10789_b200 as P  # noqa: E402
from oracle import Port, parity  # noqa: E402

PPR = 0


def main(cfgs):
    out = []
    path = os.path.join(ROOT, "gpurun_out", "parity_all_sources.json")
    for ci in cfgs:
        cfg = bench.CONFIGS[ci]
        csr = bench.make_device_csr(cfg, 0)
        off, nb = csr.to_host()
        dg = P.DeviceGraph.from_device(csr)
        csr.close()
        k = P.Kernel.ppr(cfg["param"]) if cfg["family"] == PPR else P.Kernel.hkpr(cfg["param"])
        K = P.plan_truncation(k, cfg["eps"]).cheby_steps
        c = k.cheby_coeffs(K)
        src = P.select_sources_uniform(dg.n, cfg["sources"], 1)
        tile = int(cfg.get("tile", 64))
        paths = {"batched%d" % tile: dict(batched=True, tile=tile)}
        if ci in (3, 5):
            paths["single"] = dict(batched=False)
        group = 4 if ci == 5 else 16
        for name, kw in paths.items():
            t = time.perf_counter()
            got, st = P.cheby_power_many(dg, k, src, K, **kw)
            t_gpu = time.perf_counter() - t
            worst = {"max_abs": 0.0, "l1": 0.0, "topk_equal": True}
            for g0 in range(0, len(src), group):
                want = Port.cheby_power_pull(off, nb, c, K, src[g0:g0 + group])
                for j in range(want.shape[0]):
                    p = parity(got[g0 + j], want[j], 100)
                    out.append({"config": ci, "path": name, "source": int(src[g0 + j]), **p,
                                "sum_minus_sum_c": float(got[g0 + j].sum() - c.sum())})
                    worst["max_abs"] = max(worst["max_abs"], p["max_abs"])
                    worst["l1"] = max(worst["l1"], p["l1"])
                    worst["topk_equal"] = worst["topk_equal"] and p["topk_equal"]
                del want
                with open(path, "w") as f:
                    json.dump(out, f, indent=1)
            print(f"config {ci} {name}: {len(src)} sources, GPU {t_gpu:.1f}s, worst {worst}, "
                  f"mass_err {st.mass_err_max:.2e}", flush=True)
            del got
        dg.close()
    bad = [r for r in out if r["max_abs"] > 1e-12 or r["l1"] > 1e-10 or not r["topk_equal"]]
    print(f"{len(out)} vectors, {len(bad)} outside max-abs 1e-12 / L1 1e-10 / exact top-100")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main([int(a) for a in sys.argv[1:]] or [3, 4, 5]))
