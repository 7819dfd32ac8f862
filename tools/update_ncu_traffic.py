"""Rebuild the batched entries of profiles/ncu_traffic.json (bench.py's roofline basis) from ncu
summaries written by profiles/ncu_summary.py:
    python tools/update_ncu_traffic.py <dir with ncu_c5_summary.txt, ncu_c4_summary.txt, ncu_c3b_summary.txt> <label>"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    ks, cur = [], None
    for line in open(path):
        if line.startswith("Kernel Name"):
            cur = {"name": line.split(None, 2)[2].strip()}
            ks.append(cur)
        elif cur is not None:
            p = line.split()
            if not p:
                continue
            try:
                cur[p[0]] = float(p[-1])
            except ValueError:
                pass
    return ks


def main():
    src, label = sys.argv[1], sys.argv[2]
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    t = json.load(open(path))
    for key, f in (("5:batched:16", "c5"), ("4:batched:64", "c4"), ("3:batched:64", "c3b")):
        fn = os.path.join(src, f"ncu_{f}_summary.txt")
        if not os.path.exists(fn):
            continue
        ks = parse(fn)
        if len(ks) < 2:
            continue
        old = t.get(key, {})
        ent = {"bytes": 0.0, "kernels": {}, "previous": old.get("previous")}
        for k in ks:
            m = re.search(r"(cheby_batch_\w+)<([^>]*)>", k["name"])
            name = f"{m.group(1)}<{m.group(2).replace(' ', '')}>"
            rd, wr = k["dram__bytes_read.sum"], k["dram__bytes_write.sum"]
            ent["kernels"][name] = {"read_GB": rd, "write_GB": wr, "ms": k["gpu__time_duration.sum"],
                                    "dram_pct": k["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
                                    "l2_hit_pct": k["lts__t_sector_hit_rate.pct"], "source": label}
            ent["bytes"] += (rd + wr) * 1e9
        t[key] = ent
        print(key, round(ent["bytes"] / 1e9, 2), "GB", {k: round(v["ms"], 2) for k, v in ent["kernels"].items()})
    json.dump(t, open(path, "w"), indent=2)


if __name__ == "__main__":
    main()
