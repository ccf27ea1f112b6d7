"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes per kernel name).

  python scripts/launch_summary.py <launches.csv> [--traffic out.json]

--traffic writes the mean DRAM bytes per launch (read + write) of each kernel class that
bench.py reports (gemm, K1, K2, K3) plus the classes' shares of the summed device time."""
import collections
import csv
import json
import sys

path = sys.argv[1]
lines = [ln for ln in open(path) if not ln.startswith("==")]
rows = list(csv.DictReader(lines))
agg = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"].split("(")[0][-70:]
    agg.setdefault(k, collections.defaultdict(list))[r["Metric Name"]].append(
        (r["Grid Size"], float(r["Metric Value"].replace(",", ""))))
for k, d in agg.items():
    t = d.get("gpu__time_duration.sum", [])
    print(f"{k:72s} n={len(t):4d}", end="")
    for m, v in d.items():
        vals = [x for _, x in v]
        print(f" {m.split('.')[0].split('__')[1]}: mean {sum(vals) / len(vals):.4g} max {max(vals):.4g}", end="")
    print()


def klass(name):
    if "paged_attn" in name or "attn_combine" in name:
        return "K3"
    if "rope_kv_append" in name:
        return "K2"
    if "chunk_" in name or "DeviceScan" in name:
        return "K1"
    if "pool_copy" in name:
        return "K4"
    if "gemm" in name.lower() or "cutlass" in name.lower() or "sm100" in name or "nvjet" in name:
        return "gemm"
    return "other"


if "--traffic" in sys.argv:
    out = sys.argv[sys.argv.index("--traffic") + 1]
    per = collections.defaultdict(lambda: {"n": 0, "bytes": 0.0, "ns": 0.0})
    for r in rows:
        c = klass(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"].startswith("dram__bytes"):
            per[c]["bytes"] += v
        elif r["Metric Name"] == "gpu__time_duration.sum":
            per[c]["n"] += 1
            per[c]["ns"] += v
    tot_ns = sum(p["ns"] for p in per.values())
    res = {c: p["bytes"] / max(1, p["n"]) for c, p in per.items()}
    res["_share"] = {c: p["ns"] / tot_ns for c, p in per.items()}
    res["_launches"] = {c: p["n"] for c, p in per.items()}
    res["_source"] = path
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res["_share"]))
