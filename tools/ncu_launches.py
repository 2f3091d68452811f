"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``).

usage: python tools/ncu_launches.py launches.csv [out.json]

Groups launches by kernel name and reports count, total / mean duration and
each kernel's share of the time spent in kmx kernels (the bench's own
per-kernel CUDA-event split must agree with these shares, not with the
absolute cold-cache, serialised ncu durations).
"""
import csv
import json
import re
import sys
from collections import OrderedDict


def summarise(path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
        rows.append((r["Kernel Name"], v * scale.get(r["Metric Unit"], 1e-3)))
    agg = OrderedDict()
    for name, us in rows:
        base = name.split("(")[0]
        mk = re.search(r"(k_\w+(<[^>]*>)?)", base)
        short = mk.group(1) if mk else base.replace("void ", "")
        a = agg.setdefault(short, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += us
    peaks = ("k_imad_peak", "k_tc_peak")
    kmx_total = sum(a["total_us"] for k, a in agg.items() if k.startswith("k_") and k not in peaks)
    out = []
    for k, a in agg.items():
        e = {"kernel": k, "launches": a["launches"], "total_us": round(a["total_us"], 2),
             "mean_us": round(a["total_us"] / a["launches"], 2)}
        if k.startswith("k_") and k not in peaks and kmx_total > 0:
            e["share_of_kmx_time"] = round(a["total_us"] / kmx_total, 4)
        out.append(e)
    return {"source": path, "total_launches": len(rows), "kernels": out}


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    txt = json.dumps(s, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")
    print(txt)
