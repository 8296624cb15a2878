"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel (short name) the launches, mean and total duration, and its share
of the libsg time.  python tools/launch_summary.py <csv> <title> > profiles/<name>.txt"""
import csv
import os
import sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import short  # noqa: E402

path, title = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(r for r in rows if r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
GEN = ("k_kiss", "k_list_from_order", "k_edge_keys", "k_edges_from_keys", "k_gen_")  # input generation, once
agg = OrderedDict()
gen = 0.0
unit = data[0].get("Metric Unit", "") if data else ""
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1e-6)
for d in data:
    name = d["Kernel Name"]
    if "sg::" not in name:
        continue
    k = short(name)
    v = float(d["Metric Value"].replace(",", "")) * scale
    if any(g in name for g in GEN):
        gen += v
        continue
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
print(f"# {title}")
print(f"# {os.path.basename(path)}: {len(data)} launches captured, {sum(v[0] for v in agg.values())} of them libsg's")
print("# ncu serialises launches and runs them cold: compare shares, not absolute times")
print(f"# (input generation kernels, run once before the timed steps, excluded: {gen:.3f} ms)")
print(f"{'kernel':24s} {'launches':>8s} {'mean ms':>10s} {'total ms':>10s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:24s} {c:8d} {t / c:10.4f} {t:10.4f} {t / tot:7.3f}")
