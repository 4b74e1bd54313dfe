"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel.
usage: python tools/launch_summary.py gpurun_out/TAG_launches_default.csv > profiles/TAG_launches_default.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    k = r[ki].split("(")[0][:70]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
    agg.setdefault(k, []).append(float(r[vi].replace(",", "")) * scale)
own = {k: v for k, v in agg.items() if k.startswith("iga::") or "iga::" in k}
tot = sum(sum(v) for v in own.values())
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none ({sys.argv[1].split('/')[-1]}): per kernel,"
      " cold-cache serialised launches; share = of libiga kernel time (the L2-flush fill is torch's, outside the timed events)")
for k, v in agg.items():
    sh = f"{100 * sum(v) / tot:5.1f}%" if k in own else "  -  "
    print(f"{k:72s} launches={len(v):5d} total_us={sum(v):11.1f} mean_us={sum(v) / len(v):9.2f} share={sh}")
