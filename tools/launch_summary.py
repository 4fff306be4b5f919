"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python tools/launch_summary.py <launches.csv> > profiles/launches_rNN.json
Per kernel name: launch count, average duration and share of the summed time.
"""
import collections
import csv
import io
import json
import sys

text = open(sys.argv[1]).read()
lines = [l for l in text.splitlines() if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    ns = v * {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1.0)
    k = r["Kernel Name"][:60]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += ns
tot = sum(a[1] for a in agg.values()) or 1.0
out = [{"kernel": k, "launches": n, "avg_ns": t / n, "share": t / tot}
       for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
json.dump(out, sys.stdout, indent=1)
print()
