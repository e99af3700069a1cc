"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel totals
and shares of our (qmoe) kernels' time.  Usage: summarize_launches.py launches.csv out.json 'what'"""
import collections
import csv
import json
import re
import sys

src, dst, what = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
rows = list(csv.reader(l for l in open(src) if l.startswith('"')))
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum" or "qmoe" not in r[ki]:
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("<unnamed>::", "").replace("void ", "")
    name = re.sub(r"<.*", "", name) if "ffn" not in name else name
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi]) / 1e3
tot = sum(v[1] for v in agg.values())
out = {"what": what, "qmoe_kernels": [
    {"kernel": k, "launches": n, "total_us": round(t, 1), "avg_us": round(t / n, 2), "share_of_qmoe_time": round(t / tot, 4)}
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
