"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel launches,
total device time and share (cold-cache, serialised: compare shares, not absolutes).

    python scripts/launch_summary.py launches.csv out.json
"""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
tot, n = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0]
    tot[name] += float(r[ix["Metric Value"]].replace(",", "")) * SCALE[r[ix["Metric Unit"]]]
    n[name] += 1
T = sum(tot.values())
out = {k: {"launches": n[k], "total_us": round(v, 1), "mean_us": round(v / n[k], 1), "share_pct": round(100 * v / T, 2)}
       for k, v in tot.most_common()}
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k, v in list(out.items())[:8]:
    print(k[:60], v)
