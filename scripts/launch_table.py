"""Per-kernel totals from an ncu --csv launch list (gpu__time_duration.sum):
    python scripts/launch_table.py gpurun_out/launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v = v / 1e6 if r[ix["Metric Unit"]] == "ns" else v / 1e3 if r[ix["Metric Unit"]] == "us" else v
    tot[name] += v
    cnt[name] += 1
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{tot[k]:10.3f} ms {cnt[k]:6d}  {k}")
print(f"{sum(tot.values()):10.3f} ms total")
