"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total time and share."""
import collections
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0].replace("void ", "")[:90]
    agg[k][0] += 1
    agg[k][1] += float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total_us':>10} {'share':>6}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:8d} {t / 1e3:10.1f} {100 * t / tot:5.1f}%  {k}")
