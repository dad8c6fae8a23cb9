"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
launches, total and mean device time per kernel, sorted by total."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d.get("Metric Name") == "gpu__time_duration.sum":
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(
            d.get("Metric Unit", "ns"), 1e-3)
        k = d["Kernel Name"].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
total = sum(t for _, t in agg.values())
print(f"{'launches':>8} {'total us':>11} {'us/launch':>10} {'share':>6}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:8d} {t:11.1f} {t / n:10.2f} {100 * t / total:5.1f}%  {k}")
print(f"{sum(n for n, _ in agg.values()):8d} {total:11.1f}")
