"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
data = [d for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
part = data[len(data) // 2:] if "--second-half" in sys.argv else data
agg = collections.OrderedDict()
for d in part:
    v = float(d["Metric Value"].replace(",", ""))
    v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(d["Metric Unit"], v)
    k = d["Kernel Name"].split("(")[0][:70]
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{len(part)} launches, {tot:.1f} us total")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} us {100 * t / tot:5.1f}%  n={n:5d} avg={t / n:8.2f} us  {k}")
