"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"][:70]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v[1] / 1e6:8.2f} ms {100 * v[1] / tot:5.1f}% n={v[0]:5d} avg={v[1] / v[0] / 1e3:9.1f} us  {k}")
print(f"total {tot / 1e6:.2f} ms")
