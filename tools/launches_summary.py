"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) > vi and "coru_gpu" in r[ki]:
        k = r[ki].split("(")[0].replace("void coru_gpu::<unnamed>::", "")
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", ""))
tot = sum(v for _, v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}%  n={c:4d} avg {v / c / 1e3:8.1f} us  {k}")
