"""Top source lines by warp-stall samples / instructions from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys, collections
path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur_file = None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
with open(path) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if len(r) < 8 or r[2] != "-":   # cuda-level rows have Address '-'
            continue
        try:
            st, ie = float(r[4] or 0), float(r[7] or 0)
        except ValueError:
            continue
        k = (cur_file, int(r[0]))
        agg[k][0] += st
        agg[k][1] += ie
        agg[k][2] = r[1]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts:.0f}, instructions {ti:.0f}")
for (fn, ln), (st, ie, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{100*st/ts:5.1f}% stall {100*ie/ti:5.1f}% inst  {fn}:{ln}: {src.strip()[:100]}")
