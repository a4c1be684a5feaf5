"""Summarise an ncu --set full capture of the GEMM launches: duration, DMMA pipe utilisation,
DRAM bytes per launch (traffic) vs the algorithmic bytes, for the A-pass launches."""
import csv, json, subprocess, sys
rep, cfg, m, n, d = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
res = []
for r in rows[2:]:
    dct = dict(zip(h, r))
    f = lambda k: float(dct[k].replace(",", "")) if k in dct and dct[k] not in ("", "n/a") else None
    dur = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    unit = h.index("dram__bytes_read.sum")
    res.append({"kernel": dct.get("Kernel Name", "")[:60], "grid": dct.get("launch__grid_size"),
                "duration_us": dur, "dram_read": rd, "dram_write": wr,
                "dmma_active_pct": f("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
                "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed")})
units = rows[1]
print(json.dumps({"units": {k: units[h.index(k)] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum")}, "launches": res}, indent=1))
