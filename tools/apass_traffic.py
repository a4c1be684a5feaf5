"""Summarise ncu --set full captures of A-pass launches into profiles/r01_ncu_full_apass_<cfg>.json and
the per-config `traffic` table bench.py reads (profiles/ncu_apass_traffic.json). A launch counts as
an A-pass when it reads at least 90% of A's bytes from DRAM (the small d-wide products do not)."""
import csv, json, subprocess, sys

SHAPES = {"C2q1": (4000, 4000, 8), "C3": (200000, 2000, 8), "C4": (32768, 32768, 8), "C5": (65536, 65536, 4)}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        def f(k):
            if k not in d or d[k] in ("", "n/a"):
                return None
            x = float(d[k].replace(",", ""))
            u = units[h.index(k)]
            return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}.get(u, 1.0)
        res.append({"kernel": d.get("Kernel Name", "")[:70], "grid": d.get("launch__grid_size"),
                    "duration_us": f("gpu__time_duration.sum"),
                    "dram_bytes": (f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0),
                    "tensor_pipe_active_pct": f("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
                    or f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                    "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed")})
    return res


def main():
    table_path = "profiles/ncu_apass_traffic.json"
    table = json.load(open(table_path))
    for cfg in sys.argv[1:]:
        m, n, s = SHAPES[cfg]
        a_bytes = m * n * s
        ls = launches(f"gpurun_out/prof_apass_{cfg}.ncu-rep")
        ap = [x for x in ls if x["dram_bytes"] >= 0.9 * a_bytes]
        json.dump({"config": cfg, "algorithmic_bytes_per_launch": a_bytes, "launches": ls, "apass_launches": len(ap)},
                  open(f"profiles/r01_ncu_full_apass_{cfg}.json", "w"), indent=1)
        if ap:
            table[cfg] = {"dram_bytes_per_launch": sum(x["dram_bytes"] for x in ap) / len(ap),
                          "launches_averaged": len(ap), "algorithmic_bytes_per_launch": a_bytes,
                          "source": f"profiles/r01_ncu_full_apass_{cfg}.json (ncu --set full, A-pass launches)",
                          "tensor_pipe_active_pct_avg": sum(x["tensor_pipe_active_pct"] or 0 for x in ap) / len(ap)}
        print(cfg, "A-pass launches", len(ap), [(round(x["duration_us"]), round(x["dram_bytes"] / a_bytes, 3),
                                                   x["tensor_pipe_active_pct"]) for x in ap])
    json.dump(table, open(table_path, "w"), indent=1)


if __name__ == "__main__":
    main()
