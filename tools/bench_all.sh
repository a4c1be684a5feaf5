#!/bin/bash
# Bench every BASELINE config on one GPU (A-pass roofline, e2e), both DVariants; JSON lines to
# gpurun_out/bench_all.jsonl (exact) and gpurun_out/bench_all_approx.jsonl.
mkdir -p gpurun_out
: > gpurun_out/bench_all.jsonl
: > gpurun_out/bench_all_approx.jsonl
for V in exact approx; do
  OUT=gpurun_out/bench_all.jsonl; [ $V = approx ] && OUT=gpurun_out/bench_all_approx.jsonl
  for cfg in C1 C2q1 C2q2 C3 C4 C5; do
    case $cfg in C4|C5) S=3; W=3;; C3) S=5; W=3;; *) S=20; W=3;; esac
    timeout -s KILL 600 python bench.py --config $cfg --variant $V --steps $S --warmup $W --no-cpu-baseline >> $OUT 2> gpurun_out/bench_${cfg}_$V.err
    echo "$cfg $V rc=$?"
  done
done
python - << 'PY'
import json
for f in ["gpurun_out/bench_all.jsonl", "gpurun_out/bench_all_approx.jsonl"]:
    for l in open(f):
        d = json.loads(l); r = d["roofline"]
        print(d["config"]["variant"], d["config"]["workload"][:34], "ms/step %.2f" % d["ms_per_step"], "decomps/s %.2f" % d["value"],
              "e2e %.2f" % d["e2e"]["value"], "apass %.1f TF (%.0f%%) share %.0f%%" % (r["achieved"], 100 * r["frac"], 100 * r["apass_share_of_step"]),
              "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
PY
