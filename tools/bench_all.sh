#!/bin/bash
# Bench every BASELINE config on one GPU (A-pass roofline, e2e); JSON lines to gpurun_out/bench_all.jsonl
mkdir -p gpurun_out
: > gpurun_out/bench_all.jsonl
for cfg in C1 C2q1 C2q2 C3 C4 C5; do
  case $cfg in C4|C5) S=3; W=2;; C3) S=5; W=3;; *) S=20; W=3;; esac
  timeout -s KILL 600 python bench.py --config $cfg --steps $S --warmup $W --no-cpu-baseline >> gpurun_out/bench_all.jsonl 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?"
done
python - << 'PY'
import json
for l in open("gpurun_out/bench_all.jsonl"):
    d = json.loads(l); r = d["roofline"]
    print(d["config"]["workload"][:40], "ms/step %.2f" % d["ms_per_step"], "decomps/s %.2f" % d["value"],
          "e2e %.2f" % d["e2e"]["value"], "apass %.1f TF (%.0f%%) share %.0f%%" % (r["achieved"], 100 * r["frac"], 100 * r["apass_share_of_step"]))
PY
