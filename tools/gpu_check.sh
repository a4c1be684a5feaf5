#!/bin/bash
# Quick GPU pass: all gpu tests, smoke, pinv probe, C2q1 bench (exact + approx).
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 300 python tools/pinv_probe.py
for V in exact approx; do
timeout -s KILL 300 python bench.py --config C2q1 --variant $V --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c2_$V.json 2> gpurun_out/b_c2_$V.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/b_c2_*.json")):
    try:
        d=json.load(open(f)); r=d["roofline"]; print(f, "ms/step %.3f" % d["ms_per_step"], "e2e %.1f" % d["e2e"]["value"], "apass frac %.3f" % r["frac"])
    except Exception as e: print(f, "ERR", e, open(f.replace(".json",".err")).read()[-800:])
PY
