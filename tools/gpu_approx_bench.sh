mkdir -p gpurun_out
for V in exact approx; do
timeout -s KILL 300 python bench.py --config C2q1 --variant $V --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c2_$V.json 2> gpurun_out/b_c2_$V.err
timeout -s KILL 300 python bench.py --config C1 --variant $V --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c1_$V.json 2> gpurun_out/b_c1_$V.err
done
timeout -s KILL 600 python bench.py --config C5 --variant approx --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b_c5_approx.json 2> gpurun_out/b_c5_approx.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2q1_approx.csv python bench.py --config C2q1 --variant approx --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/b_*.json")):
    try:
        d=json.load(open(f)); print(f, "ms/step %.3f" % d["ms_per_step"], "e2e %.1f" % d["e2e"]["value"], "launches", d["gpu_launches"])
    except Exception as e: print(f, "ERR", e, open(f.replace(".json",".err")).read()[-800:])
PY
python tools/launches_summary.py gpurun_out/launches_C2q1_approx.csv
