#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 200 -k "wide_qr or tsqr" > gpurun_out/t_wide.log 2>&1; echo "rc=$?" >> gpurun_out/t_wide.log
tail -15 gpurun_out/t_wide.log
timeout -s KILL 900 python -m pytest tests/test_gpu_corutv.py tests/test_gpu_fullsize.py -q -x --timeout 400 > gpurun_out/t_corutv.log 2>&1; echo "rc=$?" >> gpurun_out/t_corutv.log
tail -4 gpurun_out/t_corutv.log
timeout -s KILL 600 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout -s KILL 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python - <<'PY'
import json
for f in ["gpurun_out/bench_c5.json","gpurun_out/bench_c4.json"]:
    try:
        d=json.load(open(f)); r=d["roofline"]
        print(f, "ms/step %.1f" % d["ms_per_step"], "apass %.1f TF frac %.2f share %.2f" % (r["achieved"], r["frac"], r["apass_share_of_step"]))
    except Exception as e: print(f, "ERR", e, open(f.replace(".json",".err")).read()[-500:])
PY
