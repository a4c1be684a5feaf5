#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_rpca.py -q -x --timeout 300 2>&1 | tail -2
timeout -s KILL 600 python bench_rpca.py --no-cpu-baseline > gpurun_out/bench_rpca.json 2> gpurun_out/bench_rpca.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_rpca.json')); r=d['roofline_update']
print('ms/solve', round(d['ms_per_step'],2), 'upd ms', round(r['avg_launch_ms'],3), 'frac', round(r['frac'],3), 'apass frac', round(d['roofline']['frac'],3))"
