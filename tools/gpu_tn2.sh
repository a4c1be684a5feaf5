#!/bin/bash
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tn3.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/tn3.json'));print('C2q1', round(d['ms_per_step'],4))"
timeout -s KILL 300 python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tn4.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/tn4.json'));print('C1', round(d['ms_per_step'],4))"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tn -c 20 --csv --log-file gpurun_out/tn_launch.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/tn_launch.csv 4
timeout -s KILL 900 python -m pytest tests/test_gpu_corutv.py tests/test_gpu_approx.py tests/test_gpu_sharded.py tests/test_gpu_ooc.py -q -x --timeout 300 2>&1 | tail -1
