#!/bin/bash
# kernel + decomposition tests, C2 bench, C2 launch list (bounded)
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 > gpurun_out/t_kern.log 2>&1; echo "rc=$?" >> gpurun_out/t_kern.log
tail -4 gpurun_out/t_kern.log
timeout -s KILL 900 python -m pytest tests/test_gpu_corutv.py tests/test_gpu_sharded.py -q -x --timeout 300 > gpurun_out/t_corutv.log 2>&1; echo "rc=$?" >> gpurun_out/t_corutv.log
tail -4 gpurun_out/t_corutv.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json; tail -2 gpurun_out/bench_c2.err
CMD="python bench.py --config C2q1 --steps 3 --warmup 2 --no-cpu-baseline"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2q1.csv $CMD > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/launches_C2q1.csv | head -20
