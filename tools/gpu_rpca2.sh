#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_rpca.py tests/test_gpu_corutv.py -q -x --timeout 300 -k "rpca or wrapper" > gpurun_out/t_rpca.log 2>&1; echo "rc=$?" >> gpurun_out/t_rpca.log
tail -5 gpurun_out/t_rpca.log
timeout -s KILL 600 python bench_rpca.py > gpurun_out/bench_rpca.json 2> gpurun_out/bench_rpca.err; echo "bench rc=$?"; cat gpurun_out/bench_rpca.json; tail -5 gpurun_out/bench_rpca.err
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_rpca_lift_update -c 1 -o gpurun_out/rpca_upd python bench_rpca.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_rpca.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/rpca_launches.csv python bench_rpca.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_rpca2.log 2>&1; echo "ncu2 rc=$?"
