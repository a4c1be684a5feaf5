#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_ooc.py tests/test_gpu_corutv.py -q -x --timeout 600 > gpurun_out/t_ooc.log 2>&1; echo "rc=$?" >> gpurun_out/t_ooc.log
tail -8 gpurun_out/t_ooc.log
timeout -s KILL 900 python tools/bench_ooc.py C3 C4 C5 > gpurun_out/bench_ooc.jsonl 2> gpurun_out/bench_ooc.err; echo "bench rc=$?"; cat gpurun_out/bench_ooc.jsonl; tail -3 gpurun_out/bench_ooc.err
