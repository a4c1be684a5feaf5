#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_ooc.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -q --timeout 600 > gpurun_out/t_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu2.log
tail -8 gpurun_out/t_gpu2.log
