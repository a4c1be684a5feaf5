#!/bin/bash
# probes + tcgen05 fp32 tests + fused stream-K + QRCP + corutv tests + C2/C5 bench (all bounded)
mkdir -p gpurun_out
timeout -s KILL 60 ./tools/lat_probe > gpurun_out/probes.log 2>&1
timeout -s KILL 60 ./tools/dmma_probe >> gpurun_out/probes.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "tensor_core" --timeout 120 > gpurun_out/t_tc.log 2>&1; echo "rc=$?" >> gpurun_out/t_tc.log
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q --timeout 120 -k "not tensor_core" > gpurun_out/t_kern.log 2>&1; echo "rc=$?" >> gpurun_out/t_kern.log
timeout -s KILL 900 python -m pytest tests/test_gpu_corutv.py -q --timeout 300 > gpurun_out/t_corutv.log 2>&1; echo "rc=$?" >> gpurun_out/t_corutv.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout -s KILL 600 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cat gpurun_out/probes.log; tail -4 gpurun_out/t_tc.log; tail -4 gpurun_out/t_kern.log; tail -4 gpurun_out/t_corutv.log
cat gpurun_out/bench_c2.json gpurun_out/bench_c5.json; tail -2 gpurun_out/bench_c5.err
