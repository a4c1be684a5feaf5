#!/bin/bash
# One-off GPU-box probe: host CPU, GPU, FP64 instruction throughputs, cuBLAS DGEMM peak.
mkdir -p gpurun_out
{ lscpu | head -20; nproc; free -g; nvidia-smi; } > gpurun_out/probe_host.txt 2>&1
./tools/fp64_peak > gpurun_out/probe_fp64.txt 2>&1
python tools/dgemm_peak.py 8192 >> gpurun_out/probe_fp64.txt 2>&1
python tools/dgemm_peak.py 4096 >> gpurun_out/probe_fp64.txt 2>&1
cat gpurun_out/probe_fp64.txt
