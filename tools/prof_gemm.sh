#!/bin/bash
# ncu --set full of the A-pass GEMM kernels inside a short bench run (one op N and one op T launch)
mkdir -p gpurun_out
CFG=${1:-C2q1}
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline"
timeout -s KILL 300 $CMD > gpurun_out/prof_gemm_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_f64 -s 4 -c 2 -o gpurun_out/prof_gemm_$CFG -f $CMD > gpurun_out/prof_gemm_ncu.log 2>&1
echo "ncu rc=$?"
