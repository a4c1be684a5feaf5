#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_jacobi_svd -s 3 -c 1 -o gpurun_out/jac python tools/jacobi_ab.py > gpurun_out/ncu_jac.log 2>&1; echo "ncu rc=$?"
