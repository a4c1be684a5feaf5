#!/bin/bash
# ncu --set full of the QR kernels alone (C2 shapes); arg1 = kernel base name
mkdir -p gpurun_out
K=${1:-k_qr_blocked}
python tools/prof_qr.py > gpurun_out/prof_qr_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k $K -s 3 -c 3 -o gpurun_out/prof_$K -f python tools/prof_qr.py > gpurun_out/prof_qr_ncu.log 2>&1
echo rc=$?; tail -3 gpurun_out/prof_qr_ncu.log
