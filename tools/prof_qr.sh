#!/bin/bash
# ncu --set full of the QR kernels alone (C2 shapes): k_qr_blocked and k_qrcp
mkdir -p gpurun_out
timeout -s KILL 120 python tools/prof_qr.py > gpurun_out/prof_qr_plain.log 2>&1 || exit 1
for K in ${@:-k_qr_blocked k_qrcp}; do
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k $K -s 3 -c 1 -o gpurun_out/prof_$K -f python tools/prof_qr.py > gpurun_out/prof_qr_ncu_$K.log 2>&1
echo "$K rc=$?"
done
