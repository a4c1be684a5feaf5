#!/bin/bash
# ncu source-level (warp-stall sampling every 32 cycles) of the register TSQR factor kernel + QRCP
mkdir -p gpurun_out
timeout -s KILL 120 python tools/prof_qr.py > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k "regex:^k_qr_blocked$" -s 4 -c 1 -o gpurun_out/prof_qr_blocked -f python tools/prof_qr.py > gpurun_out/ncu_qr_reg.log 2>&1; echo "rc=$?"
timeout -s KILL 300 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k "regex:k_qrcp_reg" -s 2 -c 1 -o gpurun_out/prof_qrcp_reg -f python tools/prof_qr.py > gpurun_out/ncu_qrcp_reg.log 2>&1; echo "rc=$?"
