#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 60 ./tools/qr_reg_tl 4000 60 > gpurun_out/qr_reg_tl.log 2>&1
timeout -s KILL 60 ./tools/qr_reg_tl 1000 25 >> gpurun_out/qr_reg_tl.log 2>&1
timeout -s KILL 60 ./tools/qr_phases 4000 60 >> gpurun_out/qr_reg_tl.log 2>&1
timeout -s KILL 60 ./tools/qr_phases 1000 25 >> gpurun_out/qr_reg_tl.log 2>&1
grep -v "^[0-9]*:" gpurun_out/qr_reg_tl.log
