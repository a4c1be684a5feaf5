#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 120 python tools/tc_debug.py > gpurun_out/tc_debug.log 2>&1; echo "rc=$?" >> gpurun_out/tc_debug.log
cat gpurun_out/tc_debug.log | head -120
