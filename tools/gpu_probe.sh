#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 60 ./tools/tc_probe > gpurun_out/tc_probe.log 2>&1; echo "rc=$?" >> gpurun_out/tc_probe.log
cat gpurun_out/tc_probe.log
