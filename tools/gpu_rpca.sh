#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python tools/rpca_check.py > gpurun_out/rpca_check.jsonl 2> gpurun_out/rpca_check.err; echo "rc=$?"
cat gpurun_out/rpca_check.jsonl; tail -5 gpurun_out/rpca_check.err
