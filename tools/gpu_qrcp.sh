#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "qrcp" --timeout 120 2>&1 | tail -2
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qr.csv python tools/prof_qr.py > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/launches_qr.csv
