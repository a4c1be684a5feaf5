mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x -k qrcp --timeout 300 > gpurun_out/t_qrcp.log 2>&1; echo "rc=$?" >> gpurun_out/t_qrcp.log
timeout -s KILL 600 python -m pytest tests/test_gpu_corutv.py -q -x --timeout 300 > gpurun_out/t_corutv.log 2>&1; echo "rc=$?" >> gpurun_out/t_corutv.log
timeout -s KILL 60 ./tools/qr_phases 4000 60 > gpurun_out/qr_phases.log 2>&1
timeout -s KILL 60 ./tools/qr_phases 960 60 >> gpurun_out/qr_phases.log 2>&1
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.json 2>gpurun_out/bench2.err
CMD="python bench.py --config C2q1 --steps 3 --warmup 3 --no-cpu-baseline"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $CMD > /dev/null 2>&1
tail -3 gpurun_out/t_qrcp.log gpurun_out/t_corutv.log; head -50 gpurun_out/qr_phases.log; cat gpurun_out/bench2.json; python tools/launches_summary.py gpurun_out/launches2.csv
