#!/bin/bash
timeout -s KILL 900 python -m pytest tests/test_gpu_ooc.py -q --timeout 300 2>&1 | grep -E "^E |FAILED|passed|failed" | head -12
timeout -s KILL 600 python -m pytest tests/test_gpu_corutv.py -q -x --timeout 300 -k wrapper 2>&1 | tail -1
