#!/bin/bash
mkdir -p gpurun_out
CG=$(grep memory /proc/self/cgroup | cut -d: -f3)
{ echo "cgroup $CG"; cat /sys/fs/cgroup/memory$CG/memory.limit_in_bytes; cat /sys/fs/cgroup/memory$CG/memory.max_usage_in_bytes; } > gpurun_out/mem.txt 2>&1
python -c "
import resource, subprocess, sys
r = subprocess.run([sys.executable, '-m', 'pytest', 'tests/test_gpu_corutv.py', '-m', 'gpu', '-q', '-x', '-k', 'C3'], capture_output=True, text=True)
print(r.stdout[-3000:], r.stderr[-2000:], 'rc', r.returncode)
print('child maxrss MB', resource.getrusage(resource.RUSAGE_CHILDREN).ru_maxrss / 1024)
" > gpurun_out/c3.log 2>&1
cat /sys/fs/cgroup/memory$CG/memory.max_usage_in_bytes >> gpurun_out/mem.txt 2>&1
tail -30 gpurun_out/c3.log; cat gpurun_out/mem.txt
