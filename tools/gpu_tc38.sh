mkdir -p gpurun_out/tc38
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-230 > gpurun_out/tc38/base.txt
PT_TC_DBG=64 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-230 > gpurun_out/tc38/nofence.txt
PT_TC_DBG=2 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-230 > gpurun_out/tc38/nomma.txt
