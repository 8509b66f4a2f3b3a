mkdir -p gpurun_out/tc37
PT_TC_DBG=36 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|CTA 0" | head -3 | cut -c1-260 > gpurun_out/tc37/nowait.txt
PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|CTA 0" | head -3 | cut -c1-260 > gpurun_out/tc37/base.txt
