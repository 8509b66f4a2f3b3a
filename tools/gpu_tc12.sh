mkdir -p gpurun_out/tc12
for d in 27 3 1; do PT_TC_DBG=$d timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc12/dbg$d.txt; done
timeout 120 python tools/k3_time.py > gpurun_out/tc12/k3_h2.txt 2>&1
PT_TC_H=1 timeout 120 python tools/k3_time.py > gpurun_out/tc12/k3_h1.txt 2>&1
