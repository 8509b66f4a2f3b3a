mkdir -p gpurun_out/tc19
timeout 120 python tools/k3_time.py > gpurun_out/tc19/k3.txt 2>&1
PT_TC_H=2 timeout 120 python tools/k3_time.py > gpurun_out/tc19/k3_h2.txt 2>&1
PT_TC_DBG=32 timeout 120 python tools/k3_time.py > gpurun_out/tc19/dbg32.txt 2>&1
PT_TC_DBG=32 PT_TC_H=2 timeout 120 python tools/k3_time.py > gpurun_out/tc19/dbg32_h2.txt 2>&1
