mkdir -p gpurun_out/tc14
PT_TC_DBG=32 timeout 120 python tools/k3_time.py > gpurun_out/tc14/dbg32.txt 2>&1
PT_TC_H=1 PT_TC_DBG=32 timeout 120 python tools/k3_time.py > gpurun_out/tc14/dbg32_h1.txt 2>&1
