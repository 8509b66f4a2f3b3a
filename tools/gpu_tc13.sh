mkdir -p gpurun_out/tc13
for d in 32 59; do PT_TC_DBG=$d timeout 120 python tools/k3_time.py > gpurun_out/tc13/dbg$d.txt 2>&1; done
