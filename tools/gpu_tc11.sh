mkdir -p gpurun_out/tc11
for d in 3 11 19 27 0 16 8; do PT_TC_DBG=$d timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc11/dbg$d.txt; done
