mkdir -p gpurun_out/tc33
for d in 33 41; do PT_TC_DBG=$d timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|CTA 0" | head -3 | cut -c1-220 > gpurun_out/tc33/dbg$d.txt; done
