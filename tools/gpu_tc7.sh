mkdir -p gpurun_out/tc7
timeout 300 python tools/k3_time.py > gpurun_out/tc7/k3.txt 2>&1
for d in 1 3; do PT_TC_DBG=$d timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc7/dbg$d.txt; done
PT_TC_NT=1 PT_TC_ALPHA=2.0 timeout 300 python tools/k3_time.py > gpurun_out/tc7/k3_nt1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc7/test_tc.txt 2>&1
