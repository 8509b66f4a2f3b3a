mkdir -p gpurun_out/tc6
for d in 0 1 2 3 4 5 6 7; do PT_TC_DBG=$d timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc6/dbg$d.txt; done
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc6/test_tc.txt 2>&1
