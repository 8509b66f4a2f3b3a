mkdir -p gpurun_out/tc8
timeout 120 python tools/k3_time.py > gpurun_out/tc8/k3_pair.txt 2>&1
PT_TC_PAIR=0 timeout 120 python tools/k3_time.py > gpurun_out/tc8/k3_single.txt 2>&1
PT_TC_DBG=3 timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc8/dbg3_pair.txt
PT_TC_DBG=1 timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc8/dbg1_pair.txt
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc8/test_tc.txt 2>&1
