mkdir -p gpurun_out/tc15
PT_TC_DBG=32 timeout 120 python tools/k3_time.py > gpurun_out/tc15/dbg32.txt 2>&1
timeout 120 python tools/k3_time.py > gpurun_out/tc15/k3.txt 2>&1
PT_TC_H=1 timeout 120 python tools/k3_time.py > gpurun_out/tc15/k3_h1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc15/test_tc.txt 2>&1
