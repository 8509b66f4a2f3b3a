mkdir -p gpurun_out/tc18
timeout 60 python tools/tc_small.py > gpurun_out/tc18/small.txt 2>&1; echo "rc=$?" >> gpurun_out/tc18/small.txt
PT_TC_DBG=32 timeout 120 python tools/k3_time.py > gpurun_out/tc18/dbg32.txt 2>&1
timeout 120 python tools/k3_time.py > gpurun_out/tc18/k3.txt 2>&1
PT_TC_H=2 timeout 120 python tools/k3_time.py > gpurun_out/tc18/k3_h2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc18/test_tc.txt 2>&1
