mkdir -p gpurun_out/tc20
timeout 120 python tools/k3_time.py > gpurun_out/tc20/k3.txt 2>&1
PT_TC_H=2 timeout 120 python tools/k3_time.py > gpurun_out/tc20/k3_h2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc20/test_tc.txt 2>&1
