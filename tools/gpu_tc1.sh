mkdir -p gpurun_out/tc1
timeout 120 ./tools/ubench_tc8 > gpurun_out/tc1/probe.txt 2>&1
timeout 300 python tools/k3_time.py > gpurun_out/tc1/k3_tc.txt 2>&1
PT_EXH_TIER=u8 timeout 300 python tools/k3_time.py > gpurun_out/tc1/k3_u8.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/tc1/test_tc.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_q8.py -x -q > gpurun_out/tc1/test_parity.txt 2>&1
