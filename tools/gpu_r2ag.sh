mkdir -p gpurun_out
( timeout 300 python tools/k3_time.py; PT_EXH_TIER=fp16 timeout 300 python tools/k3_time.py ) > gpurun_out/r2ag.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_dist.py -q -x >> gpurun_out/r2ag.txt 2>&1
