mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_q8.py tests/test_gpu_edges.py tests/test_gpu_fleet.py tests/test_gpu_paths.py -q > gpurun_out/r2ai.txt 2>&1
