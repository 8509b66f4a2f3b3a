mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_q8.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_dist.py -q > gpurun_out/r2ah.txt 2>&1
timeout 300 python tools/k3_time.py >> gpurun_out/r2ah.txt 2>&1
bash tools/sanitize.sh > gpurun_out/r2ah_san.txt 2>&1
