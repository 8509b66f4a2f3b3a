mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kmeans.py tests/test_gpu_fleet.py -x -q > gpurun_out/r2s.txt 2>&1
timeout 600 python tools/kmeans_scale.py >> gpurun_out/r2s.txt 2>&1
