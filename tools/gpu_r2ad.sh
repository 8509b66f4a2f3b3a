mkdir -p gpurun_out; timeout 600 python -m pytest tests/test_gpu_kmeans.py tests/test_gpu_dist.py -q > gpurun_out/r2ad.txt 2>&1
