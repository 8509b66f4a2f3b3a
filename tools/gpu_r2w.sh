mkdir -p gpurun_out; timeout 600 python -m pytest tests/test_gpu_kmeans.py -x -q > gpurun_out/r2w.txt 2>&1; timeout 600 python tools/kmeans_scale.py >> gpurun_out/r2w.txt 2>&1
