mkdir -p gpurun_out; timeout 600 python tools/kmeans_scale.py > gpurun_out/r2r.txt 2>&1
