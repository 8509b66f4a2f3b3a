mkdir -p gpurun_out
timeout 300 python tools/fleet_time.py > gpurun_out/r2q.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fleet.py tests/test_gpu_dist.py -x -q >> gpurun_out/r2q.txt 2>&1
