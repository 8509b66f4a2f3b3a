mkdir -p gpurun_out
timeout 120 python tools/quick_time.py > gpurun_out/r2p.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q >> gpurun_out/r2p.txt 2>&1
