mkdir -p gpurun_out
timeout 300 python tools/rank_step.py weighted > gpurun_out/r2ac.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not scaled" >> gpurun_out/r2ac.txt 2>&1
