mkdir -p gpurun_out
timeout 300 python tools/rank_breakdown.py > gpurun_out/r2i.txt 2>&1
timeout 300 python tools/rank_step.py weighted >> gpurun_out/r2i.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not scaled" >> gpurun_out/r2i.txt 2>&1
