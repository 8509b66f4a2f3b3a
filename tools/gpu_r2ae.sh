mkdir -p gpurun_out
( echo "== cluster"; timeout 120 python tools/quick_time.py 2>&1 | grep greedy; echo "== cooperative"; PT_GREEDY_KERNEL=1 timeout 120 python tools/quick_time.py 2>&1 | grep greedy ) > gpurun_out/r2ae.txt 2>&1
timeout 300 python tools/rank_step.py weighted >> gpurun_out/r2ae.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not scaled" >> gpurun_out/r2ae.txt 2>&1
