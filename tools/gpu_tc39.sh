mkdir -p gpurun_out/tc39
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x > gpurun_out/tc39/tests.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tc39/bench.txt 2>&1
timeout 600 python tools/rank_step.py weighted > gpurun_out/tc39/rank_step.txt 2>&1
