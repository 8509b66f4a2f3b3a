mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_pytest.txt 2>&1
tail -5 gpurun_out/r2e_pytest.txt
timeout 600 python bench.py > gpurun_out/r2e_bench.txt 2>&1
tail -c 3000 gpurun_out/r2e_bench.txt
