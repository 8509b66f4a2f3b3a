set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
for a in "check 16" "check 8" "mma 128 16" "mma 128 8" "mma 64 8" "mma 128 32" "mma 128 64" "mma 128 256" "sttm 4 8" "sttm 4 16" "sttm 8 16" "sttm 16 16" "sttm 16 8"; do
  echo "== $a"; timeout 60 ./tools/ubench_tc $a
done > gpurun_out/r2a_tc.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.txt 2>&1
timeout 300 python bench.py > gpurun_out/r2a_bench.txt 2>&1
tail -3 gpurun_out/r2a_pytest.txt
