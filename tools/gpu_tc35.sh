mkdir -p gpurun_out/tc35
for i in 1 2; do
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc35/h1.txt
PT_TC_H=2 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc35/h2.txt
done
PT_TC_H=2 timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc35/tests_h2.txt 2>&1
