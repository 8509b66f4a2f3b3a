mkdir -p gpurun_out/tc42
for i in 1 2; do
PT_LIB=variants/libpt_prev.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-200 >> gpurun_out/tc42/prev.txt
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-200 >> gpurun_out/tc42/cur.txt
done
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -x > gpurun_out/tc42/tests.txt 2>&1
