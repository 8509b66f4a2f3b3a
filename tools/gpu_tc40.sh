mkdir -p gpurun_out/tc40
for i in 1 2; do
PT_LIB=variants/libpt_prev.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-200 >> gpurun_out/tc40/prev.txt
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-200 >> gpurun_out/tc40/cur.txt
PT_TC_BPAIR=1 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-200 >> gpurun_out/tc40/bpair.txt
done
PT_TC_BPAIR=1 timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc40/tests.txt 2>&1
