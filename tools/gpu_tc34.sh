mkdir -p gpurun_out/tc34
for i in 1 2; do
PT_LIB=variants/libpt_prev.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc34/prev.txt
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc34/split.txt
done
PT_TC_SPLIT=0 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc34/nosplit.txt
PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m3 "CTA 0" > gpurun_out/tc34/dbg32.txt
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_dist.py -q -x > gpurun_out/tc34/tests.txt 2>&1
