mkdir -p gpurun_out/tc25
for i in 1 2; do
PT_LIB=variants/libpt_head.so timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc25/head.txt
timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc25/cur.txt
done
PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m3 "CTA 0" > gpurun_out/tc25/dbg32.txt
timeout 1500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_dist.py -q > gpurun_out/tc25/tests.txt 2>&1
