mkdir -p gpurun_out/tc24
for i in 1 2; do
PT_LIB=variants/libpt_head.so timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc24/head.txt
timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc24/groups.txt
done
PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m2 "CTA 0" > gpurun_out/tc24/dbg32.txt
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_dist.py -q -x > gpurun_out/tc24/tests.txt 2>&1
