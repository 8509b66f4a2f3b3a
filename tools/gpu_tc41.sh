mkdir -p gpurun_out/tc41
for i in 1 2; do
PT_LIB=variants/libpt_prev.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-200 >> gpurun_out/tc41/prev.txt
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median" | cut -c1-200 >> gpurun_out/tc41/lean.txt
done
PT_LIB=variants/libpt_diag.so PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m2 "CTA 0" > gpurun_out/tc41/diag.txt
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc41/tests.txt 2>&1
