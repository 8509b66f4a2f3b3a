mkdir -p gpurun_out/tc30
for i in 1 2; do
PT_LIB=variants/libpt_prev.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc30/prev.txt
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc30/mi1.txt
PT_TC_MI=2 timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc30/mi2.txt
done
PT_TC_MI=2 PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m3 "CTA 0" > gpurun_out/tc30/dbg32.txt
PT_TC_MI=2 timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc30/tests_mi2.txt 2>&1
