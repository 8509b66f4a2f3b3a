mkdir -p gpurun_out/tc23
for i in 1 2; do
timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc23/ab2.txt
PT_TC_AB=1 timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc23/ab1.txt
done
PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m2 "CTA 0" > gpurun_out/tc23/dbg32.txt
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc23/test_tc.txt 2>&1
