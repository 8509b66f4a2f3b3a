mkdir -p gpurun_out/tc22
for i in 1 2; do
PT_LIB=variants/libpt_afd.so timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc22/afd.txt
timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc22/cur.txt
PT_TC_H=2 timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc22/cur_h2.txt
done
PT_TC_DBG=32 timeout 120 python tools/k3_time.py > gpurun_out/tc22/dbg32.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc22/test_tc.txt 2>&1
