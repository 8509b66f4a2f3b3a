mkdir -p gpurun_out/tc21
for i in 1 2; do
PT_LIB=variants/libpt_afd.so timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc21/afd.txt
timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc21/cur.txt
PT_TC_H=2 timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 >> gpurun_out/tc21/cur_h2.txt
done
