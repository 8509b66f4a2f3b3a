mkdir -p gpurun_out/tc29
for i in 1 2; do
PT_LIB=variants/libpt_prev.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc29/prev.txt
timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc29/cur.txt
done
PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m3 "CTA 0" > gpurun_out/tc29/dbg32.txt
