mkdir -p gpurun_out/tc27
for i in 1 2; do
PT_LIB=variants/libpt_prev.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc27/prev.txt
PT_LIB=variants/libpt_sleep.so timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-200 >> gpurun_out/tc27/sleep.txt
done
PT_LIB=variants/libpt_sleep.so PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m3 "CTA 0" > gpurun_out/tc27/dbg32.txt
