mkdir -p gpurun_out; PT_LIB=tools/variants/libpt_tcprobe.so timeout 120 python tools/k3_once.py > gpurun_out/r2o.txt 2>&1
