mkdir -p gpurun_out
for i in 1 2; do
for lib in default variants/libpt_wait1.so variants/libpt_wait2.so variants/libpt_wait3.so; do
  if [ $lib = default ]; then timeout 120 python tools/k3_time.py; else PT_LIB=$lib timeout 120 python tools/k3_time.py; fi
done; done > gpurun_out/r2aa.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_kmeans.py -q >> gpurun_out/r2aa.txt 2>&1
timeout 300 python tools/quick_time.py 2>&1 | tail -2 >> gpurun_out/r2aa.txt
