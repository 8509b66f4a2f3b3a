mkdir -p gpurun_out/tc2
for nt in 1 2 3; do for a in 1.0 1.5 2.0; do PT_TC_NT=$nt PT_TC_ALPHA=$a timeout 300 python tools/k3_time.py > gpurun_out/tc2/k3_nt${nt}_a${a}.txt 2>&1; done; done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/tc2/pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/tc2/bench.txt 2>&1
