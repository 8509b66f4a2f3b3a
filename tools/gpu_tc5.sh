mkdir -p gpurun_out/tc5
timeout 300 python tools/k3_time.py > gpurun_out/tc5/k3.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc5/test_tc.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exh_tc -c 1 -o gpurun_out/tc5/k3tc python tools/k3_once.py > gpurun_out/tc5/k3_ncu.txt 2>&1
