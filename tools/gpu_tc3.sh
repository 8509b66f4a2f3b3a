mkdir -p gpurun_out/tc3
for cl in 1 2 4; do PT_TC_CL=$cl timeout 300 python tools/k3_time.py > gpurun_out/tc3/k3_cl$cl.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_q8.py -q -x > gpurun_out/tc3/test_tc.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exh_tc -c 1 -o gpurun_out/tc3/k3tc python tools/k3_once.py > gpurun_out/tc3/k3_ncu.txt 2>&1
PT_TC_CL=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exh_tc -c 1 -o gpurun_out/tc3/k3tc_cl2 python tools/k3_once.py > gpurun_out/tc3/k3_ncu_cl2.txt 2>&1
