mkdir -p gpurun_out/tc10
timeout 120 python tools/k3_time.py > gpurun_out/tc10/k3_h2.txt 2>&1
PT_TC_H=1 timeout 120 python tools/k3_time.py > gpurun_out/tc10/k3_h1.txt 2>&1
PT_TC_DBG=3 timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc10/dbg3_h2.txt
PT_TC_DBG=1 timeout 120 python tools/k3_time.py 2>&1 | head -1 | cut -c1-200 > gpurun_out/tc10/dbg1_h2.txt
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc10/test_tc.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exh_tc -c 1 -o gpurun_out/tc10/k3tc python tools/k3_once.py > gpurun_out/tc10/k3_ncu.txt 2>&1
