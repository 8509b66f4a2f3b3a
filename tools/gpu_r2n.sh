mkdir -p gpurun_out
( echo "== tc"; timeout 120 python tools/quick_time.py; echo "== tree"; PT_EXH_KERNEL=tree timeout 120 python tools/quick_time.py ) > gpurun_out/r2n.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -k "not scaled" >> gpurun_out/r2n.txt 2>&1
