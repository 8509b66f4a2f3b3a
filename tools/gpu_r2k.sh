mkdir -p gpurun_out
PT_TRACE=1 timeout 300 python tools/trace_rank.py > gpurun_out/r2k.txt 2>&1
