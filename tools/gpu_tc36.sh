mkdir -p gpurun_out/tc36
for it in 16 1 2 3; do PT_TC_SWAP_ITERS=$it timeout 120 python tools/k3_time.py 2>&1 | grep -E "median|whole" | cut -c1-260 > gpurun_out/tc36/it$it.txt; done
