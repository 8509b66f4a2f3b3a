mkdir -p gpurun_out
timeout 120 ./tools/ubench_tc mma2 > gpurun_out/r2c_tc.txt 2>&1
