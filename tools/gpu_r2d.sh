timeout 120 ./tools/ubench_tc mma3 > gpurun_out/r2d_tc.txt 2>&1
