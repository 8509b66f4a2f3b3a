mkdir -p gpurun_out; timeout 120 ./tools/ubench_tc acc > gpurun_out/r2m.txt 2>&1; timeout 60 ./tools/ubench_tc check 8 >> gpurun_out/r2m.txt 2>&1
