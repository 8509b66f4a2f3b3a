mkdir -p gpurun_out
( ./tools/ubench; ./tools/ubench_sad ) > gpurun_out/r2af.txt 2>&1
