mkdir -p gpurun_out
for a in "mma 128 8 1" "mma 128 8 2" "mma 128 8 4" "mma 128 8 8" "mma 128 8 16" "mma 128 16 8" "mma 128 16 16" "mma 64 8 16" "mma 128 32 8" "mmass 128 8 1" "mmass 128 8 8" "mmass 128 16 8" "mmass 128 64 4" "mmass 128 256 1"; do
  echo "== $a"; timeout 60 ./tools/ubench_tc $a
done > gpurun_out/r2b_tc.txt 2>&1
