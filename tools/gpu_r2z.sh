# round-2 measurement set: tests, bench, ncu launch list + full captures, sanitizer
mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02/bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02/bench_reference.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-scaled --no-next > gpurun_out/r02/launches_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exh_tiled -c 1 -o gpurun_out/r02/k3 python tools/k3_once.py > gpurun_out/r02/k3_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_greedy_scan --launch-skip 5 -c 1 -o gpurun_out/r02/scan python tools/scaled_time.py > gpurun_out/r02/scan_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_exh_tiled -c 1 -o gpurun_out/r02/fleet3 python tools/fleet_time.py > gpurun_out/r02/fleet_ncu.txt 2>&1
bash tools/sanitize.sh > gpurun_out/r02/sanitizer.txt 2>&1
