# round-2 measurement set after the u8 tier: tests, bench, launch list, k_exh_q8 full capture
mkdir -p gpurun_out/r02b
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02b/pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02b/bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b/bench_reference.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02b/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-scaled --no-next > gpurun_out/r02b/launches_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exh_q8 -c 1 -o gpurun_out/r02b/k3q8 python tools/k3_once.py > gpurun_out/r02b/k3_ncu.txt 2>&1
timeout 300 python tools/k3_time.py > gpurun_out/r02b/k3_time.txt 2>&1
