# round-2 measurement set after the tc tier: tests, bench, reference arm, launch list,
# k_exh_tc full capture, MMA-thread phase profile, memcheck of the tc path
mkdir -p gpurun_out/r02f  # (r02f: same commands, output dir r02f)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02f/pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02f/bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02f/bench_reference.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02f/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-scaled --no-next > gpurun_out/r02f/launches_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exh_tc -c 1 -o gpurun_out/r02f/k3tc python tools/k3_once.py > gpurun_out/r02f/k3_ncu.txt 2>&1
timeout 300 python tools/k3_time.py > gpurun_out/r02f/k3_time.txt 2>&1
PT_TC_DBG=32 timeout 120 python tools/k3_time.py 2>&1 | grep -m2 "CTA 0" > gpurun_out/r02f/k3_phase_profile.txt
timeout 900 python tools/rank_step.py weighted > gpurun_out/r02f/rank_step.txt 2>&1
