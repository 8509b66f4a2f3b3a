mkdir -p gpurun_out; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_launches.csv python tools/km_once_scaled.py > gpurun_out/r2t.txt 2>&1
