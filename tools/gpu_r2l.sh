mkdir -p gpurun_out
timeout 300 python tools/rank_step.py weighted > gpurun_out/r2l.txt 2>&1
BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-scaled > gpurun_out/r2l_n2.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2l_bench.txt 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2l_ref.txt 2>&1
