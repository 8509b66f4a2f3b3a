mkdir -p gpurun_out
( timeout 300 python tools/rank_breakdown.py; echo "== PT_EXH_SEED=none"; PT_EXH_SEED=none timeout 300 python tools/rank_breakdown.py ) > gpurun_out/r2f.txt 2>&1
