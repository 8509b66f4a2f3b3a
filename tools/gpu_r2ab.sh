mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fleet.py tests/test_gpu_kmeans.py -q > gpurun_out/r2ab.txt 2>&1
timeout 300 python - >> gpurun_out/r2ab.txt 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth
T, dev = synth.paper_matrix(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
pt.pt_set_fleet(ctx, np.array([5.0, 2.0, 1.0, 3.0, 4.0]), np.ones(len(dev)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record(); idx, rt, gp = pt.pt_greedy_select(ctx, 24, objective=pt.PT_OBJ_FLEET); e1.record(); torch.cuda.synchronize()
    print("fleet greedy k=24", idx[:6], f"{e0.elapsed_time(e1):.3f} ms", pt.pt_get_stats(ctx)["greedy_ms"])
for rep in range(3):
    e0.record(); sel = pt.pt_kmeans_select(ctx, 24); e1.record(); torch.cuda.synchronize()
    print("kmeans k=24 paper", sel[2], f"{e0.elapsed_time(e1):.3f} ms")
PY
