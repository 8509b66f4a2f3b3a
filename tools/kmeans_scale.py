"""k-means selector at the scaled shape (development aid): 4,096 environments x 65,536
configurations, k = 32 -- device time of pt_kmeans_select (CUDA events) and its passes."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402
T, dev = synth.scaled(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    l0 = pt.pt_get_stats(ctx)["launches"]
    e0.record()
    t0 = time.perf_counter()
    sel, G, iters = pt.pt_kmeans_select(ctx, 32, max_iter=100)
    e1.record()
    torch.cuda.synchronize()
    print(f"kmeans k=32 on 4096 x 65536: {e0.elapsed_time(e1):.1f} ms device, {1e3*(time.perf_counter()-t0):.1f} ms wall, "
          f"iterations {iters}, {len(sel)} selected, G {G:.6f}, launches {pt.pt_get_stats(ctx)['launches'] - l0}",
          flush=True)
print(sel)
