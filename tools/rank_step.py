"""Per-rank step time of the N-GPU bench, emulated on one GPU (development aid):
rank r's calls (load, its unsharded part, its k=2/k=3 shards) timed with CUDA events;
the N-GPU step is about the max over ranks plus the NCCL exchanges."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

WEIGHTED = len(sys.argv) > 1 and sys.argv[1] == "weighted"   # the bench's shard weights
T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for N in (1, 2, 4, 8):
    worst = []
    for r in range(N):
        ms = []
        for rep in range(3):
            torch.cuda.synchronize()
            e0.record()
            ctx = pt.pt_load_perf(dT, dev)
            if N > 1 and WEIGHTED:
                extra = [0.0] * N
                extra[0] += 0.24
                extra[1 % N] += 0.16
                extra[2 % N] += 0.12
                pt.pt_set_shard_weights(ctx, [max(0.2, 1.0 - x * N / 12.0) for x in extra])
            if r == 0:
                pt.pt_greedy_select(ctx, 24)
            if N == 1 or r == 2 % N:      # k=2 unsharded on one rank (bench.py)
                pt.pt_exhaustive_best(ctx, 2)
            pt.pt_exhaustive_best(ctx, 3, shard_rank=r, shard_count=N)
            if r == 1 % N:
                pt.pt_eval_holdout_all(ctx, 5, 5)
            pt.pt_free(ctx)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        worst.append(float(np.median(ms)))
    print(f"N={N} per-rank ms {[round(x, 3) for x in worst]} max={max(worst):.3f} "
          f"speedup vs N=1 = {None if N == 1 else round(base / max(worst), 2)}", flush=True)
    if N == 1:
        base = max(worst)
