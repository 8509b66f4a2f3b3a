"""Per-call breakdown of one rank's bench step at N ranks, emulated on one GPU
(development aid): CUDA events around load, the k=2 shard (incl. its greedy seed when
no trace is cached) and the k=3 shard of a rank that runs neither greedy k=24 nor the
holdout.  Prints ms per call and the fp16-tier survivors."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for N in (1, 8):
    r = N - 1
    rows = []
    for rep in range(5):
        torch.cuda.synchronize()
        ev[0].record()
        ctx = pt.pt_load_perf(dT, dev)
        ev[1].record()
        pt.pt_exhaustive_best(ctx, 2, shard_rank=r, shard_count=N)
        c2 = pt.pt_get_stats(ctx)["exh_candidates"]
        ev[2].record()
        pt.pt_exhaustive_best(ctx, 3, shard_rank=r, shard_count=N)
        st = pt.pt_get_stats(ctx)
        ev[3].record()
        torch.cuda.synchronize()
        rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)] + [st["exh_main_ms"], c2, st["exh_candidates"]])
        pt.pt_free(ctx)
    m = np.median(np.array(rows), axis=0)
    print(f"N={N} rank {r}: load {m[0]:.3f} ms, k=2 shard {m[1]:.3f} ms ({int(m[4])} cand), "
          f"k=3 shard {m[2]:.3f} ms (kernel {m[3]:.3f}, {int(m[5])} cand), total {m[:3].sum():.3f} ms", flush=True)
