"""Per-shard k=3 kernel time at the paper shape for N = 2, 4, 8 shards, run one after
another on one GPU (development aid): the max over shards is the N-GPU kernel time.
LIB=path selects a variant build."""
import os
import sys

sys.path.insert(0, ".")
import paper_2507_15277_b200.pt as pt  # noqa: E402
if os.environ.get("LIB"):
    pt.LIB_PATH = os.environ["LIB"]
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2507_15277_b200 import synth  # noqa: E402

T, dev = synth.paper_matrix(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
pt.pt_exhaustive_best(ctx, 3)
full = pt.pt_get_stats(ctx)["exh_main_ms"]
for N in (2, 4, 8):
    ms = []
    for r in range(N):
        pt.pt_exhaustive_best(ctx, 3, shard_rank=r, shard_count=N)
        pt.pt_exhaustive_best(ctx, 3, shard_rank=r, shard_count=N)
        ms.append(pt.pt_get_stats(ctx)["exh_main_ms"])
    ms = np.array(ms)
    print(f"{os.environ.get('LIB', 'default')} N={N} full={full:.3f} shard ms max={ms.max():.3f} "
          f"mean={ms.mean():.3f} ideal={full / N:.3f} eff={full / N / ms.max():.3f} {np.round(ms, 3).tolist()}",
          flush=True)
