"""One N=8 rank step (rank 7: load + k=2 shard + k=3 shard), twice -- for an ncu launch list."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402
T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
for rep in range(2):
    ctx = pt.pt_load_perf(dT, dev)
    pt.pt_exhaustive_best(ctx, 2, shard_rank=7, shard_count=8)
    pt.pt_exhaustive_best(ctx, 3, shard_rank=7, shard_count=8)
    pt.pt_free(ctx)
torch.cuda.synchronize()
