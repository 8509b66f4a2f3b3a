"""One k-means k=32 on the scaled matrix (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402
T, dev = synth.scaled(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
print(pt.pt_kmeans_select(ctx, 32, max_iter=100))
