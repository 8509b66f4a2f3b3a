import sys
sys.path.insert(0, ".")
import torch
from paper_2507_15277_b200 import pt, synth
T, dev = synth.paper_matrix(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
print(pt.pt_kmeans_select(ctx, 24))
