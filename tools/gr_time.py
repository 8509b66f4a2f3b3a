"""greedy k=24 device time at the paper shape for a variant build (development aid)"""
import os
import sys

sys.path.insert(0, ".")
import paper_2507_15277_b200.pt as pt  # noqa: E402
if os.environ.get("LIB"):
    pt.LIB_PATH = os.environ["LIB"]
import torch  # noqa: E402
from paper_2507_15277_b200 import synth  # noqa: E402

T, dev = synth.paper_matrix(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
ms = []
for r in range(6):
    idx, _, _ = pt.pt_greedy_select(ctx, 24)
    ms.append(pt.pt_get_stats(ctx)["greedy_ms"])
print(os.environ.get("LIB", "default"), idx[:6], [round(x, 3) for x in ms[1:]], flush=True)
