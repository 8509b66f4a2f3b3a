"""Per-rank time of the column-sharded scaled greedy (development aid, 1 GPU):
rank 0 of W scans its 1/W of the 65,536 x 4,096 matrix per step; the other
ranks' records are emulated as empty (so the picks come from shard 0 only --
the per-step scan/pick cost is what a rank of a real W-GPU run pays, minus the
all-gather)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2507_15277_b200 import pt, synth  # noqa: E402

T, dev = synth.scaled(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
del T
pt.pt_greedy_select(ctx, 32)
base = [pt.pt_greedy_select(ctx, 32) and pt.pt_get_stats(ctx)["greedy_ms"] for _ in range(3)]
print("unsharded greedy k=32 ms", [round(x, 3) for x in base], flush=True)
for W in (2, 4, 8):
    def ag(mine, W=W):
        return np.concatenate([mine] + [np.array([np.inf, np.inf, 2**31 - 1, 2**31 - 1])] * (W - 1))
    ms = []
    for _ in range(4):
        pt.pt_greedy_sharded(ctx, 32, ag, 0, W)
        ms.append(pt.pt_get_stats(ctx)["greedy_ms"])
    print(f"shard 0 of {W}: k=32 ms", [round(x, 3) for x in ms[1:]], flush=True)

# stream-ordered (device) exchange flavour: the other ranks' records emulated on device
for W in (2, 4, 8):
    fill = torch.tensor([np.inf, np.inf, 2**31 - 1, 2**31 - 1] * (W - 1), dtype=torch.float64, device="cuda")

    def dag(mine, out, stream, W=W, fill=fill):
        with torch.cuda.stream(stream):
            out[:4].copy_(mine)
            out[4:].copy_(fill)
    ms = []
    for _ in range(4):
        pt.pt_greedy_sharded_dev(ctx, 32, dag, 0, W)
        ms.append(pt.pt_get_stats(ctx)["greedy_ms"])
    print(f"dev shard 0 of {W}: k=32 ms", [round(x, 3) for x in ms[1:]], flush=True)
