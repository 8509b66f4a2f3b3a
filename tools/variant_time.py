"""Time k=3 for alternative builds of libpt (development aid): LIB=path python tools/variant_time.py"""
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
for rep in range(4):
    r = pt.pt_exhaustive_best(ctx, 3)
    ms.append(pt.pt_get_stats(ctx)["exh_main_ms"])
print(os.environ.get("LIB", "default"), r["best"], "k3 ms", [round(x, 3) for x in ms[1:]],
      "cand", pt.pt_get_stats(ctx)["exh_candidates"], flush=True)
