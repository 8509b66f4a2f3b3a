"""k=3 kernel time at the paper shape, 5 reps (development aid; PT_LIB selects a variant)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402
T, dev = synth.paper_matrix(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
ms = []
for rep in range(6):
    r = pt.pt_exhaustive_best(ctx, 3)
    ms.append(pt.pt_get_stats(ctx)["exh_main_ms"])
st = pt.pt_get_stats(ctx)
print(os.environ.get("PT_LIB", "default"), os.environ.get("PT_EXH_TIER", "u8"), r["best"], r["runner"], r["G"],
      "k3 kernel ms", [round(x, 3) for x in ms[1:]], "median", round(float(np.median(ms[1:])), 3),
      "kernel", st["exh_kernel"], "candidates", st["exh_candidates"], "passes", st["exh_passes"],
      "nt", st["exh_tc_nt"], "tc_survivors", st["exh_tc_survivors"], flush=True)
# whole call (swap search + operands + kernel + refine), CUDA events around it
s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
calls = []
for rep in range(5):
    torch.cuda.synchronize()
    s_.record()
    pt.pt_exhaustive_best(ctx, 3)
    e_.record()
    torch.cuda.synchronize()
    calls.append(s_.elapsed_time(e_))
print("k3 whole call ms", [round(x, 3) for x in calls], flush=True)
for k in (2, 4):
    r = pt.pt_exhaustive_best(ctx, k)
    r = pt.pt_exhaustive_best(ctx, k)
    st = pt.pt_get_stats(ctx)
    print("k", k, r["best"], r["runner"], "ms", round(st["exh_main_ms"], 3), "kernel", st["exh_kernel"],
          "candidates", st["exh_candidates"], flush=True)
