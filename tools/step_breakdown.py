"""Host-side breakdown of one bench step (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
for rep in range(4):
    tt = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = pt.pt_load_perf(dT, dev)
    tt["load"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pt.pt_greedy_select(ctx, 24)
    tt["greedy24"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pt.pt_exhaustive_best(ctx, 2)
    tt["exh2"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pt.pt_exhaustive_best(ctx, 3)
    tt["exh3"] = time.perf_counter() - t0
    tt["exh3_kernel"] = pt.pt_get_stats(ctx)["exh_main_ms"] / 1e3
    t0 = time.perf_counter()
    for d in range(5):
        pt.pt_eval_holdout(ctx, d, 5, 0)
    tt["holdout5"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pt.pt_free(ctx)
    tt["free"] = time.perf_counter() - t0
    print(" ".join(f"{k}={v*1e3:.2f}ms" for k, v in tt.items()), flush=True)
