"""Host-side breakdown of one bench step (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(6):
    tt = {}
    if rep >= 3:   # the bench flushes L2 before every step
        flush.fill_(rep)
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
    st = pt.pt_get_stats(ctx)
    tt["exh3_kernel"] = st["exh_main_ms"] / 1e3
    tt["exh3_greedyseed"] = st["greedy_ms"] / 1e3
    t0 = time.perf_counter()
    pt.pt_eval_holdout_all(ctx, 5, 5)
    tt["holdout_all"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pt.pt_free(ctx)
    tt["free"] = time.perf_counter() - t0
    print(" ".join(f"{k}={v*1e3:.2f}ms" for k, v in tt.items()), flush=True)
