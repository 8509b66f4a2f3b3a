"""Wall vs device time of each non-k3 call in the bench step (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
ctx = pt.pt_load_perf(dT, dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def probe(name, fn, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(((time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1)))
    st = pt.pt_get_stats(ctx)
    print(f"{name:14s} wall/event ms " + " ".join(f"{w:.3f}/{d:.3f}" for w, d in out[1:]),
          f"greedy_ms={st['greedy_ms']:.3f} exh_main_ms={st['exh_main_ms']:.3f}", flush=True)


probe("greedy24", lambda: pt.pt_greedy_select(ctx, 24))
probe("greedy3", lambda: pt.pt_greedy_select(ctx, 3))
probe("exh2", lambda: pt.pt_exhaustive_best(ctx, 2))
probe("holdout_all", lambda: pt.pt_eval_holdout_all(ctx, 5, 5))
probe("load", lambda: pt.pt_free(pt.pt_load_perf(dT, dev)))
