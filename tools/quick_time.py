"""Quick device timing of the hot path at paper shape (development aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

T, dev = synth.paper_matrix(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
for k in (2, 3):
    for rep in range(3):
        t0 = time.time()
        r = pt.pt_exhaustive_best(ctx, k)
        wall = time.time() - t0
        st = pt.pt_get_stats(ctx)
        evals = st["exh_sets"] * 320
        print(f"k={k} best={r['best']} G={r['G']:.12f} wall={wall*1e3:.2f}ms kernel={st['exh_main_ms']:.3f}ms "
              f"sets={st['exh_sets']} slots={st['exh_slots']} cand={st['exh_candidates']} "
              f"Gevals/s={evals/st['exh_main_ms']/1e6:.1f}", flush=True)
for rep in range(3):
    t0 = time.time()
    idx, gt, gp = pt.pt_greedy_select(ctx, 24)
    print("greedy24", idx[:5], gt[-1], f"wall={(time.time()-t0)*1e3:.2f}ms dev={pt.pt_get_stats(ctx)['greedy_ms']:.3f}ms")
