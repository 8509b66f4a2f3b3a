"""Fleet (Eq. 2) exhaustive k=2/k=3 at the paper shape (development aid): tiled path
timing (kernel CUDA events) beside the geomean k=3."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402
T, dev = synth.paper_matrix(1)
ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
pt.pt_set_fleet(ctx, np.array([5.0, 2.0, 1.0, 3.0, 4.0]), np.ones(len(dev)))
for k in (2, 3):
    for rep in range(2):
        r = pt.pt_exhaustive_best(ctx, k, objective=pt.PT_OBJ_FLEET)
        st = pt.pt_get_stats(ctx)
        print(f"fleet k={k} best={r['best']} R={r['G']:.12g} runner={r['runner']} R2={r['G_runner']:.12g} "
              f"kernel={st['exh_main_ms']:.3f}ms path={st['exh_kernel']} cand={st['exh_candidates']} "
              f"passes={st['exh_passes']}", flush=True)
r = pt.pt_exhaustive_best(ctx, 3)
print("geomean k=3 kernel", pt.pt_get_stats(ctx)["exh_main_ms"])
