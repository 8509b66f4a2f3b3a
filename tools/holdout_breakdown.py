import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth
T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
for rep in range(3):
    ctx = pt.pt_load_perf(dT, dev)
    tt = {}
    for d in range(5):
        tr = (dev != d).astype(np.uint8); te = (dev == d).astype(np.uint8)
        for name, fn in (("greedy_train", lambda: pt.pt_greedy_select(ctx, 5, env_mask=tr)),
                         ("score_test", lambda: pt.pt_score_sets(ctx, np.zeros((1, 5), np.int32), env_mask=te)),
                         ("greedy_test", lambda: pt.pt_greedy_select(ctx, 5, env_mask=te)),
                         ("greedy_train_again", lambda: pt.pt_greedy_select(ctx, 5, env_mask=tr)),
                         ("holdout", lambda: pt.pt_eval_holdout(ctx, d, 5, 0))):
            torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); tt[name] = tt.get(name, 0) + time.perf_counter() - t0
    print(" ".join(f"{k}={v*1e3/5:.3f}ms" for k, v in tt.items()), "greedy_dev_ms", round(pt.pt_get_stats(ctx)["greedy_ms"], 3))
    pt.pt_free(ctx)
