"""Small end-to-end run of every pt_* call, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): tools/sanitize.sh."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

T, dev = synth.small_matrix(3, n_cfg=150, n_dev=3, n_inputs=8)
for flags in (0, pt.PT_GREEDY_STREAM, pt.PT_EXACT_FP64):
    ctx = pt.pt_load_perf(T, dev, flags=flags)
    print(pt.pt_greedy_select(ctx, 6)[0])
    for k in (1, 2, 3, 4):
        print(k, pt.pt_exhaustive_best(ctx, k)["best"])
    print(pt.pt_exhaustive_best(ctx, 3, shard_rank=1, shard_count=3)["best"])
    print(pt.pt_score_sets(ctx, np.array([[0, 1, 2], [5, 6, 7]], np.int32)))
    print(pt.pt_eval_holdout(ctx, 1, 3, 1)["idx"])
    mask = (dev != 0).astype(np.uint8)
    print(pt.pt_exhaustive_best(ctx, 2, env_mask=mask)["best"])
    pt.pt_free(ctx)
print("sanitize driver done")
