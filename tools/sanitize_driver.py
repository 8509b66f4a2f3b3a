"""Small end-to-end run of every pt_* call, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): tools/sanitize.sh.  LIB=path selects a
variant build (e.g. the opt-in tensor-summed exhaustive kernel)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2507_15277_b200.pt as pt  # noqa: E402
if os.environ.get("LIB"):
    pt.LIB_PATH = os.environ["LIB"]
from paper_2507_15277_b200 import synth  # noqa: E402

T, dev = synth.small_matrix(3, n_cfg=150, n_dev=3, n_inputs=8)
for flags in (0, pt.PT_GREEDY_STREAM, pt.PT_EXACT_FP64, pt.PT_GREEDY_LAZY):
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
ctx = pt.pt_load_perf(T, dev)
print("holdout_all", [h["idx"] for h in pt.pt_eval_holdout_all(ctx, 3, 3)])
print("swap", pt.pt_swap_search(ctx, 4))
print("kmeans", pt.pt_kmeans_select(ctx, 3))
print("sharded host", pt.pt_greedy_sharded(ctx, 5, lambda m: m, 0, 1)[0])
print("sharded dev", pt.pt_greedy_sharded_dev(ctx, 5, lambda m, o, s: o.copy_(m), 0, 1)[0])
qd = np.arange(1, 4, dtype=np.float64)
qe = np.ones(T.shape[0], np.float64)
pt.pt_set_fleet(ctx, qd, qe)
print("fleet greedy", pt.pt_greedy_select(ctx, 3, objective=pt.PT_OBJ_FLEET)[0])
print("fleet exh", pt.pt_exhaustive_best(ctx, 2, objective=pt.PT_OBJ_FLEET)["best"])
print("fleet score", pt.pt_score_sets(ctx, np.array([[0, 1]], np.int32), objective=pt.PT_OBJ_FLEET))
print("fleet exh tiled k3", pt.pt_exhaustive_best(ctx, 3, objective=pt.PT_OBJ_FLEET)["best"],
      pt.pt_get_stats(ctx)["exh_kernel"])
print("fleet exh tiled shard", pt.pt_exhaustive_best(ctx, 3, shard_rank=1, shard_count=2,
                                                     objective=pt.PT_OBJ_FLEET)["best"])
# the library-side record exchange + device merge (world 1, stream-ordered callback)
print("sharded exhaustive", pt.pt_exhaustive_best_sharded(ctx, 3, 0, 1, allgather=lambda m, o, s: o.copy_(m))["best"])
print("sharded fleet", pt.pt_exhaustive_best_sharded(ctx, 2, 0, 1, allgather=lambda m, o, s: o.copy_(m),
                                                     objective=pt.PT_OBJ_FLEET)["best"])
print("kmeans k8", pt.pt_kmeans_select(ctx, 8, max_iter=4))
pt.pt_free(ctx)
print("sanitize driver done")
# multi-stage column tiles (E_pad = 192: three 64-env stages per tile, the ring wraps
# inside a tile) for the producer-less release protocol
T2, dev2 = synth.small_matrix(4, n_cfg=200, n_dev=3, n_inputs=64)
ctx = pt.pt_load_perf(T2, dev2)
pt.pt_greedy_select(ctx, 5)
print("k3 multi-stage", pt.pt_exhaustive_best(ctx, 3)["best"], pt.pt_exhaustive_best(ctx, 2)["best"])
pt.pt_free(ctx)
print("sanitize driver done (multi-stage)")
