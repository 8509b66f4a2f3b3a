"""PT_TRACE host timeline of one N=8 rank's k=2 + k=3 calls (development aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402
T, dev = synth.paper_matrix(1)
dT = torch.from_numpy(T).cuda()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = pt.pt_load_perf(dT, dev)
    t1 = time.perf_counter()
    pt.pt_exhaustive_best(ctx, 2, shard_rank=7, shard_count=8)
    t2 = time.perf_counter()
    pt.pt_exhaustive_best(ctx, 3, shard_rank=7, shard_count=8)
    t3 = time.perf_counter()
    pt.pt_free(ctx)
    t4 = time.perf_counter()
    print(f"python: load {1e6*(t1-t0):.0f} us, k2 {1e6*(t2-t1):.0f} us, k3 {1e6*(t3-t2):.0f} us, free {1e6*(t4-t3):.0f} us", file=sys.stderr, flush=True)
