"""Scaled greedy (BASELINE config 5: 65,536 configs x 4,096 envs, k=32) timing."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth  # noqa: E402

t0 = time.time()
T, dev = synth.scaled(1)
print(f"gen {time.time()-t0:.1f}s", flush=True)
dT = torch.from_numpy(T).cuda()
ctx = pt.pt_load_perf(dT, dev)
for rep in range(3):
    t0 = time.perf_counter()
    idx, gt, gp = pt.pt_greedy_select(ctx, 32)
    wall = time.perf_counter() - t0
    st = pt.pt_get_stats(ctx)
    ms = st["greedy_ms"]
    sets = sum(65536 - t for t in range(32))
    gbs = 32 * 65536 * 4096 * 4 / (ms * 1e-3) / 1e9
    print(f"greedy32 wall={wall*1e3:.2f}ms dev={ms:.3f}ms sets/s={sets/(ms*1e-3):.3e} "
          f"l32-stream GB/s={gbs:.0f} G={gt[-1]:.6f} first={idx[:4]} cand={st['greedy_candidates']}", flush=True)
