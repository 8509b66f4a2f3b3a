"""Write tests/golden/paper_exhaustive.json: the CPU oracle's exhaustive k=2/k=3
results on the full paper-shaped synthetic matrices (1,775 configs x 320 envs).

Calls ONLY oracle/ (and the seeded generator).  The stored values are what the
full-size GPU parity tests compare against; regenerate with
    python scripts/make_golden.py [--seeds 1 2 3] [--threads N]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Oracle, default_threads  # noqa: E402
from paper_2507_15277_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, nargs="+", default=[1, 2, 3])
ap.add_argument("--ks", type=int, nargs="+", default=[2, 3])
ap.add_argument("--threads", type=int, default=default_threads())
ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "paper_exhaustive.json"))
a = ap.parse_args()

res = json.load(open(a.out)) if os.path.exists(a.out) else {}
for seed in a.seeds:
    T, dev = synth.paper_matrix(seed)
    o = Oracle(T, dev)
    for k in a.ks:
        t0 = time.time()
        b, gb, ru, gr = o.exhaustive(k, threads=a.threads)
        dt = time.time() - t0
        res[f"seed{seed}_k{k}"] = {"best": list(b), "G": gb, "runner": list(ru), "G_runner": gr,
                                   "oracle_seconds": round(dt, 2), "threads": a.threads}
        print(seed, k, b, gb, ru, gr, f"{dt:.1f}s", flush=True)
        json.dump(res, open(a.out, "w"), indent=1, sort_keys=True)
