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
ap.add_argument("--fleet", action="store_true",
                help="the fleet objective (Eq. 2) instead: q_dev = FLEET_QDEV, q_env = 1 -> seed<S>_fleet_k<K>")
a = ap.parse_args()
FLEET_QDEV = [5.0, 2.0, 1.0, 3.0, 4.0]   # fleet mix of bench.py next_rows (invented quantities)

res = json.load(open(a.out)) if os.path.exists(a.out) else {}
for seed in a.seeds:
    T, dev = synth.paper_matrix(seed)
    o = Oracle(T, dev)
    if a.fleet:
        o.set_fleet(FLEET_QDEV, [1.0] * T.shape[0])
    for k in a.ks:
        t0 = time.time()
        if a.fleet:
            b, gb, ru, gr = o.fleet_exhaustive_par(k, threads=a.threads)
            key, vals = f"seed{seed}_fleet_k{k}", {"R": gb, "R_runner": gr, "q_dev": FLEET_QDEV, "q_env": 1.0}
        else:
            b, gb, ru, gr = o.exhaustive(k, threads=a.threads)
            key, vals = f"seed{seed}_k{k}", {"G": gb, "G_runner": gr}
        dt = time.time() - t0
        res[key] = dict(vals, best=list(b), runner=list(ru), oracle_seconds=round(dt, 2), threads=a.threads)
        print(seed, k, b, gb, ru, gr, f"{dt:.1f}s", flush=True)
        json.dump(res, open(a.out, "w"), indent=1, sort_keys=True)
