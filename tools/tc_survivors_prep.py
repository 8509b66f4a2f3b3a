"""Write /tmp/l.bin for tools/tc_survivors.c: the paper-shaped synthetic matrix's
log-slowdowns l[c][e] = log(T[e][c] / min_c T[e][c]) (fp64, config-major)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2507_15277_b200 import synth  # noqa: E402

T, dev = synth.paper_matrix(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
T = T.astype(np.float64)
l = np.log(T / T.min(axis=1, keepdims=True)).T.copy()
with open("/tmp/l.bin", "wb") as f:
    f.write(np.array([l.shape[1], l.shape[0]], dtype=np.int32).tobytes())
    f.write(l.tobytes())
