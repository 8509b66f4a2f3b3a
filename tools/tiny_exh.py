import sys
sys.path.insert(0, ".")
from paper_2507_15277_b200 import pt, synth
T, dev = synth.tiny(1)
ctx = pt.pt_load_perf(T, dev)
print(pt.pt_exhaustive_best(ctx, 2))
