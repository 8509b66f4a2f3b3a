"""B200-native hot path of portability tuning (arXiv 2507.15277).

The compute lives in ``libpt.so`` (hand-written sm_100a CUDA behind the C ABI
declared in ``include/pt.h``); ``paper_2507_15277_b200.pt`` is the thin ctypes
binding.  Importing this package does not load the library: ``synth`` (the
seeded input generator) is usable on a CPU-only box.
"""
__all__ = ["pt", "synth"]
