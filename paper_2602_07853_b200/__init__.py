"""B200-native (sm_100a) MPM Lite solve-time hot path.

The product is the C-ABI CUDA library ``libmpmlite.so`` (include/mpmlite.h) and its thin
Python binding ``paper_2602_07853_b200.mpl``.  ``scenes`` holds the seeded synthetic input
generators (no method arithmetic).  Importing this package does not load the library; import
``paper_2602_07853_b200.mpl`` for that (it raises if the library is missing — no CPU fallback).
"""
__all__ = ["scenes", "mpl", "build"]
