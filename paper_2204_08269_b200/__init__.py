"""B200-native forward joint time-frequency scattering (arXiv 2204.08269).

The compute path is the C-ABI library ``libjtfs.so`` (hand-written sm_100a
CUDA, ``csrc/``) declared in ``include/jtfs.h``; ``jtfs.py`` is the thin ctypes
binding with the same names.  ``signals.py`` holds the seeded synthetic inputs.
"""
__all__ = ["jtfs", "signals"]
