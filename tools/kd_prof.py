"""Per-role wait cycles of every KD launch (plan flag JTFS_KD_PROF: the instrumented
kernel; the library prints one KDPROF line per alpha to stderr).  Measurement only.

    python tools/kd_prof.py [B] [nopair]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_08269_b200 import build, jtfs, signals  # noqa: E402

build.build()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
extra = jtfs.JTFS_KD_NOPAIR if "nopair" in sys.argv[2:] else 0
plan = jtfs.Plan(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4, flags=jtfs.JTFS_KD_PROF | extra)
x = torch.from_numpy(signals.notes(B, seed0=1000)).cuda()
plan.forward(x)
torch.cuda.synchronize()
print("---- second forward ----", file=sys.stderr, flush=True)
plan.forward(x)
torch.cuda.synchronize()
