"""One c3 micro-batch forward for ncu captures (warm-up forward first).

    python tools/prof_c3.py [B]        # B signals (default 64 = one micro-batch)
ncu: -k regex:k_kd_tc -s <launches of the warm-up forward> -c 2   (alpha 0, alpha 1)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_08269_b200 import build, jtfs, signals  # noqa: E402

build.build()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
plan = jtfs.Plan(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
x = torch.from_numpy(signals.notes(B, seed0=1000)).cuda()
out = plan.forward(x)
torch.cuda.synchronize()
plan.forward(x, out)
torch.cuda.synchronize()
print("ok", float(out.abs().sum()))
