"""One Scattering1D forward (P:309-310 setting, 64 notes) after a warm-up, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_08269_b200 import build, jtfs, signals  # noqa: E402

build.build()
plan = jtfs.Plan(N=2 ** 16, J=13, Q=16, J_fr=5, T=2 ** 11, F=4)
x = torch.from_numpy(signals.notes(64, seed0=1000)).cuda()
out = plan.scattering1d(x)
torch.cuda.synchronize()
plan.profile_enable(True)
plan.scattering1d(x, out)
torch.cuda.synchronize()
print({k: round(v[0], 3) for k, v in plan.profile_read().items()})
