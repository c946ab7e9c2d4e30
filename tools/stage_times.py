"""Per-stage times (profiled pass) and the whole forward of one c3 micro-batch, plus an
output digest -- for A/B runs of two library builds (JTFS_LIB=...).  Measurement only.

    python tools/stage_times.py [B]
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_08269_b200 import build, jtfs, signals  # noqa: E402

if not os.environ.get("JTFS_LIB"):
    build.build()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
plan = jtfs.Plan(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
x = torch.from_numpy(signals.notes(B, seed0=1000)).cuda()
out = plan.forward(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    plan.forward(x, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
plan.profile_read(reset=True)
plan.profile_enable(True)
plan.forward(x, out)
plan.profile_enable(False)
st = plan.profile_read(reset=True)
dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{os.path.basename(os.environ.get('JTFS_LIB') or 'libjtfs.so')}: forward {ms:.2f} ms ({B / ms * 1e3:.0f} signals/s) "
      + " ".join(f"{k}={v[0]:.2f}" for k, v in st.items()) + f" digest={dig}", flush=True)
