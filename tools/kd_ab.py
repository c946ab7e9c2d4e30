"""A/B of KD plan flags at c3 (or another preset): output agreement and per-alpha KD times
(profiled pass) plus the whole forward (events).  Measurement only.

    python tools/kd_ab.py [B] [FLAGS_A] [FLAGS_B] [preset]
FLAGS_* are '+'-joined names without the JTFS_ prefix (e.g. KD_NOTP+KD_NOPAIR) or 0;
preset: c3 (default), c2, p42.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_08269_b200 import build, jtfs, signals  # noqa: E402

build.build()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
fa = sys.argv[2] if len(sys.argv) > 2 else "KD_NOTP"
fb = sys.argv[3] if len(sys.argv) > 3 else "0"
preset = sys.argv[4] if len(sys.argv) > 4 else "c3"
KW = {"c3": dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4),
      "c2": dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False),
      "p42": dict(N=2 ** 16, J=13, Q=16, J_fr=6, T=2 ** 11, F=4)}[preset]


def flags(s):
    return 0 if s == "0" else sum(getattr(jtfs, "JTFS_" + n) for n in s.split("+"))


x = torch.from_numpy(signals.notes(B, N=KW["N"], seed0=1000)).cuda()
res = {}
for name in (fa, fb):
    plan = jtfs.Plan(**KW, flags=flags(name))
    out = plan.forward(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        plan.forward(x, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    plan.profile_read_kd(reset=True)
    plan.profile_enable(True)
    plan.forward(x, out)
    plan.profile_enable(False)
    kd = plan.profile_read_kd(reset=True)
    res[name] = out.clone()
    print(f"{name}: forward {ms:.2f} ms ({B / ms * 1e3:.0f} signals/s); KD per alpha (ms, serialised): "
          + " ".join(f"{v:.2f}" for v in kd), flush=True)
a, b = res[fa].double(), res[fb].double()
d = b - a
rel = float(d.norm() / a.norm())
per = (d.norm(dim=1) / a.norm(dim=1)).max()
print(f"{fb} vs {fa}: rel L2 {rel:.3e} (max per signal {float(per):.3e}), max abs {float(d.abs().max()):.3e}, "
      f"bit-identical {bool(torch.equal(res[fa], res[fb]))}", flush=True)
