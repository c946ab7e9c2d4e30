"""CTA-pair KD (cta_group::2) against the single-CTA KD (plan flag JTFS_KD_NOPAIR) at c3:
output agreement and per-alpha KD times (profiled pass) plus the whole forward (events).
Measurement only.

    python tools/pair_check.py [B]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_08269_b200 import build, jtfs, signals  # noqa: E402

build.build()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
kw = dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
x = torch.from_numpy(signals.notes(B, seed0=1000)).cuda()
res = {}
for name, flags in (("nopair", jtfs.JTFS_KD_NOPAIR), ("pair", 0)):
    plan = jtfs.Plan(**kw, flags=flags)
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
d = (res["pair"] - res["nopair"]).double()
rel = float(d.norm() / res["nopair"].double().norm())
print(f"pair vs nopair: rel L2 {rel:.3e}, max abs {float(d.abs().max()):.3e}, "
      f"bit-identical {bool(torch.equal(res['pair'], res['nopair']))}", flush=True)
