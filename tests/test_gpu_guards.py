"""Out-of-bounds write checks (compute-sanitizer is closed on this GPU pool; these are the
library's own bounds checks):

* a validation build of the library (-DJTFS_WS_GUARDS) gives every workspace region a
  trailing 64 KiB guard band that jtfs_forward fills before and checks after the forward:
  any overflow of one region into the next is an error.  Run on every benchmarked config
  (c1 Eq. 3/4 + periodic, c2, c3 at the bench's 256-signal launch and a ragged batch, c4 in
  the path-sharded latency plan, the Sec. 4.2 preset), in a subprocess (JTFS_LIB selects the
  build);
* with the production library, rows of `out` and `partials` beyond the batch stay untouched.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import numpy as np, torch
from paper_2204_08269_b200 import jtfs, signals
cases = [
    (dict(N=2**10, J=6, Q=8, J_fr=3, T=2**6, F=8), 0, 5),
    (dict(N=2**10, J=6, Q=8, J_fr=3, T=2**6, F=8, average_fr=False), 0, 3),
    (dict(N=2**10, J=6, Q=8, J_fr=3, T=2**6, F=8, pad_mode=jtfs.JTFS_PAD_PERIODIC), 0, 3),
    (dict(N=2**13, J=8, Q=16, J_fr=4, T=2**13, F=16, average_fr=False), 0, 67),
    (dict(N=2**16, J=12, Q=16, J_fr=5, T=2**13, F=4), 0, 256),
    (dict(N=2**16, J=12, Q=16, J_fr=5, T=2**13, F=4), 0, 70),
    (dict(N=2**17, J=13, Q=16, J_fr=5, T=2**13, F=4), jtfs.JTFS_LATENCY, 1),
    (dict(N=2**16, J=13, Q=16, J_fr=6, T=2**11, F=4), 0, 9),
]
for kw, flags, B in cases:
    plan = jtfs.Plan(**kw, flags=flags)
    x = torch.from_numpy(signals.white(B, kw["N"], seed=B)).cuda()
    plan.forward(x)           # raises JTFSError if a guard band was overwritten
    torch.cuda.synchronize()
print("guards ok")
'''


def test_workspace_region_guards():
    from paper_2204_08269_b200 import build
    lib = os.path.join(ROOT, "paper_2204_08269_b200", "libjtfs_guards.so")
    build.build(defines=["JTFS_WS_GUARDS"], lib=lib)
    env = dict(os.environ, JTFS_LIB=lib)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "guards ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_caller_buffers_untouched_beyond_the_batch():
    import torch
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs, signals
    for kw, B in ((dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8), 3),
                  (dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4), 65)):
        plan = jtfs.Plan(**kw)
        x = torch.from_numpy(signals.white(B, kw["N"], seed=2)).cuda()
        big = torch.full((B + 2, plan.floats_per_signal), 7.25, device="cuda")
        plan.forward(x, big[:B])
        torch.cuda.synchronize()
        assert torch.all(big[B:] == 7.25)
    kw = dict(N=2 ** 17, J=13, Q=16, J_fr=5, T=2 ** 13, F=4)
    plan = jtfs.Plan(**kw, flags=jtfs.JTFS_LATENCY)
    x = torch.from_numpy(signals.bird_texture(seed=7)[None, :].copy()).cuda()
    part = torch.full((2, plan.partials_size), 3.5, device="cuda")
    out = torch.full((2, plan.floats_per_signal), 3.5, device="cuda")
    units = list(range(len(plan.units())))
    plan.forward_unitset(x, plan.unitset(units), part[:1], out[:1])
    plan.reduce_pack(part[:1], out[:1])
    torch.cuda.synchronize()
    assert torch.all(part[1:] == 3.5) and torch.all(out[1:] == 3.5)
