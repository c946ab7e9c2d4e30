"""Small workload for compute-sanitizer runs (memcheck / racecheck / synccheck), one tool
per gpurun call (profiles/r2_sanitizer_*.log):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Covers the forward path (KA..KE incl. the tcgen05 KD and KC's fp16 store), the SIMT KD,
the backward (VJP), the joint-stage debug entry, path sharding with a bound unit set, time
scattering and the K-NN kernels, on the c1 config and a 3-signal c2 batch.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2204_08269_b200 import build, jtfs, shard, signals  # noqa: E402

build.build()
C1 = dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8)
C2 = dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False)
x1 = torch.from_numpy(np.stack([signals.am_chirp(2 ** 10, 1024.0, 64.0, 8.0, 2.0),
                                signals.white(1, 2 ** 10, seed=3)[0]])).cuda()
p1 = jtfs.Plan(**C1)
o1 = p1.forward(x1)
o1s = jtfs.Plan(**C1, flags=jtfs.JTFS_KD_SIMT).forward(x1)
dx = p1.backward(x1, torch.ones_like(o1))
y2 = p1.debug_tap(2, x1).reshape(2, -1)
yp = p1.debug_tap(3, x1).reshape(2, -1)
oj = p1.debug_joint(y2, yp)
pu = jtfs.Plan(**C1, flags=jtfs.JTFS_LATENCY)
osh = shard.forward_sharded(pu, x1[:1].contiguous())
s1 = p1.scattering1d(x1)
x2 = torch.from_numpy(signals.chirp_grid(n=2)[1][:3].copy()).cuda()
p2 = jtfs.Plan(**C2)
o2 = p2.forward(x2)
nbr, _, _ = jtfs.knn_regress(o2, None, 2)
torch.cuda.synchronize()
print("ok", float(o1.abs().sum()), float((o1 - o1s).abs().max()), float(dx.abs().sum()), float(oj.abs().sum()),
      float(osh.abs().sum()), float(s1.abs().sum()), float(o2.abs().sum()), int(nbr.sum()))
