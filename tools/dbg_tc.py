import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08269_b200 import jtfs, signals
kw = dict(N=2**10, J=6, Q=8, J_fr=3, T=2**6, F=8)
if len(sys.argv) > 1 and sys.argv[1] == "c3":
    kw = dict(N=2**16, J=12, Q=16, J_fr=5, T=2**13, F=4)
X = signals.white(2, kw["N"], seed=3)
x = torch.from_numpy(X).cuda()
os.environ["JTFS_KD"] = "simt"; pa = jtfs.Plan(**kw); a = pa.forward(x).cpu().numpy()
os.environ["JTFS_KD"] = "tc"; pb = jtfs.Plan(**kw); b = pb.forward(x).cpu().numpy()
torch.cuda.synchronize()
_, _, sa = pa.unpack(a); _, _, sb = pb.unpack(b)
paths = pa.paths()
for i in range(sa.shape[1]):
    na = np.linalg.norm(sa[0, i]); nb = np.linalg.norm(sb[0, i]); d = np.linalg.norm(sa[0, i] - sb[0, i])
    print(i, paths[i][:4], "simt %.4e tc %.4e rel %.3e ratio %.4f" % (na, nb, d / max(na, 1e-30), nb / max(na, 1e-30)))
print("S2 sample simt", sa[0, 0, :2, :4]); print("S2 sample tc", sb[0, 0, :2, :4])
