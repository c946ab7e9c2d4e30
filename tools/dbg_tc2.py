# dump first tile data of the tcgen05 KD (alpha slot 0) and compare with host math
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_08269_b200 import jtfs, signals
kw = dict(N=2**10, J=6, Q=8, J_fr=3, T=2**6, F=8)
os.environ["JTFS_KD"] = "tc"
os.environ["JTFS_TC_DEBUG"] = "gpurun_out/tcdbg.bin"
X = signals.white(1, kw["N"], seed=3)
x = torch.from_numpy(X).cuda()
p = jtfs.Plan(**kw)
y2 = p.debug_tap(2, x).cpu().numpy()   # planar Y2 (runs through KC only)
out = p.forward(x)
torch.cuda.synchronize()
np.save("gpurun_out/y2.npy", y2)
d = np.fromfile("gpurun_out/tcdbg.bin", dtype=np.float32)
print("Y smem first 64:", d[:64])
print("TMEM lanes 0..3 first 16 cols:", d[8192:8192+64].reshape(4,16))
print("A stage first 64:", d[8192+2048:8192+2048+64])
print("nonzero counts: Y", np.count_nonzero(d[:8192]), "TMEM", np.count_nonzero(d[8192:8192+2048]), "A", np.count_nonzero(d[10240:18432]))
print("Y2 planar first row first 32:", y2[:32])
