"""Exploration: K-NN error ratios on the c2 chirp grid with GPU JTFS features."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2204_08269_b200 import jtfs as jt, signals

C2 = dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False)
theta, X = signals.chirp_grid()
plan = jt.Plan(**C2)
x = torch.from_numpy(X).cuda()
S = plan.forward(x)
torch.cuda.synchronize()
L = plan.layout
th = torch.from_numpy(theta).cuda()
res = {}
def q(r):
    return {nm: [round(float(v), 3) for v in np.quantile(r[:, k], [0.05, 0.25, 0.5, 0.75, 0.95])]
            for k, nm in enumerate(("f_c", "f_m", "gamma"))}
feats = {
  "raw_all": S,
  "raw_s2": S[:, L.off_s2:],
  "log1p_all_1e-3": torch.log1p(S.clamp_min(0) / (1e-3 * S.abs().mean(0, keepdim=True) + 1e-30)),
  "mulog": plan.mulog_apply(S, plan.mulog_mu(S), 0.1),
  "mulog_s2": plan.mulog_apply(S, plan.mulog_mu(S), 0.1)[:, L.off_s2:],
}
for k, F in feats.items():
    F = F.contiguous() if not F.is_contiguous() and F.stride(1) != 1 else F
    nb, hat, ratio = jt.knn_regress(F, th, 40)
    res[k] = q(ratio.cpu().numpy())
    print(k, json.dumps(res[k]), flush=True)

# Isomap of the raw records: Spearman correlation of each component with each parameter
import time
from scipy.stats import spearmanr
torch.cuda.synchronize(); t0 = time.perf_counter()
E, w = jt.isomap(S, 40, 3)
torch.cuda.synchronize(); print("isomap s", round(time.perf_counter() - t0, 3), "eig", w.cpu().numpy())
E = E.cpu().numpy()
for k in range(3):
    print("component", k, [round(float(spearmanr(E[:, k], theta[:, p]).correlation), 3) for p in range(3)])
