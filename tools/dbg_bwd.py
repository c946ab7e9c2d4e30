"""Per-component check of jtfs_backward vs the oracle VJP (debugging aid)."""
import numpy as np
import torch

from oracle import jtfs_grad as Gd
from oracle import jtfs_oracle as O
from paper_2204_08269_b200 import build, signals

build.build()
from paper_2204_08269_b200 import jtfs  # noqa: E402

C1 = dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8)
plan = jtfs.Plan(**C1)
prm = O.Params(**C1)
s = O.schedule(prm)
lay = plan.layout
X = signals.white(1, 2 ** 10, seed=4)
rng = np.random.default_rng(3)
full = rng.standard_normal(plan.floats_per_signal).astype(np.float32)
kinds = [p[0] for p in plan.paths()]
fr = lay.n_frames
masks = {}
m = np.zeros_like(full); m[lay.off_s0:lay.off_s1] = 1; masks["S0"] = m
m = np.zeros_like(full); m[lay.off_s1:lay.off_s2] = 1; masks["S1"] = m
for k, name in [(0, "spin"), (1, "psi_phi"), (2, "phi_psi"), (3, "phi_phi")]:
    m = np.zeros_like(full)
    for pi, kk in enumerate(kinds):
        if kk == k:
            o = lay.off_s2 + pi * lay.lambda_out * fr
            m[o:o + lay.lambda_out * fr] = 1
    masks[name] = m
x = torch.from_numpy(X).cuda()
for name, m in masks.items():
    D = (full * m)[None, :]
    dx = plan.backward(x, torch.from_numpy(D).cuda()).cpu().numpy()[0].astype(np.float64)
    ref = Gd.vjp(X[0].astype(np.float64), D[0].astype(np.float64), prm, s)
    print(f"{name:8s} rel err {np.linalg.norm(dx - ref) / max(np.linalg.norm(ref), 1e-30):.3e}  |ref| {np.linalg.norm(ref):.3e} |gpu| {np.linalg.norm(dx):.3e}  corr {dx @ ref / (np.linalg.norm(dx) * np.linalg.norm(ref) + 1e-30):.4f}")
