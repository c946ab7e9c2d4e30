"""Compare backward intermediates (S1-only dout) with a numpy emulation of the adjoint."""
import numpy as np
import torch

from oracle import jtfs_oracle as O
from paper_2204_08269_b200 import build, signals

build.build()
from paper_2204_08269_b200 import jtfs  # noqa: E402

C1 = dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8)
plan = jtfs.Plan(**C1)
prm = O.Params(**C1)
s = O.schedule(prm)
lay = plan.layout
x = signals.white(1, 2 ** 10, seed=4)[0]
rng = np.random.default_rng(3)
dout = np.zeros(plan.floats_per_signal, np.float32)
dS1 = rng.standard_normal((s.n1, s.n_frames)).astype(np.float32)
dout[lay.off_s1:lay.off_s2] = dS1.ravel()
xt = torch.from_numpy(x[None, :].copy()).cuda()
dx = plan.backward(xt, torch.from_numpy(dout[None, :]).cuda())
torch.cuda.synchronize()
off = plan.backward_regions(1)
ws = plan._bws.cpu().numpy()
def region(i, dtype, n):
    return np.frombuffer(ws[off[i]:off[i] + n * np.dtype(dtype).itemsize].tobytes(), dtype=dtype)
u1_total = sum(s.N_pad >> int(s.k1[l]) for l in range(s.n1))
gu1hat = region(11, np.complex64, u1_total)
gu1 = region(12, np.float32, u1_total)
wb = region(13, np.complex64, u1_total)
gw = region(14, np.complex64, u1_total)
gxhat = region(15, np.complex64, s.N_pad)
# emulation
Np = s.N_pad
X = np.fft.fft(O.pad_signal(x.astype(np.float64), s))
o = 0
gX = np.zeros(Np, complex)
for lam in range(s.n1):
    k1 = int(s.k1[lam]); L1 = Np >> k1; d = 2 ** (s.log2T - k1)
    psi = O.morlet_hat(s.xi1[lam], s.sigma1[lam], Np, Np)
    W = np.fft.ifft(X * psi)[::2 ** k1]
    phi = O.gauss_hat(s.sigma_T, L1, Np)
    gs = np.zeros(L1); gs[O.time_frames(s) * d] = dS1[lam]
    gUh = np.conj(phi) * np.fft.fft(gs) / L1
    gU1 = np.real(np.fft.ifft(gUh) * L1)
    gW = gU1 * W / np.abs(W)
    GW = np.fft.fft(gW)
    up = np.zeros(Np, complex); up[::2 ** k1] = gW
    gX += np.conj(psi) * np.fft.fft(up) / Np
    def rel(a, b):
        return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    if lam % 8 == 0 or lam == s.n1 - 1:
        print(f"lam {lam:3d} L1 {L1:5d} gU1hat {rel(gu1hat[o:o+L1], gUh):.2e} gU1 {rel(gu1[o:o+L1], gU1):.2e} "
              f"W {rel(wb[o:o+L1], W):.2e} GW {rel(gw[o:o+L1], GW):.2e}")
    o += L1
print("gXhat", np.linalg.norm(gxhat - gX) / np.linalg.norm(gX))
