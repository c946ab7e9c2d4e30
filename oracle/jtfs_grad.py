"""Gradient oracle of the forward JTFS: texture resynthesis by
gradient descent through the adjoint of the transform.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, smoke() and
bench.py's CPU legs may use it.  It shares no code with the CUDA path.

`forward_torch` is a plain PyTorch fp64 CPU transcription of
`jtfs_oracle.jtfs_forward` (same steps O1-O12, same readings R1-R20, filter
spectra and schedule taken from jtfs_oracle), so torch.autograd gives the exact
vector-Jacobian product of the transform ("reverse-ordered Hermitian adjoints of
the forward scattering operations").  At a zero of |.| autograd
uses the subgradient 0 (torch's sgn(0) = 0); the CUDA path does the same.

  * loss E(y) = ||S x - S y|| / ||S x|| (normalised error);
  * update y <- y - mu grad E (P:358 writes "+"; descent needs the minus sign);
  * bold driver: mu *= up if E decreased, else mu *= down.

Pinned by tests/test_oracle_grad.py: forward_torch equals the numpy oracle,
the gradient equals central finite differences along random directions.
"""
from __future__ import annotations

import numpy as np
import torch

from . import jtfs_oracle as O


def _t(a):
    return torch.as_tensor(np.asarray(a))


def _reflect_index(s: O.Schedule) -> np.ndarray:
    """Index map of numpy 'reflect' padding (reading R6): xp[i] = x[idx[i]]."""
    N = s.p.N
    if s.p.pad == "periodic":
        return np.arange(N)
    i = np.arange(s.N_pad) - s.pad_left
    i = np.abs(i)
    i = np.where(i >= N, 2 * (N - 1) - i, i)
    return i


def forward_torch(x: torch.Tensor, p: O.Params, s: O.Schedule | None = None) -> torch.Tensor:
    """Packed out_3D record [S0 | S1 | S2] of one signal x (fp64 torch tensor, (N,)),
    differentiable.  Step-for-step the numpy oracle (jtfs_oracle.jtfs_forward)."""
    s = s or O.schedule(p)
    fft, ifft = torch.fft.fft, torch.fft.ifft
    N_pad, T = s.N_pad, p.T
    frames = _t(O.time_frames(s))
    xp = x[_t(_reflect_index(s))]
    X = fft(xp)                                                           # O2
    S0 = ifft(X * _t(O.gauss_hat(s.sigma_T, N_pad, N_pad))).real[frames * T]   # O3
    S1, Yphi, Uh = [], [], []
    for lam in range(s.n1):                                               # O4-O5
        k1 = int(s.k1[lam])
        psi = _t(O.morlet_hat(s.xi1[lam], s.sigma1[lam], N_pad, N_pad))
        U1 = torch.abs(ifft(X * psi))[:: 2 ** k1]
        uh = fft(U1)
        Uh.append(uh)
        L1 = N_pad >> k1
        smooth = ifft(uh * _t(O.gauss_hat(s.sigma_T, L1, N_pad))).real
        d = 2 ** (s.log2T - k1)
        S1.append(smooth[frames * d])
        Yphi.append(smooth[torch.arange(N_pad // T) * d])
    S1 = torch.stack(S1)
    Yphi = torch.stack(Yphi)
    Y2 = {}
    for a in s.alphas:                                                    # O6
        ka = s.k_alpha[a]
        rows = []
        for lam in s.adm[a]:
            k1 = int(s.k1[lam])
            L1 = N_pad >> k1
            psi_a = _t(O.morlet_hat(s.xi2[a], s.sigma2[a], L1, N_pad))
            rows.append(ifft(Uh[lam] * psi_a)[:: 2 ** (ka - k1)])
        Y2[a] = torch.stack(rows)

    def phi_T_pool(rows, k):
        L = rows.shape[-1]
        ph = _t(O.gauss_hat(s.sigma_T, L, N_pad))
        full = ifft(fft(rows, dim=-1) * ph, dim=-1).real
        return full[..., frames * 2 ** (s.log2T - k)]

    def phi_F_pool(cols, k):
        R = cols.shape[0]
        ph = _t(O.gauss_hat(s.sigma_F, R, s.N_fr))
        full = ifft(fft(cols, dim=0) * ph[:, None], dim=0).real
        return full[torch.arange(s.lam_out) * 2 ** (s.log2F - k)]

    def grid(rows_by_lambda, width, dtype):
        G = torch.zeros((s.N_fr, width), dtype=dtype)
        for lam, row in rows_by_lambda.items():
            G = G.index_copy(0, torch.tensor([lam]), row[None])
        return G

    avg = p.average_fr
    S2 = []
    gY = {a: fft(grid(dict(zip(s.adm[a], Y2[a])), Y2[a].shape[1], torch.complex128), dim=0) for a in s.alphas}
    gphi = fft(grid({lam: Yphi[lam] for lam in range(s.n1)}, Yphi.shape[1], torch.float64), dim=0)
    for kind, theta, a, b in s.paths:                                     # O7-O9, path order R-O11
        if kind in (O.SPIN, O.PSI_T_PHI_F):
            if kind == O.SPIN:
                fh, k = _t(O.psi_fr_hat(b, theta, s)), int(s.kf[b])
            else:
                fh, k = _t(O.gauss_hat(s.sigma_F, s.N_fr, s.N_fr)), (s.log2F if avg else 0)
            U2 = torch.abs(ifft(gY[a] * fh[:, None], dim=0))[:: 2 ** k]
            P = phi_T_pool(U2, s.k_alpha[a])
            S2.append(phi_F_pool(P, k) if avg else P[: s.n1])
        elif kind == O.PHI_T_PSI_F:
            k = int(s.kf[b])
            U2 = torch.abs(ifft(gphi * _t(O.psi_fr_hat(b, +1, s))[:, None], dim=0))[:: 2 ** k]
            P = phi_T_pool(U2, s.log2T)
            S2.append(phi_F_pool(P, k) if avg else P[: s.n1])
        else:
            k = s.log2F if avg else 0
            V = ifft(gphi * _t(O.gauss_hat(s.sigma_F, s.N_fr, s.N_fr))[:, None], dim=0).real
            S2.append(V[:: 2 ** k][: s.lam_out][:, frames])
    return torch.cat([S0.reshape(-1), S1.reshape(-1), torch.stack(S2).reshape(-1)])


def loss_and_grad(y: np.ndarray, Sx: np.ndarray, p: O.Params, s: O.Schedule | None = None):
    """E(y) = ||Sx - Sy|| / ||Sx|| and dE/dy (fp64)."""
    s = s or O.schedule(p)
    yt = torch.tensor(np.asarray(y, dtype=np.float64), requires_grad=True)
    Sy = forward_torch(yt, p, s)
    Sxt = torch.as_tensor(np.asarray(Sx, dtype=np.float64))
    E = torch.linalg.vector_norm(Sxt - Sy) / torch.linalg.vector_norm(Sxt)
    E.backward()
    return float(E.item()), yt.grad.numpy().copy()


def vjp(x: np.ndarray, dout: np.ndarray, p: O.Params, s: O.Schedule | None = None) -> np.ndarray:
    """d<dout, S(x)>/dx: the vector-Jacobian product of the packed forward record."""
    s = s or O.schedule(p)
    xt = torch.tensor(np.asarray(x, dtype=np.float64), requires_grad=True)
    Sy = forward_torch(xt, p, s)
    (Sy * torch.as_tensor(np.asarray(dout, dtype=np.float64))).sum().backward()
    return xt.grad.numpy().copy()


def resynthesize(Sx: np.ndarray, p: O.Params, y0: np.ndarray, iters: int, mu0: float = 1.0,
                 up: float = 1.2, down: float = 0.5, s: O.Schedule | None = None):
    """Bold-driver gradient descent on E.  Returns (y, [E_n])."""
    s = s or O.schedule(p)
    y, mu = np.asarray(y0, dtype=np.float64).copy(), mu0
    E, g = loss_and_grad(y, Sx, p, s)
    hist = [E]
    for _ in range(iters):
        cand = y - mu * g
        Ec, gc = loss_and_grad(cand, Sx, p, s)
        if Ec < E:
            y, E, g, mu = cand, Ec, gc, mu * up
        else:
            mu *= down
        hist.append(E)
    return y, hist
