"""Pins of the gradient oracle (oracle/jtfs_grad.py).

The torch transcription must equal the pinned numpy oracle, and its autograd
VJP must equal central finite differences of the numpy oracle itself along
random directions (so a slip in either transcription shows up)."""
import numpy as np
import pytest

from oracle import jtfs_grad as Gd
from oracle import jtfs_oracle as O

CASES = [
    O.Params(N=2 ** 8, J=4, Q=4, J_fr=2, T=2 ** 4, F=4),
    O.Params(N=2 ** 8, J=4, Q=4, J_fr=2, T=2 ** 4, F=4, pad="periodic"),
    O.Params(N=2 ** 8, J=4, Q=3, J_fr=2, T=2 ** 5, F=2, average_fr=False),
]
IDS = ["reflect", "periodic", "eq4"]


@pytest.mark.parametrize("prm", CASES, ids=IDS)
def test_torch_forward_equals_numpy_oracle(prm):
    import torch
    rng = np.random.default_rng(5)
    x = rng.standard_normal(prm.N)
    a = Gd.forward_torch(torch.tensor(x), prm).numpy()
    b = O.pack(O.jtfs_forward(x, prm))
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


@pytest.mark.parametrize("prm", CASES, ids=IDS)
def test_vjp_equals_central_differences(prm):
    rng = np.random.default_rng(prm.N + prm.T)
    s = O.schedule(prm)
    x = rng.standard_normal(prm.N)
    dout = rng.standard_normal(O.unpack_layout(s)["total"])
    g = Gd.vjp(x, dout, prm, s)
    for _ in range(3):
        v = rng.standard_normal(prm.N)
        eps = 1e-5
        fp = O.pack(O.jtfs_forward(x + eps * v, prm, s=s)) @ dout
        fm = O.pack(O.jtfs_forward(x - eps * v, prm, s=s)) @ dout
        fd = (fp - fm) / (2 * eps)
        assert abs(g @ v - fd) <= 1e-6 * max(abs(fd), 1e-12 * np.linalg.norm(g) * np.linalg.norm(v)), (g @ v, fd)


def test_resynthesis_decreases_error():
    prm = CASES[0]
    rng = np.random.default_rng(1)
    x = rng.standard_normal(prm.N)
    s = O.schedule(prm)
    Sx = O.pack(O.jtfs_forward(x, prm, s=s))
    y, hist = Gd.resynthesize(Sx, prm, rng.standard_normal(prm.N), iters=15, s=s)
    assert all(b <= a for a, b in zip(hist, hist[1:]))
    assert hist[-1] < 0.7 * hist[0]
