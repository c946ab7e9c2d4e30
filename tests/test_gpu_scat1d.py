"""GPU parity of second-order time scattering (jtfs_scattering1d)
against the fp64 oracle's time_scattering, per-path relative L2 <= 1e-4."""
import numpy as np
import pytest

from oracle import jtfs_oracle as O
from paper_2204_08269_b200 import signals

from .parity import TOL, path_errors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def jt():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a visible CUDA device")
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    return jtfs


def _blocks(s0, s1, s2):
    return [s0] + [s1[i] for i in range(s1.shape[0])] + [s2[i] for i in range(s2.shape[0])]


def _check(jt, kw, X, rows=None):
    import torch
    plan = jt.Plan(**kw)
    out = plan.scattering1d(torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda())
    torch.cuda.synchronize()
    prm = O.Params(**kw)
    s = O.schedule(prm)
    O.set_workers(8)
    for b in range(len(X)):
        ref = O.time_scattering(X[b].astype(np.float64), prm, s=s)
        g0, g1, g2 = plan.unpack_scat1d(out[b].cpu().numpy().astype(np.float64))
        blocks_g, blocks_o = _blocks(g0, g1, g2), _blocks(ref["S0"], ref["S1"], ref["S2"])
        sel = list(range(len(blocks_o))) if rows is None else rows
        e = path_errors(blocks_g, blocks_o, sel)
        assert e.max() <= TOL, (float(e.max()), sel[int(np.argmax(e))])


def test_scat1d_c1(jt):
    up = signals.am_chirp(2 ** 10, 1024.0, 64.0, 8.0, 2.0)
    X = np.stack([up, up[::-1].copy(), signals.white(1, 2 ** 10, seed=5)[0]])
    _check(jt, dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8), X)


def test_scat1d_c3_notes(jt):
    _check(jt, dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4), signals.notes(2, seed0=1300))


def test_scat1d_paper_setting(jt):
    # Q = 16, J = 13, T = 2^11, 32 frames
    _check(jt, dict(N=2 ** 16, J=13, Q=16, J_fr=5, T=2 ** 11, F=4), signals.notes(1, seed0=1400))
