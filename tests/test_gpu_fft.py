"""The FFT engine alone (jtfs_debug_fft) against numpy's fp64 FFT for every length the
path uses, 2^1 .. 2^18: the fp32 engine of KB / KC (shared-memory
Stockham rows up to 4096, four-step above) in both directions and the fp64 engine of KA
(forward).  Bars: relative L2 error <= 4 eps log2 L (fp32: eps = 2^-24; fp64: 2^-53)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def plan():
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    # a cheap plan whose twiddle tables reach N_pad = 2^18 (periodic: N_pad = N)
    return jtfs.Plan(N=2 ** 18, J=4, Q=1, J_fr=2, T=2 ** 13, F=4, pad_mode=jtfs.JTFS_PAD_PERIODIC)


@pytest.mark.parametrize("lg", list(range(1, 19)))
def test_fft_engine_fp32(plan, lg):
    import torch
    L = 1 << lg
    rows = max(1, min(64, (1 << 20) // L))
    rng = np.random.default_rng(lg)
    x = (rng.standard_normal((rows, L)) + 1j * rng.standard_normal((rows, L))).astype(np.complex64)
    xd = torch.from_numpy(x).cuda()
    for d, ref in ((-1, np.fft.fft(x.astype(np.complex128), axis=1)),
                   (+1, np.fft.ifft(x.astype(np.complex128), axis=1) * L)):
        y = plan.debug_fft(xd, d).cpu().numpy().astype(np.complex128)
        err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        assert err <= 4 * 2.0 ** -24 * max(lg, 1), (lg, d, err)


@pytest.mark.parametrize("lg", list(range(1, 19)))
def test_fft_engine_fp64(plan, lg):
    import torch
    L = 1 << lg
    rows = max(1, min(16, (1 << 18) // L))
    rng = np.random.default_rng(100 + lg)
    x = rng.standard_normal((rows, L)) + 1j * rng.standard_normal((rows, L))
    y = plan.debug_fft(torch.from_numpy(x).cuda(), -1).cpu().numpy()
    ref = np.fft.fft(x, axis=1)
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert err <= 4 * 2.0 ** -53 * max(lg, 1), (lg, err)


def test_fft_engine_rejects_bad_args(plan):
    import torch
    from paper_2204_08269_b200 import jtfs
    x = torch.zeros(2, 8, dtype=torch.complex128, device="cuda")
    with pytest.raises(jtfs.JTFSError):
        plan.debug_fft(x, +1)                     # the fp64 engine is forward only
