"""Results-level pin of the GPU pipeline against the paper's K-NN regression claims
(Fig. 4), on the c2 AM/FM chirp grid (16^3 signals).

JTFS (Eq. (4), no frequential averaging as in P:164; c2 plan of BASELINE configs[1]) of
all 4096 signals, then K = 40 nearest-neighbour regression of (f_c, f_m, gamma) on the
plain Euclidean distance between the records.  The paper: "All feature
representations are capable of regressing carrier frequency f_c with error ratios close
to 1 ... time scattering and JTFS excel at linearizing modulation frequency ... with error
ratios within range of 0.75 to 1.5 ... all features except MFCCs extract chirp rate within
error ratios between 0.75 to 1.25".  Reading R24: "within range" = the 5th-95th percentile
of the per-example error ratios; "close to 1" = within [0.9, 1.1].
"""
import numpy as np
import pytest

from paper_2204_08269_b200 import signals

pytestmark = pytest.mark.gpu

C2 = dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False)


def test_knn_error_ratios_on_the_chirp_grid_match_fig4():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a visible CUDA device")
    from paper_2204_08269_b200 import jtfs as jt
    theta, X = signals.chirp_grid()
    plan = jt.Plan(**C2)
    S = plan.forward(torch.from_numpy(X).cuda())
    nb, hat, ratio = jt.knn_regress(S, torch.from_numpy(theta).cuda(), K=40)
    r = ratio.cpu().numpy()
    lo, hi = np.quantile(r, 0.05, axis=0), np.quantile(r, 0.95, axis=0)
    assert 0.9 <= lo[0] and hi[0] <= 1.1, (lo, hi)          # f_c: close to 1
    assert 0.75 <= lo[1] and hi[1] <= 1.5, (lo, hi)         # f_m: 0.75 .. 1.5
    assert 0.75 <= lo[2] and hi[2] <= 1.25, (lo, hi)        # gamma: 0.75 .. 1.25
    # the neighbours are other examples, and every estimate is their mean
    nbh = nb.cpu().numpy()
    assert not np.any(nbh == np.arange(len(theta))[:, None])
    np.testing.assert_allclose(hat.cpu().numpy(), theta[nbh].mean(axis=1), rtol=1e-13)


def test_isomap_components_align_with_the_three_parameters():
    # Fig. 3(d): "the dataset of AM/FM signals is represented as a 3-D mesh
    # where the principal components align independently with f_c, f_m and gamma".
    # Reading R26: each parameter has its own Isomap component with |Spearman rho| >= 0.8,
    # and every other (component, parameter) pair has |rho| <= 0.3.
    import torch
    from scipy.stats import spearmanr
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a visible CUDA device")
    from paper_2204_08269_b200 import jtfs as jt
    theta, X = signals.chirp_grid()
    plan = jt.Plan(**C2)
    S = plan.forward(torch.from_numpy(X).cuda())
    E, w = jt.isomap(S, K=40, n_components=3)
    E = E.cpu().numpy()
    assert np.all(np.diff(w.cpu().numpy()) <= 0)
    rho = np.array([[abs(spearmanr(E[:, k], theta[:, p]).correlation) for p in range(3)] for k in range(3)])
    best = rho.argmax(axis=0)                       # component of each parameter
    assert sorted(best) == [0, 1, 2], rho
    assert np.all(rho[best, range(3)] >= 0.8), rho
    mask = np.ones((3, 3), bool)
    mask[best, range(3)] = False
    assert np.all(rho[mask] <= 0.3), rho
