"""GPU parity of the K-NN regression through the C ABI.

Seeded synthetic feature sets (never GPU outputs) vs oracle/knn.py: neighbour indices
bit-exact (the key order is total: fp64 distance, then index), theta~ and the ratios
to 1e-13; exact ties (duplicated examples); full size n = 4096, d = 6936 (the c2 record)
on sampled query rows.  The results-level check against the paper's Fig. 4 claims on the
c2 chirp grid runs the whole GPU pipeline (JTFS + K-NN) and lives in test_gpu_knn_grid.
"""
import numpy as np
import pytest

from oracle import knn as Kn

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


def _gpu(jt, F, th, K):
    import torch
    Fd = torch.from_numpy(np.ascontiguousarray(F, dtype=np.float32)).cuda()
    thd = torch.from_numpy(np.ascontiguousarray(th, dtype=np.float64)).cuda()
    nb, hat, ratio = jt.knn_regress(Fd, thd, K)
    return nb.cpu().numpy(), hat.cpu().numpy(), ratio.cpu().numpy()


@pytest.mark.parametrize("n,d,K", [(600, 300, 40), (65, 1, 64), (130, 77, 5), (2, 3, 1)])
def test_knn_vs_oracle(jt, n, d, K):
    rng = np.random.default_rng(n + d)
    F = (rng.standard_normal((n, d)) * np.exp(rng.uniform(-3, 3, size=d))).astype(np.float32)
    th = rng.uniform(0.5, 4.0, size=(n, 3))
    nb, hat, ratio = _gpu(jt, F, th, K)
    nb_o, hat_o, ratio_o = Kn.knn_regress(F, th, K)
    assert np.array_equal(nb, nb_o)
    np.testing.assert_allclose(hat, hat_o, rtol=1e-13)
    np.testing.assert_allclose(ratio, ratio_o, rtol=1e-13)


def test_knn_exact_ties_go_to_smaller_index(jt):
    rng = np.random.default_rng(8)
    base = rng.standard_normal((20, 16)).astype(np.float32)
    F = np.concatenate([base, base, base[:5]])            # exact duplicates -> equal distances
    th = rng.uniform(1, 2, size=(45, 2))
    nb, hat, _ = _gpu(jt, F, th, 7)
    nb_o, hat_o, _ = Kn.knn_regress(F, th, 7)
    assert np.array_equal(nb, nb_o)
    assert nb[0][0] == 20 and nb[0][1] == 40               # the duplicates of example 0 first, by index
    np.testing.assert_allclose(hat, hat_o, rtol=1e-13)


def test_knn_full_size_sampled_rows(jt):
    # the c2 setting: 4096 examples x 6936 floats (jtfs record of N = 2^13, J = 8, Q = 16, Eq. (4))
    n, d, K = 4096, 6936, 40
    rng = np.random.default_rng(42)
    F = (rng.gamma(0.7, 1.0, size=(n, d)) * np.exp(rng.uniform(-4, 1, size=d))).astype(np.float32)
    th = rng.uniform(0.5, 4.0, size=(n, 3))
    nb, hat, ratio = _gpu(jt, F, th, K)
    rows = list(rng.choice(n, size=24, replace=False)) + [0, n - 1]
    D = Kn.sq_dist_rows(F, rows)
    for r, i in enumerate(rows):
        ref = Kn.knn_row(D[r], i, K)
        assert np.array_equal(nb[i], ref), i
        np.testing.assert_allclose(hat[i], th[ref].mean(axis=0), rtol=1e-13)
        np.testing.assert_allclose(ratio[i], th[ref].mean(axis=0) / th[i], rtol=1e-13)


def test_knn_rejects_bad_args(jt):
    import torch
    F = torch.zeros(10, 4, dtype=torch.float32, device="cuda")
    with pytest.raises(jt.JTFSError):
        jt.knn_regress(F, None, K=10)
    with pytest.raises(jt.JTFSError):
        jt.knn_regress(F[:1], None, K=1)


# ---- Isomap ----
def _iso(jt, F, K, c):
    import torch
    Fd = torch.from_numpy(np.ascontiguousarray(F, dtype=np.float32)).cuda()
    E, w = jt.isomap(Fd, K, c)
    return E.cpu().numpy(), w.cpu().numpy()


def _align(E, R):
    s = np.sign(np.sum(E * R, axis=0))
    s[s == 0] = 1
    return E * s


@pytest.mark.parametrize("n,K", [(500, 10), (130, 7)])
def test_isomap_vs_oracle_anisotropic_box(jt, n, K):
    # points of an anisotropic 3-D box (well separated spectrum) rotated into 40 dims
    rng = np.random.default_rng(n)
    P = rng.uniform(-1, 1, size=(n, 3)) * np.array([10.0, 4.0, 1.5])
    R = np.linalg.qr(rng.standard_normal((40, 40)))[0][:, :3]
    F = (P @ R.T + 0.01 * rng.standard_normal((n, 40))).astype(np.float32)
    E, w = _iso(jt, F, K, 3)
    Eo, wo = Kn.isomap(F, K, 3)
    np.testing.assert_allclose(w, wo, rtol=1e-9)
    np.testing.assert_allclose(_align(E, Eo), Eo, atol=1e-7 * np.abs(Eo).max())
    # deterministic, sign convention: largest-magnitude entry of each eigenvector positive
    E2, _ = _iso(jt, F, K, 3)
    assert np.array_equal(E, E2)
    assert np.all(E[np.argmax(np.abs(E), axis=0), range(3)] > 0)


def test_isomap_helix_vs_oracle(jt):
    t = np.linspace(0, 4 * np.pi, 300)
    F = np.stack([np.cos(t), np.sin(t), 0.3 * t], axis=1).astype(np.float32)
    E, w = _iso(jt, F, 4, 2)
    Eo, wo = Kn.isomap(F, 4, 2)
    np.testing.assert_allclose(w, wo, rtol=1e-9)
    np.testing.assert_allclose(_align(E, Eo), Eo, atol=1e-7 * np.abs(Eo).max())
    assert abs(np.corrcoef(E[:, 0], t)[0, 1]) > 0.999


def test_isomap_disconnected_graph_is_an_error(jt):
    rng = np.random.default_rng(0)
    F = np.concatenate([rng.standard_normal((40, 3)), 1000 + rng.standard_normal((40, 3))]).astype(np.float32)
    with pytest.raises(jt.JTFSError):
        _iso(jt, F, 5, 3)
