"""Pins of the K-NN regression oracle.

* the sort-based neighbour sets equal the paper's greedy argmin recursion, literally
  transcribed, on small random sets;
* points on a line with known gaps: the neighbour sets are known by hand;
* K = n - 1: theta~_i = (sum theta - theta_i) / (n - 1) (closed form);
* invariances of Euclidean K-NN: a translation / orthogonal rotation of the features
  changes nothing; a permutation of the examples permutes the result;
* the distance routine against the Gram-matrix identity ||a-b||^2 = a.a + b.b - 2 a.b.
"""
import numpy as np
import pytest

from oracle import knn as Kn


def test_sets_equal_paper_greedy_recursion():
    rng = np.random.default_rng(0)
    for n, d, K in ((12, 3, 5), (30, 7, 11), (9, 2, 8)):
        F = rng.standard_normal((n, d))
        D = Kn.pairwise_sq_dist(F)
        nb = Kn.knn_sets(D, K)
        for i in range(n):
            assert list(nb[i]) == Kn.knn_greedy(D, K, i)


def test_ties_break_by_index_like_the_greedy_argmin():
    F = np.array([[0.0], [1.0], [-1.0], [2.0], [-2.0]])   # equal distances on both sides
    D = Kn.pairwise_sq_dist(F)
    nb = Kn.knn_sets(D, 4)
    assert list(nb[0]) == [1, 2, 3, 4] == Kn.knn_greedy(D, 4, 0)


def test_points_on_a_line():
    x = np.array([0.0, 1.0, 3.0, 7.0, 15.0])               # gaps 1, 2, 4, 8
    nb = Kn.knn_sets(Kn.pairwise_sq_dist(x[:, None]), 2)
    assert [list(r) for r in nb] == [[1, 2], [0, 2], [1, 0], [2, 1], [3, 2]]


def test_k_equals_n_minus_one_closed_form():
    rng = np.random.default_rng(1)
    F = rng.standard_normal((10, 4))
    th = rng.uniform(1, 2, size=(10, 3))
    _, hat, ratio = Kn.knn_regress(F, th, K=9)
    np.testing.assert_allclose(hat, (th.sum(0) - th) / 9, rtol=1e-14)
    np.testing.assert_allclose(ratio, hat / th, rtol=1e-15)


def test_invariances():
    rng = np.random.default_rng(2)
    F = rng.standard_normal((40, 6))
    th = rng.uniform(1, 2, size=(40, 2))
    nb, hat, _ = Kn.knn_regress(F, th, K=7)
    Qm, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    nb2, hat2, _ = Kn.knn_regress(F @ Qm + 3.0, th, K=7)
    assert np.array_equal(nb, nb2)
    np.testing.assert_allclose(hat, hat2, rtol=1e-14)
    perm = rng.permutation(40)
    nb3, hat3, _ = Kn.knn_regress(F[perm], th[perm], K=7)
    inv = np.argsort(perm)
    np.testing.assert_allclose(hat3, hat[perm], rtol=1e-14)
    assert all(set(perm[nb3[k]]) == set(nb[perm[k]]) for k in range(40))
    del inv


def test_distance_against_gram_identity():
    rng = np.random.default_rng(3)
    F = rng.standard_normal((25, 11))
    G = F @ F.T
    ref = np.diag(G)[:, None] + np.diag(G)[None, :] - 2 * G
    np.testing.assert_allclose(Kn.pairwise_sq_dist(F), ref, atol=1e-12)


def test_rejects_bad_k():
    with pytest.raises(ValueError):
        Kn.knn_sets(np.zeros((4, 4)), 4)


def test_row_helpers_equal_full_matrix():
    rng = np.random.default_rng(4)
    F = rng.standard_normal((30, 5))
    D = Kn.pairwise_sq_dist(F)
    rows = [0, 7, 29]
    np.testing.assert_array_equal(Kn.sq_dist_rows(F, rows), D[rows])
    nb = Kn.knn_sets(D, 6)
    for i in rows:
        assert np.array_equal(Kn.knn_row(D[i], i, 6), nb[i])


# ---- Isomap (NEXT-3) ----
def _align(E, R):
    """Per-component sign alignment of E to R (eigenvector signs are arbitrary)."""
    s = np.sign(np.sum(E * R, axis=0))
    s[s == 0] = 1
    return E * s


def test_isomap_of_points_on_a_line_recovers_the_arc_length():
    # collinear points: every geodesic is the Euclidean distance along the line, so
    # the first coordinate is the centred position (exact), the others vanish
    t = np.sort(np.random.default_rng(6).uniform(0, 10, 60))
    F = np.outer(t, [0.6, 0.8, 0.0])
    E, w = Kn.isomap(F, K=5, n_components=1)
    ref = (t - t.mean())[:, None]
    np.testing.assert_allclose(_align(E, ref), ref, atol=1e-9)
    np.testing.assert_allclose(w[0], np.sum((t - t.mean()) ** 2), rtol=1e-9)


def test_isomap_complete_graph_is_classical_mds():
    # K = n - 1: geodesics = Euclidean distances; classical MDS recovers a centred
    # point cloud up to an orthogonal map: equal Gram matrices
    rng = np.random.default_rng(7)
    P = rng.standard_normal((30, 3)) * np.array([5.0, 2.0, 0.5])
    F = P @ np.linalg.qr(rng.standard_normal((3, 3)))[0].T
    E, w = Kn.isomap(F, K=29, n_components=3)
    Pc = P - P.mean(0)
    np.testing.assert_allclose(E @ E.T, Pc @ Pc.T, atol=1e-9)
    np.testing.assert_allclose(np.sort(w)[::-1], np.sort(np.linalg.eigvalsh(Pc.T @ Pc))[::-1], rtol=1e-9)


def test_isomap_unrolls_a_helix_by_arc_length():
    # a helix is a 1-D manifold curled in 3-D: with a small K the geodesic distance is
    # the arc length, so the top Isomap coordinate is monotone in the curve parameter
    t = np.linspace(0, 4 * np.pi, 200)
    F = np.stack([np.cos(t), np.sin(t), 0.3 * t], axis=1)
    E, _ = Kn.isomap(F, K=4, n_components=1)
    c = np.corrcoef(E[:, 0], t)[0, 1]
    assert abs(c) > 0.999, c
    # the Euclidean embedding (complete graph) does not unroll it
    Ee, _ = Kn.isomap(F, K=199, n_components=1)
    assert abs(np.corrcoef(Ee[:, 0], t)[0, 1]) < abs(c)


def test_isomap_disconnected_graph_raises():
    F = np.concatenate([np.zeros((5, 2)), np.ones((5, 2)) * 100]) + \
        np.random.default_rng(0).standard_normal((10, 2)) * 0.01
    with pytest.raises(ValueError):
        Kn.isomap(F, K=2)
