"""Plain fp64 oracle of the K-nearest-neighbour parameter regression.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA path.

PAPER.md Sec. 3.5 "Regression from Nearest Neighbors":
  * neighbour sets built greedily, Eq.:
        N_0 = {},  N_{k+1}(theta_i) = N_k(theta_i) U { argmin_{theta_j not in N_k} ||S g(theta_j) - S g(theta_i)||_2 },
    "pairwise Euclidean distance with all other examples" -- so j != i (reading R23);
  * estimate theta~_i = (1/K) sum_{theta_j in N_K(theta_i)} theta_j;
  * error ratio theta~_i / theta_i per parameter;
  * K = 40, the Isomap neighbour count.
Readings (R23): distances in fp64 on the fp32 features; ties in the
argmin broken by the smaller example index (the paper is silent; the greedy argmin
with this tie-break equals a stable sort by (distance, index)).
"""
from __future__ import annotations

import numpy as np


def pairwise_sq_dist(F: np.ndarray) -> np.ndarray:
    """D[i, j] = ||F_i - F_j||_2^2 in fp64, written as the plain sum of squared differences."""
    F = np.asarray(F, dtype=np.float64)
    n = F.shape[0]
    D = np.empty((n, n))
    for i in range(n):
        diff = F - F[i]
        D[i] = np.einsum("jd,jd->j", diff, diff)
    return D


def sq_dist_rows(F: np.ndarray, rows) -> np.ndarray:
    """Rows `rows` of pairwise_sq_dist(F) only (for sampled checks at full size)."""
    F = np.asarray(F, dtype=np.float64)
    out = np.empty((len(rows), F.shape[0]))
    for r, i in enumerate(rows):
        diff = F - F[i]
        out[r] = np.einsum("jd,jd->j", diff, diff)
    return out


def knn_row(Drow: np.ndarray, i: int, K: int) -> np.ndarray:
    """N_K(theta_i) from example i's distance row (same rule as knn_sets)."""
    idx = np.arange(len(Drow))
    order = np.lexsort((idx, Drow))
    return order[order != i][:K]


def knn_sets(D: np.ndarray, K: int) -> np.ndarray:
    """N_K(theta_i) for every i, in the order the greedy recursion of P:201-209 adds
    them: row i = the K indices j != i of smallest D[i, j], ties -> smaller j."""
    n = D.shape[0]
    if not 1 <= K < n:
        raise ValueError("need 1 <= K < n")
    out = np.empty((n, K), dtype=np.int64)
    idx = np.arange(n)
    for i in range(n):
        order = np.lexsort((idx, D[i]))          # primary key distance, then index
        order = order[order != i]
        out[i] = order[:K]
    return out


def knn_greedy(D: np.ndarray, K: int, i: int) -> list:
    """The paper's recursion for one example, literally: K argmin steps over the
    examples not yet chosen (and not i itself).  Small cases only."""
    chosen = []
    for _ in range(K):
        best = None
        for j in range(D.shape[0]):
            if j == i or j in chosen:
                continue
            if best is None or D[i, j] < D[i, best]:
                best = j
        chosen.append(best)
    return chosen


def knn_regress(F: np.ndarray, theta: np.ndarray, K: int = 40):
    """Returns (neighbours [n, K], theta_hat [n, P], ratio [n, P])."""
    theta = np.asarray(theta, dtype=np.float64)
    D = pairwise_sq_dist(F)
    nb = knn_sets(D, K)
    theta_hat = theta[nb].mean(axis=1)
    return nb, theta_hat, theta_hat / theta


# ----------------------------------------------------------------------------
# Isomap (Fig. 3): the manifold embedding built on the same K = 40
# neighbour graph (Tenenbaum et al. 2000, cited at P:157)
# ----------------------------------------------------------------------------
def isomap(F: np.ndarray, K: int = 40, n_components: int = 3):
    """Isomap of the rows of F, the algorithm the paper applies: "Isomap
    assembles a geodesic distance matrix by using neighborhood relationships from
    high-dimensional Euclidean distances", 40 nearest neighbours, three components.
    Steps (reading R25, the standard algorithm of the cited reference):
      1. neighbour graph: edge (i, j) of length ||F_i - F_j|| if j in N_K(i) or i in N_K(j)
         (N_K as in knn_sets);
      2. geodesic distances G = all-pairs shortest paths on that graph (library routine);
      3. classical MDS: B = -1/2 H (G o G) H, H = I - 11^T / n;
      4. embedding = top n_components eigenvectors of B scaled by sqrt(eigenvalue).
    Returns (embedding [n, c], eigenvalues [c]); raises if the graph is disconnected."""
    from scipy.sparse.csgraph import shortest_path
    D = pairwise_sq_dist(F)
    nb = knn_sets(D, K)
    n = D.shape[0]
    W = np.zeros((n, n))
    for i in range(n):
        for j in nb[i]:
            W[i, j] = W[j, i] = np.sqrt(D[i, j])
    G = shortest_path(W, method="D", directed=False)
    if not np.all(np.isfinite(G)):
        raise ValueError("neighbour graph is disconnected")
    H = np.eye(n) - np.ones((n, n)) / n
    B = -0.5 * H @ (G * G) @ H
    w, V = np.linalg.eigh(B)
    order = np.argsort(w)[::-1][:n_components]
    w, V = w[order], V[:, order]
    return V * np.sqrt(np.maximum(w, 0.0)), w
