"""Pins of the NEXT-4 oracle functions: mu-log compression
(Eqs. (adalog:mu), (adalog)) and the Fig. 1 scale-rate map.

The u2_map values themselves are pinned against the no-FFT brute force in
test_oracle_bruteforce.py; here: the paper's qualitative Fig. 1 claim on the map,
and invariants / closed forms of mu-log that a dropped term, a wrong axis or a
wrong normalisation would break.
"""
import numpy as np

from oracle import jtfs_oracle as O
from paper_2204_08269_b200 import signals

C1 = O.Params(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8)


def test_u2_map_fig1_up_chirp_energy_on_theta_minus_one():
    # Fig. 1(a) bottom: for an upward chirp the map of Psi_{alpha,beta,-1}
    # holds more energy than Psi_{alpha,beta,+1}; the time-reversed chirp the opposite.
    s = O.schedule(C1)
    up = signals.am_chirp(C1.N, 1024.0, 64.0, 8.0, 2.0).astype(np.float64)
    down = up[::-1].copy()
    spin = {(th, a, b): pi for pi, (k, th, a, b) in enumerate(s.paths) if k == O.SPIN}
    # the (alpha, beta) pair with the most theta=-1 energy for the up-chirp
    e = {key: np.sum(O.u2_map(up, C1, pi, s) ** 2) for key, pi in spin.items() if key[0] == -1}
    _, a, b = max(e, key=e.get)
    em, ep = (np.sum(O.u2_map(up, C1, spin[(th, a, b)], s) ** 2) for th in (-1, +1))
    dm, dp = (np.sum(O.u2_map(down, C1, spin[(th, a, b)], s) ** 2) for th in (-1, +1))
    assert em > 2 * ep and dp > 2 * dm, (em, ep, dm, dp)


def test_u2_map_shape_covers_lambda_and_time_axes():
    s = O.schedule(C1)
    for pi, (k, th, a, b) in enumerate(s.paths):
        if k not in (O.SPIN, O.PSI_T_PHI_F):
            continue
        rows, cols = O.u2_map_shape(s, pi)
        kf = int(s.kf[b]) if k == O.SPIN else s.log2F
        assert (rows - 1) * 2 ** kf < s.n1 <= rows * 2 ** kf        # the whole lambda axis
        assert cols * 2 ** s.k_alpha[a] >= C1.N > (cols - 1) * 2 ** s.k_alpha[a]  # the whole signal


def _maps(rng, B=3, P=5, lam=4, fr=6):
    return rng.random((B, P, lam, fr)) * rng.random((1, P, 1, 1)) * 10


def test_mulog_closed_form_constant_maps():
    # constant map c over (lambda, t) for every example: mu = c lam fr, so
    # S~ = log(1 + 1 / (eps lam fr)) whatever c
    lam, fr, eps = 4, 6, 0.1
    c = np.array([0.5, 2.0, 7.0])
    S = np.broadcast_to(c[None, :, None, None], (2, 3, lam, fr)).copy()
    mu = O.mulog_mu(S)
    np.testing.assert_allclose(mu, c * lam * fr, rtol=1e-15)
    np.testing.assert_allclose(O.mulog(S, mu, eps), np.log(1 + 1 / (eps * lam * fr)), rtol=1e-14)
    # S = eps mu (e - 1)  ->  exactly 1
    S1 = (eps * mu * (np.e - 1))[None, :, None, None] * np.ones((1, 3, lam, fr))
    np.testing.assert_allclose(O.mulog(S1, mu, eps), 1.0, rtol=1e-14)


def test_mulog_scale_invariance_and_batch_mean():
    rng = np.random.default_rng(5)
    S = _maps(rng)
    ref = O.mulog(S, O.mulog_mu(S))
    # invariant under a global gain (loudness): mu scales with S
    np.testing.assert_allclose(O.mulog(3.7 * S, O.mulog_mu(3.7 * S)), ref, rtol=1e-13)
    # per-path gains are also removed (mu is per lambda_2)
    g = rng.random(S.shape[1])[None, :, None, None] + 0.5
    np.testing.assert_allclose(O.mulog(g * S, O.mulog_mu(g * S)), ref, rtol=1e-13)
    # mu is the mean over examples of each map's (lambda, t) sum
    np.testing.assert_allclose(O.mulog_mu(S), np.mean([O.mulog_mu(S[i:i + 1]) for i in range(3)], axis=0),
                               rtol=1e-14)
    # zero maps -> 0, monotone in S
    Z = np.zeros_like(S)
    Z[:, 0] = S[:, 0]
    out = O.mulog(Z, O.mulog_mu(Z))
    assert np.all(out[:, 1:] == 0) and np.all(np.isfinite(out))
    assert np.all(np.diff(np.sort(S.ravel())) >= 0)
    a = O.mulog(S, O.mulog_mu(S))
    mu = O.mulog_mu(S)
    assert np.all(O.mulog(S * 1.01, mu) > a - 1e-15)
