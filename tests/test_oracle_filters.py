"""Pins of the oracle's filter generator against closed forms and paper values.

Cites: P:67-70 (Morlet, analytic, Q per octave), P:241 (44 x 32 preset),
SURVEY §8(c) (readings R1-R5) and Appendix A (independent scratch values).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import jtfs_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


BANKS = [(6, 8), (12, 16), (13, 16), (14, 8), (12, 12), (5, 1), (8, 16)]


@pytest.mark.parametrize("J,Q", BANKS)
def test_psi_hat_dc_is_exactly_zero(J, Q):
    # P:68-69 analytic, zero-mean Morlet: psi_hat[0] = 0 exactly (reading R1)
    xi, sg, _ = O.morlet_bank(J, Q)
    for L, n in [(2 ** 11, 2 ** 11), (2 ** 8, 2 ** 11), (512, 512)]:
        for a, b in zip(xi, sg):
            assert O.morlet_hat(a, b, L, n)[0] == 0.0


@pytest.mark.parametrize("J,Q", BANKS)
def test_constant_q_ladder_ratio(J, Q):
    # "Q filters per octave": xi_{i+1}/xi_i = 2^{-1/Q} in the constant-Q region
    xi, sg, _ = O.morlet_bank(J, Q)
    c = sg / xi
    cq = np.isclose(c, c[0], rtol=1e-12)
    n_cq = int(np.argmin(cq)) if not cq.all() else len(xi)
    r = xi[1:n_cq] / xi[: n_cq - 1]
    np.testing.assert_allclose(r, 2.0 ** (-1.0 / Q), rtol=1e-12)
    # linear tail: Q-1 equally spaced filters below the last constant-Q one
    tail = xi[n_cq:]
    assert len(tail) == Q - 1
    if Q > 2:
        np.testing.assert_allclose(np.diff(tail), -xi[n_cq - 1] / Q, rtol=1e-9)


@pytest.mark.parametrize("Q", [1, 2, 8, 12, 16])
def test_neighbours_cross_at_r(Q):
    # reading R2: sigma = c xi is chosen so adjacent Gabor bumps cross at amplitude 1/sqrt(2).
    # Solve the crossing of two Gaussians independently (bisection on the difference).
    xi0 = 0.3
    xi1 = xi0 * 2.0 ** (-1.0 / Q)
    c = O.sigma_ratio(Q)

    def g(w, xi):
        return math.exp(-((w - xi) ** 2) / (2 * (c * xi) ** 2))

    lo, hi = xi1, xi0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if g(mid, xi1) > g(mid, xi0):
            lo = mid
        else:
            hi = mid
    assert abs(g(lo, xi0) - 1 / math.sqrt(2)) < 1e-9


def test_gabor_peak_bin_spec_example():
    # (xi=0.25, sigma=0.025, n=1024) -> argmax bin 256 +- 1 and psi_hat[0] = 0
    h = O.morlet_hat(0.25, 0.025, 1024, 1024)
    assert abs(int(np.argmax(np.abs(h))) - 256) <= 1
    assert h[0] == 0.0


def test_gauss_pair_closed_form():
    # phi_hat[0]=1; phi_hat[k]=phi_hat[L-k]; value = exp(-2 pi^2 sigma_t^2 (k/L)^2),
    # sigma_t = 1/(2 pi sigma)  (Gaussian Fourier pair written in time-domain parameters)
    L, sigma = 256, 0.01
    p = O.gauss_hat(sigma, L, L)
    assert p[0] == 1.0
    np.testing.assert_array_equal(p[1:128], p[255:128:-1])
    st = 1.0 / (2 * np.pi * sigma)
    k = np.arange(128)
    np.testing.assert_allclose(p[:128], np.exp(-2 * np.pi ** 2 * st ** 2 * (k / L) ** 2), rtol=1e-13)
    # and its inverse DFT is the sampled (periodised) time Gaussian of unit mass
    t = np.fft.ifft(O.gauss_hat(0.05, 1024, 1024)).real
    n = np.arange(1024)
    n = np.where(n < 512, n, n - 1024)
    s_t = 1.0 / (2 * np.pi * 0.05)
    ref = np.exp(-n ** 2 / (2 * s_t ** 2)) / (math.sqrt(2 * np.pi) * s_t)
    np.testing.assert_allclose(t, ref, atol=1e-12)


def test_morlet_time_domain_is_modulated_gaussian():
    # P:69 "a complex sinusoid modulated by a Gaussian envelope": away from the small
    # kappa correction, IDFT(psi_hat) = Gaussian * exp(2 pi i xi n) - kappa * Gaussian
    L, xi, sigma = 4096, 0.2, 0.02
    h = np.fft.ifft(O.morlet_hat(xi, sigma, L, L))
    n = np.arange(L)
    n = np.where(n < L // 2, n, n - L)
    st = 1.0 / (2 * np.pi * sigma)
    gauss = np.exp(-n ** 2 / (2 * st ** 2)) / (math.sqrt(2 * np.pi) * st)
    kappa = math.exp(-xi ** 2 / (2 * sigma ** 2))
    ref = gauss * np.exp(2j * np.pi * xi * n) - kappa * gauss
    np.testing.assert_allclose(h, ref, atol=1e-12)


def test_paper_preset_44_by_32():
    # P:241 (Sec. 4.2): J=13, Q=16, Q2=1, F=4, T=2^11, J_fr=6, N=2^16 -> 44 x 32
    g = _gold("paper_pins.json")["sec4_2_preset"]
    pr = g["params"]
    s = O.schedule(O.Params(N=pr["N"], J=pr["J"], Q=pr["Q"], J_fr=pr["J_fr"], T=pr["T"],
                            F=pr["F"], Q2=pr["Q2"], Q_fr=pr["Q_fr"]))
    assert (s.lam_out, s.n_frames) == (g["lambda_out"], g["frames"])
    assert s.n1 == 175


def test_survey_appendix_a_cross_check():
    g = _gold("survey_appendix_a.json")
    for key, n in g["bank_sizes"].items():
        J, Q = map(int, key.split(","))
        assert len(O.morlet_bank(J, Q)[0]) == n
    for q, v in g["xi_max"].items():
        assert abs(O.xi_max(int(q)) - v) < 1e-6
    for q, v in g["sigma_max"].items():
        assert abs(O.sigma_ratio(int(q)) * O.xi_max(int(q)) - v) < 1e-6
    for key, v in g["xi_min"].items():
        J, Q = map(int, key.split(","))
        xi = O.morlet_bank(J, Q)[0]
        assert abs(xi.min() - v) / v < 2e-3     # the last tail filter
    xi, sg, j = O.morlet_bank(6, 8)
    np.testing.assert_allclose(xi, g["c1_G6_8"]["xi"], rtol=2e-5)
    assert list(j) == g["c1_G6_8"]["j"]
    assert abs(sg[-1] - g["c1_G6_8"]["tail_sigma"]) < 1e-6
    xi2, _, j2 = O.morlet_bank(6, 1)
    np.testing.assert_allclose(xi2, g["c1_G6_1"]["xi"], rtol=1e-9)
    assert list(j2) == g["c1_G6_1"]["j"]
    s = O.schedule(O.Params(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8))
    assert [len(s.adm[a]) for a in s.alphas] == g["c1_active_alpha_rows"]
    assert [s.N_pad >> s.k_alpha[a] for a in s.alphas] == g["c1_L_alpha"]


def test_littlewood_paley_upper_frame_bound():
    # Frame bounds of the first-order bank (T2): sum_lambda |psi_hat|^2 over the constant-Q
    # band stays within the survey's measured [1.0002, 1.1258] (J=12, Q=16, L=2^17).
    lo_ref, hi_ref = _gold("survey_appendix_a.json")["lp_sum_J12_Q16_L2p17"]
    L = 2 ** 17
    xi, sg, _ = O.morlet_bank(12, 16)
    lp = np.zeros(L)
    for a, b in zip(xi, sg):
        lp += O.morlet_hat(a, b, L, L) ** 2
    c = sg / xi
    ncq = int(np.sum(np.isclose(c, c[0], rtol=1e-12)))
    band = slice(int(np.ceil(xi[ncq - 1] * L)), int(np.floor(xi[0] * L)) + 1)
    assert lp[band].min() > lo_ref - 1e-3 and lp[band].max() < hi_ref + 1e-3
    assert lp[band].max() > 1.0          # not a tight Parseval frame (no renormalisation, R4)


def test_dyadic_rule_is_alias_free():
    # reading R5: every filter's support edge xi + 5 sigma lies below the Nyquist of its
    # subsampled grid, i.e. (xi + 5 sigma) * 2^(j+1) <= 1 ... up to the 1/2 cap
    for J, Q in BANKS:
        xi, sg, j = O.morlet_bank(J, Q)
        edge = np.minimum(xi + 5 * sg, 0.5)
        assert np.all(edge * 2.0 ** (j + 1) <= 1.0 + 1e-12)
        # ... and j is the largest such exponent (critical) unless clamped at 0
        assert np.all((edge * 2.0 ** (j + 2) > 1.0) | (j == 0))
