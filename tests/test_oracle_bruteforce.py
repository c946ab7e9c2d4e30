"""Brute-force pin of the oracle's pipeline at tiny N (T3).

A second, independent transcription of SURVEY §8(c) O1-O11 in which every
convolution is an explicit circular convolution with time-domain taps obtained
by an explicit inverse-DFT sum (no FFT anywhere), and every decimation is done
by index arithmetic written out here.  It reuses only the oracle's *filter
spectra* (pinned separately in test_oracle_filters.py) and its schedule
(pinned by the count tests).  A dropped term, a wrong sign, a transposed
operand, a wrong decimation index or an FFT scaling slip in the oracle makes
these tests fail.
"""
import numpy as np
import pytest

from oracle import jtfs_oracle as O


def idft_explicit(fh):
    L = len(fh)
    n = np.arange(L)
    E = np.exp(2j * np.pi * np.outer(n, n) / L) / L
    return E @ fh


def dft_explicit(v):
    L = len(v)
    n = np.arange(L)
    E = np.exp(-2j * np.pi * np.outer(n, n) / L)
    return E @ v


def circ_matrix(h):
    """C[n, t] = h[(n - t) mod L] so that (C @ x)[n] = sum_t h[n - t] x[t]."""
    L = len(h)
    n = np.arange(L)
    return h[(n[:, None] - n[None, :]) % L]


def circconv(x, h):
    return circ_matrix(h) @ x


def reflect_index(p, pad_left, N):
    i = p - pad_left
    if i < 0:
        i = -i
    if i >= N:
        i = 2 * (N - 1) - i
    return i


def brute_jtfs(x, prm):
    s = O.schedule(prm)
    N, N_pad, T = prm.N, s.N_pad, prm.T
    if prm.pad == "reflect":
        xp = np.array([x[reflect_index(p, s.pad_left, N)] for p in range(N_pad)], float)
    else:
        xp = x.astype(float)
    frames = [s.frame0 + i for i in range(s.n_frames)]
    # S0
    hT = idft_explicit(O.gauss_hat(s.sigma_T, N_pad, N_pad))
    y = circconv(xp, hT)
    S0 = np.array([y[m * T].real for m in frames])
    # first order
    S1 = np.zeros((s.n1, s.n_frames))
    Yphi = np.zeros((s.n1, N_pad // T))
    U1 = []
    for lam in range(s.n1):
        k1 = int(s.k1[lam])
        h = idft_explicit(O.morlet_hat(s.xi1[lam], s.sigma1[lam], N_pad, N_pad))
        w = circconv(xp, h)
        u = np.abs(np.array([w[n * 2 ** k1] for n in range(N_pad >> k1)]))
        U1.append(u)
        L1 = N_pad >> k1
        hphi = idft_explicit(O.gauss_hat(s.sigma_T, L1, N_pad))
        sm = circconv(u, hphi).real
        d = 2 ** (s.log2T - k1)
        S1[lam] = [sm[m * d] for m in frames]
        Yphi[lam] = [sm[n * d] for n in range(N_pad // T)]
    # second order in time
    Y2 = {}
    for a in s.alphas:
        ka = s.k_alpha[a]
        rows = []
        for lam in s.adm[a]:
            k1 = int(s.k1[lam])
            L1 = N_pad >> k1
            h = idft_explicit(O.morlet_hat(s.xi2[a], s.sigma2[a], L1, N_pad))
            w = circconv(U1[lam].astype(complex), h)
            rows.append([w[n * 2 ** (ka - k1)] for n in range(N_pad >> ka)])
        Y2[a] = np.array(rows)

    Nfr = s.N_fr

    def fr_taps(kind, b, theta):
        if kind == "psi":
            fh = O.morlet_hat(s.xif[b], s.sigmaf[b], Nfr, Nfr)
            if theta == +1:
                fh = np.array([fh[(-m) % Nfr] for m in range(Nfr)])
        else:
            fh = O.gauss_hat(s.sigma_F, Nfr, Nfr)
        return idft_explicit(fh)

    def time_pool(U, k):
        L = U.shape[1]
        hphi = idft_explicit(O.gauss_hat(s.sigma_T, L, N_pad))
        Cm = circ_matrix(hphi)
        d = 2 ** (s.log2T - k)
        P = (U @ Cm.T).real                      # each row convolved with phi_T
        return P[:, [m * d for m in frames]]

    def lam_pool(P, k):
        R = P.shape[0]
        hphi = idft_explicit(O.gauss_hat(s.sigma_F, R, Nfr))
        Q = (circ_matrix(hphi) @ P).real
        return Q[[q * 2 ** (s.log2F - k) for q in range(s.lam_out)]]

    avg = prm.average_fr
    S2 = []
    U2maps = {}
    for pi, (kind, theta, a, b) in enumerate(s.paths):
        if kind in (O.SPIN, O.PSI_T_PHI_F):
            G = np.zeros((Nfr, Y2[a].shape[1]), complex)
            for i, lam in enumerate(s.adm[a]):
                G[lam] = Y2[a][i]
            if kind == O.SPIN:
                h, k = fr_taps("psi", b, theta), int(s.kf[b])
            else:
                h, k = fr_taps("phi", 0, 0), (s.log2F if avg else 0)
            Z = circ_matrix(h) @ G                                     # conv along lambda
            U2 = np.abs(Z[[r * 2 ** k for r in range(Nfr >> k)]])
            U2maps[pi] = (U2, k)
            P = time_pool(U2, s.k_alpha[a])
            S2.append(lam_pool(P, k) if avg else P[: s.n1])
        else:
            G = np.zeros((Nfr, N_pad // T))
            G[: s.n1] = Yphi
            if kind == O.PHI_T_PSI_F:
                k = int(s.kf[b])
                Z = circ_matrix(fr_taps("psi", b, +1)) @ G
                U2 = np.abs(Z[[r * 2 ** k for r in range(Nfr >> k)]])
                P = time_pool(U2, s.log2T)
                S2.append(lam_pool(P, k) if avg else P[: s.n1])
            else:
                k = s.log2F if avg else 0
                V = (circ_matrix(fr_taps("phi", 0, 0)) @ G).real
                V = V[[r * 2 ** k for r in range(s.lam_out)]]
                S2.append(V[:, frames])
    S2t = [time_pool(np.abs(Y2[a]), s.k_alpha[a]) for a in s.alphas]
    return dict(S0=S0, S1=S1, S2=np.array(S2), S2t=np.concatenate(S2t, axis=0), U2=U2maps)


CASES = [
    O.Params(N=2 ** 8, J=4, Q=4, J_fr=2, T=2 ** 4, F=4),
    O.Params(N=2 ** 8, J=4, Q=4, J_fr=2, T=2 ** 4, F=4, pad="periodic"),
    O.Params(N=2 ** 8, J=4, Q=3, J_fr=2, T=2 ** 5, F=2, average_fr=False),
    O.Params(N=2 ** 7, J=3, Q=2, J_fr=2, T=2 ** 3, F=2, Q2=2),
]


@pytest.mark.parametrize("prm", CASES, ids=lambda p: f"N{p.N}J{p.J}Q{p.Q}T{p.T}F{p.F}{p.pad[0]}{int(p.average_fr)}Q2{p.Q2}")
def test_oracle_equals_bruteforce(prm):
    rng = np.random.default_rng(prm.N + prm.Q)
    x = rng.standard_normal(prm.N)
    s = O.schedule(prm)
    assert len(s.alphas) >= 2 and len(s.paths) > 4
    a = O.jtfs_forward(x, prm)
    b = brute_jtfs(x, prm)
    for key in ("S0", "S1", "S2"):
        ref = b[key]
        err = np.max(np.abs(a[key] - ref)) / np.max(np.abs(ref))
        assert err < 1e-11, (key, err)


@pytest.mark.parametrize("prm", CASES[:2] + CASES[3:], ids=lambda p: f"N{p.N}J{p.J}Q{p.Q}{p.pad[0]}Q2{p.Q2}")
def test_time_scattering_equals_bruteforce(prm):
    # Scattering1D second order (NEXT-2): |U1 * psi_alpha| * phi_T, no lambda convolution
    rng = np.random.default_rng(prm.N + 7)
    x = rng.standard_normal(prm.N)
    a = O.time_scattering(x, prm)
    b = brute_jtfs(x, prm)
    s = O.schedule(prm)
    assert a["S2"].shape == (sum(len(s.adm[al]) for al in s.alphas), s.n_frames)
    for key, ref in (("S0", b["S0"]), ("S1", b["S1"]), ("S2", b["S2t"])):
        err = np.max(np.abs(a[key] - ref)) / np.max(np.abs(ref))
        assert err < 1e-11, (key, err)


def test_dft_primitive_against_explicit_matrix():
    rng = np.random.default_rng(3)
    for L in (16, 64, 128, 96):
        v = rng.standard_normal(L) + 1j * rng.standard_normal(L)
        np.testing.assert_allclose(O._fft(v), dft_explicit(v), atol=1e-11)
        np.testing.assert_allclose(O._ifft(v), idft_explicit(v), atol=1e-13)


def test_reflect_pad_index_map():
    prm = O.Params(N=2 ** 6, J=3, Q=2, J_fr=1, T=2 ** 2, F=2)
    s = O.schedule(prm)
    x = np.arange(prm.N, dtype=float) + 1
    xp = O.pad_signal(x, s)
    ref = np.array([x[reflect_index(p, s.pad_left, prm.N)] for p in range(s.N_pad)])
    np.testing.assert_array_equal(xp, ref)


@pytest.mark.parametrize("prm", CASES[:3], ids=lambda p: f"N{p.N}J{p.J}Q{p.Q}{p.pad[0]}{int(p.average_fr)}")
def test_u2_map_equals_bruteforce(prm):
    # NEXT-4 scale-rate map (Fig. 1): |X * Psi| before Phi, rows r' 2^k < n1,
    # columns of the unpadded signal on the alpha grid (reading R21)
    rng = np.random.default_rng(prm.N + 11)
    x = rng.standard_normal(prm.N)
    s = O.schedule(prm)
    b = brute_jtfs(x, prm)
    assert set(b["U2"]) == {pi for pi, pth in enumerate(s.paths) if pth[0] in (O.SPIN, O.PSI_T_PHI_F)}
    for pi, (U2, k) in b["U2"].items():
        a = s.paths[pi][2]
        ka = s.k_alpha[a]
        rows = len([r for r in range(s.N_fr >> k) if r * 2 ** k < s.n1])
        c0 = -(-s.pad_left // 2 ** ka)
        ref = U2[:rows, c0: c0 + -(-prm.N // 2 ** ka)]
        got = O.u2_map(x, prm, pi, s)
        assert got.shape == ref.shape == O.u2_map_shape(s, pi)
        assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref)), pi


def _textbook_fft(v, sign):
    """Iterative radix-2 decimation-in-time DFT sum_n v[n] e^{sign 2 pi i k n / L} (fp64),
    twiddles from exact integer range reduction: written independently of scipy / numpy.fft."""
    L = len(v)
    bits = L.bit_length() - 1
    idx = np.arange(L)
    rev = np.zeros(L, dtype=np.int64)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    a = np.asarray(v, dtype=np.complex128)[rev].copy()
    span = 1
    while span < L:
        k = np.arange(span)
        w = np.exp(sign * 2j * np.pi * k / (2 * span))
        a = a.reshape(-1, 2 * span)
        top, bot = a[:, :span].copy(), a[:, span:] * w
        a[:, :span] = top + bot
        a[:, span:] = top - bot
        a = a.reshape(-1)
        span *= 2
    return a


def test_dft_primitive_against_textbook_fft_every_length():
    # the oracle's DFT primitive (scipy.fft / pocketfft) against an independent textbook
    # radix-2 FFT at every power-of-two length the path uses (2^1 .. 2^18): pins the library
    # routine at the sizes where the explicit-matrix check (L <= 128) cannot reach
    rng = np.random.default_rng(12)
    for lg in range(1, 19):
        L = 2 ** lg
        v = rng.standard_normal(L) + 1j * rng.standard_normal(L)
        ref_f = _textbook_fft(v, -1)
        ref_i = _textbook_fft(v, +1) / L
        sc = np.linalg.norm(ref_f)
        assert np.linalg.norm(O._fft(v) - ref_f) <= 1e-13 * sc * lg, lg
        assert np.linalg.norm(O._ifft(v) - ref_i) <= 1e-13 * np.linalg.norm(ref_i) * lg, lg


def test_textbook_fft_against_explicit_matrix():
    # the textbook FFT itself, pinned to the definition on small lengths
    rng = np.random.default_rng(13)
    for L in (2, 8, 64, 256):
        v = rng.standard_normal(L) + 1j * rng.standard_normal(L)
        np.testing.assert_allclose(_textbook_fft(v, -1), dft_explicit(v), atol=1e-10)
