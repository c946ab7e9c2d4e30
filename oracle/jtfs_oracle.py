"""Plain, slow fp64 oracle of the forward joint time-frequency scattering (JTFS).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, smoke() and
bench.py's CPU-baseline legs may use it.  It shares no code with the CUDA path.

What it computes (PAPER.md = "P:<line>"):
  * scalogram X(t, lambda) = |x * psi_lambda| (Sec. 2), critically
    subsampled per centre frequency;
  * Eq. (1): psi_alpha(t) = 2^a psi(2^a t), psi_{beta,theta}(lambda)
    = 2^b psi(theta 2^b lambda);
  * Eq. (2): separable joint wavelet Psi = psi_alpha(t) psi_beta(lambda);
  * Eq. (3): S2 = | X *_{t,lambda} Psi | *_{t,lambda} Phi_{T,F};
  * Eq. (4): the same without frequential averaging;
  * first-order S1 = U1 * phi_T, no Phi_F, out_3D layout;
  * the phi-only lowpass paths (north_star; readings R11 of DESIGN.md);
  * second-order time scattering (Scattering1D; `time_scattering`).
Everything the paper leaves unstated (filter constants, ladder, subsampling
rule, padding, admissibility, lambda-axis boundary, spin orientation, path
order) follows the readings R1-R20 of DESIGN.md §3 (= SURVEY.md §8(c)).

Every convolution is written the plain way: DFT on the stated grid, multiply
by the sampled filter, inverse DFT at full rate, THEN decimate by indexing.
No folding, no truncation, no blocking.  scipy.fft (pocketfft, fp64) is the
DFT library primitive; tests pin it against an explicit DFT matrix (L <= 128) and
against an independent textbook radix-2 FFT at every length 2^1 .. 2^18.

Pinned by tests/test_oracle_*.py (closed forms, the paper's 44 x 32 shape,
brute-force time-domain convolution at tiny N, exact invariants, Fig. 1 spin
selectivity).  Parity unpinned: the absolute coefficient values of S2 beyond
these (the paper prints none) -- see DESIGN.md §3.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.fft as sfft

# --- constants of the filter generator G(J', Q')  (reading R2) ---
SIGMA0 = 0.1                   # lowpass width constant: sigma_phi = SIGMA0 / T
R_PSI = 1.0 / math.sqrt(2.0)   # adjacent-filter crossing amplitude (~ -3 dB)
ALPHA_C = 5.0                  # support multiplier in the critical-rate rule (R5)

_WORKERS = 1


def set_workers(n: int) -> None:
    """Threads used by the DFT primitive (scipy.fft workers)."""
    global _WORKERS
    _WORKERS = max(1, int(n))


def _fft(a, axis=-1):
    return sfft.fft(a, axis=axis, workers=_WORKERS)


def _ifft(a, axis=-1):
    return sfft.ifft(a, axis=axis, workers=_WORKERS)


# ----------------------------------------------------------------------------
# Filters  (P:67-70 Morlet / "Q filters per octave", P:88 Gaussian Phi)
# ----------------------------------------------------------------------------
def xi_max(Q: int) -> float:
    """Highest centre frequency of G(J', Q') in cycles/sample (reading R2)."""
    return max(1.0 / (1.0 + 2.0 ** (3.0 / Q)), 0.35)


def sigma_ratio(Q: int) -> float:
    """sigma / xi in the constant-Q region: neighbours cross at amplitude R_PSI."""
    q = 2.0 ** (-1.0 / Q)
    return (1.0 - q) / (1.0 + q) / math.sqrt(2.0 * math.log(1.0 / R_PSI))


def dyadic_j(xi: float, sigma: float) -> int:
    """Critical subsampling exponent j = floor(-log2 min(xi + 5 sigma, 1/2)) - 1 >= 0
    (reading R5: "the critical sample rate should depend on centre frequency")."""
    return max(int(math.floor(-math.log2(min(xi + ALPHA_C * sigma, 0.5)))) - 1, 0)


def morlet_bank(J: int, Q: int):
    """G(J, Q): lists (xi, sigma, j) ordered by decreasing xi (reading R2).

    Constant-Q ladder xi_i = xi_max 2^{-i/Q}, sigma_i = c xi_i while
    sigma_i > sigma0 / 2^J, then Q-1 linearly spaced tail filters at sigma_min.
    """
    xm, c, smin = xi_max(Q), sigma_ratio(Q), SIGMA0 / 2.0 ** J
    xis, sigmas = [], []
    i = 0
    while True:
        xi = xm * 2.0 ** (-i / Q)
        s = c * xi
        if not s > smin:
            break
        xis.append(xi)
        sigmas.append(s)
        i += 1
    if not xis:
        raise ValueError(f"G({J},{Q}) has no constant-Q filter")
    xi_last = xis[-1]
    for q in range(1, Q):
        xis.append((Q - q) / Q * xi_last)
        sigmas.append(smin)
    js = [dyadic_j(x, s) for x, s in zip(xis, sigmas)]
    return np.array(xis), np.array(sigmas), np.array(js, dtype=np.int64)


def _grid_freqs(L: int, n_grid: int):
    """Bin m of a length-L grid <-> physical frequency (reading R8):
    one-sided w+ = m / n_grid (m in [0, L)); two-sided w+- = fftfreq."""
    m = np.arange(L, dtype=np.float64)
    w_plus = m / n_grid
    w_pm = np.where(m < L / 2, m, m - L) / n_grid
    return w_plus, w_pm


def morlet_hat(xi: float, sigma: float, L: int, n_grid: int) -> np.ndarray:
    """Sampled Morlet spectrum (reading R1): Gabor bump at xi on the one-sided
    grid minus kappa * Gaussian at DC, kappa chosen so psi_hat[0] = 0 exactly."""
    w_plus, w_pm = _grid_freqs(L, n_grid)
    gabor = np.exp(-((w_plus - xi) ** 2) / (2.0 * sigma * sigma))
    kappa = gabor[0]          # = exp(-xi^2 / (2 sigma^2)), the same rounding as bin 0
    return gabor - kappa * np.exp(-(w_pm ** 2) / (2.0 * sigma * sigma))


def gauss_hat(sigma: float, L: int, n_grid: int) -> np.ndarray:
    """Sampled Gaussian lowpass spectrum phi_hat, phi_hat[0] = 1 (reading R4)."""
    _, w_pm = _grid_freqs(L, n_grid)
    return np.exp(-(w_pm ** 2) / (2.0 * sigma * sigma))


# ----------------------------------------------------------------------------
# Parameters and the derived schedule
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Params:
    """Operator parameters (Sec. 4.2; Sec. 3.3; reading R12/R14).

    N: signal length (pow2); J: octaves; Q: first-order filters per octave;
    J_fr, Q_fr: frequential bank; T: temporal lowpass support (pow2);
    F: frequential lowpass support (pow2; 0 -> 2^J_fr); Q2: second-order Q;
    average_fr: True = Eq. (3), False = Eq. (4); pad: 'reflect' | 'periodic'.
    """
    N: int
    J: int
    Q: int
    J_fr: int
    T: int
    F: int = 0
    Q2: int = 1
    Q_fr: int = 1
    average_fr: bool = True
    pad: str = "reflect"


def _ilog2(v: int) -> int:
    if v < 1 or v & (v - 1):
        raise ValueError(f"{v} is not a power of two")
    return v.bit_length() - 1


@dataclass
class Schedule:
    p: Params
    N_pad: int = 0
    pad_left: int = 0
    log2T: int = 0
    F: int = 0
    log2F: int = 0
    xi1: np.ndarray = field(default=None)
    sigma1: np.ndarray = field(default=None)
    j1: np.ndarray = field(default=None)
    k1: np.ndarray = field(default=None)
    n1: int = 0
    xi2: np.ndarray = field(default=None)
    sigma2: np.ndarray = field(default=None)
    j2: np.ndarray = field(default=None)
    alphas: list = field(default_factory=list)       # active alpha indices into bank 2
    adm: dict = field(default_factory=dict)          # alpha -> admissible lambda list
    k_alpha: dict = field(default_factory=dict)
    xif: np.ndarray = field(default=None)
    sigmaf: np.ndarray = field(default=None)
    jf: np.ndarray = field(default=None)
    kf: np.ndarray = field(default=None)
    N_fr: int = 0
    frame0: int = 0
    n_frames: int = 0
    lam_out: int = 0
    paths: list = field(default_factory=list)        # (kind, theta, alpha, beta)

    @property
    def sigma_T(self) -> float:
        return SIGMA0 / self.p.T

    @property
    def sigma_F(self) -> float:
        return SIGMA0 / self.F


# path kinds (reading R11, order R-O11)
SPIN, PSI_T_PHI_F, PHI_T_PSI_F, PHI_T_PHI_F = 0, 1, 2, 3


def schedule(p: Params) -> Schedule:
    """All derived quantities of the operator (readings R2, R5-R7, R9, R12)."""
    s = Schedule(p=p)
    log2N = _ilog2(p.N)
    s.log2T = _ilog2(p.T)
    if p.T > p.N or 2 ** p.J > p.N or p.J < 1 or p.Q < 1 or p.J_fr < 1:
        raise ValueError("invalid parameters")
    s.F = p.F if p.F else 2 ** p.J_fr
    s.log2F = _ilog2(s.F)
    if p.pad == "reflect":
        s.N_pad, s.pad_left = 2 * p.N, p.N // 2
    elif p.pad == "periodic":
        s.N_pad, s.pad_left = p.N, 0
    else:
        raise ValueError(p.pad)
    del log2N
    s.xi1, s.sigma1, s.j1 = morlet_bank(p.J, p.Q)
    s.n1 = len(s.xi1)
    if s.n1 < 4:
        raise ValueError("n1 < 4")
    s.k1 = np.minimum(s.j1, s.log2T)
    s.xi2, s.sigma2, s.j2 = morlet_bank(p.J, p.Q2)
    for a in range(len(s.xi2)):
        A = [lam for lam in range(s.n1) if s.j1[lam] < s.j2[a]]
        if A:                                   # alphas with empty A(alpha) are dropped
            s.alphas.append(a)
            s.adm[a] = A
            s.k_alpha[a] = int(min(s.j2[a], s.log2T))
    s.xif, s.sigmaf, s.jf = morlet_bank(p.J_fr, p.Q_fr)
    s.kf = (np.minimum(s.jf, s.log2F) if p.average_fr
            else np.zeros_like(s.jf))
    s.N_fr = 2 ** ((s.n1 - 1).bit_length() + 1)    # 2^(ceil(log2 n1) + 1)
    if s.F > s.N_fr:
        raise ValueError("F larger than the frequential grid")
    s.frame0 = -(-s.pad_left // p.T)               # U(k) = [ceil(pad_left/2^k), +ceil(N/2^k))
    s.n_frames = -(-p.N // p.T)
    s.lam_out = -(-s.n1 // s.F) if p.average_fr else s.n1
    nb = len(s.xif)
    for theta in (-1, +1):
        for a in s.alphas:
            for b in range(nb):
                s.paths.append((SPIN, theta, a, b))
    for a in s.alphas:
        s.paths.append((PSI_T_PHI_F, 0, a, -1))
    for b in range(nb):
        s.paths.append((PHI_T_PSI_F, 0, -1, b))
    s.paths.append((PHI_T_PHI_F, 0, -1, -1))
    return s


# ----------------------------------------------------------------------------
# Pieces of the forward operator
# ----------------------------------------------------------------------------
def pad_signal(x: np.ndarray, s: Schedule) -> np.ndarray:
    """O1: numpy 'reflect' padding to N_pad = 2N, centred (reading R6)."""
    if s.p.pad == "periodic":
        return x.astype(np.float64)
    right = s.N_pad - s.p.N - s.pad_left
    return np.pad(x.astype(np.float64), (s.pad_left, right), mode="reflect")


def time_frames(s: Schedule) -> np.ndarray:
    """Retained output frames m in U(log2 T)."""
    return np.arange(s.frame0, s.frame0 + s.n_frames)


def phi_T_pool(rows: np.ndarray, k: int, s: Schedule) -> np.ndarray:
    """O9 (time): rows (..., L) at exponent k -> IDFT_L(DFT_L(row) phi_T^(L))
    sampled at m 2^(log2T - k), m in U(log2 T).  (Phi_T of Eq. (3)/(4).)"""
    L = rows.shape[-1]
    ph = gauss_hat(s.sigma_T, L, s.N_pad)
    full = _ifft(_fft(rows, axis=-1) * ph, axis=-1).real
    return full[..., time_frames(s) * 2 ** (s.log2T - k)]


def phi_F_pool(cols: np.ndarray, k: int, s: Schedule) -> np.ndarray:
    """O9 (log-frequency, Eq. (3) only): rows axis 0 of length R = N_fr / 2^k ->
    IDFT_R(DFT_R(col) phi_F^(R)) sampled at q 2^(log2F - k), q < ceil(n1/F)."""
    R = cols.shape[0]
    ph = gauss_hat(s.sigma_F, R, s.N_fr)
    full = _ifft(_fft(cols, axis=0) * ph[:, None], axis=0).real
    return full[np.arange(s.lam_out) * 2 ** (s.log2F - k)]


def first_order(x: np.ndarray, s: Schedule):
    """O1-O6.  Returns S0 (frames), S1 (n1, frames), Yphi (n1, N_pad/T),
    U1hat (list per lambda), Y2 (dict alpha -> (K_alpha, L_alpha) complex)."""
    xp = pad_signal(x, s)
    X = _fft(xp)                                                     # O2
    N_pad, T = s.N_pad, s.p.T
    # O3  S0[m] = IDFT(X phi_T)[m T]
    S0 = _ifft(X * gauss_hat(s.sigma_T, N_pad, N_pad)).real[time_frames(s) * T]
    S1 = np.zeros((s.n1, s.n_frames))
    Yphi = np.zeros((s.n1, N_pad // T))
    U1hat = []
    for lam in range(s.n1):
        k1 = int(s.k1[lam])
        psi = morlet_hat(s.xi1[lam], s.sigma1[lam], N_pad, N_pad)
        U1 = np.abs(_ifft(X * psi))[:: 2 ** k1]                       # O4 scalogram row
        Uh = _fft(U1)                                                # O5
        U1hat.append(Uh)
        L1 = N_pad >> k1
        smooth = _ifft(Uh * gauss_hat(s.sigma_T, L1, N_pad)).real
        d = 2 ** (s.log2T - k1)
        S1[lam] = smooth[time_frames(s) * d]
        Yphi[lam] = smooth[np.arange(N_pad // T) * d]
    Y2 = {}
    for a in s.alphas:                                               # O6
        ka = s.k_alpha[a]
        rows = []
        for lam in s.adm[a]:
            k1 = int(s.k1[lam])
            L1 = N_pad >> k1
            psi_a = morlet_hat(s.xi2[a], s.sigma2[a], L1, N_pad)
            rows.append(_ifft(U1hat[lam] * psi_a)[:: 2 ** (ka - k1)])
        Y2[a] = np.array(rows)
    return S0, S1, Yphi, U1hat, Y2


def psi_fr_hat(b: int, theta: int, s: Schedule) -> np.ndarray:
    """Frequential wavelet psi_{beta,theta} on the N_fr grid (reading R10):
    theta = -1 <-> psi_hat[m] (analytic along the DESCENDING row axis),
    theta = +1 <-> psi_hat[(-m) mod N_fr]."""
    h = morlet_hat(s.xif[b], s.sigmaf[b], s.N_fr, s.N_fr)
    if theta == +1:
        h = h[(-np.arange(s.N_fr)) % s.N_fr]
    return h


def _grid(rows_by_lambda: dict, width: int, s: Schedule, dtype) -> np.ndarray:
    """Zero-padded circular lambda grid of N_fr rows (reading R9)."""
    G = np.zeros((s.N_fr, width), dtype=dtype)
    for lam, row in rows_by_lambda.items():
        G[lam] = row
    return G


def joint_stage(Y2: dict, Yphi: np.ndarray, s: Schedule, paths=None) -> dict:
    """O7-O9: frequential wavelet transform along lambda, modulus, Phi_{T,F}.

    Y2: alpha -> array (len(adm[alpha]), L_alpha); Yphi: (n1, N_pad/T).
    Returns {path_index: (lam_out, n_frames)} for the requested paths."""
    want = set(range(len(s.paths))) if paths is None else set(paths)
    out = {}
    avg = s.p.average_fr
    by_alpha = {}
    for pi, (kind, theta, a, b) in enumerate(s.paths):
        if pi in want and kind in (SPIN, PSI_T_PHI_F):
            by_alpha.setdefault(a, []).append(pi)
    for a, pis in by_alpha.items():
        ka = s.k_alpha[a]
        G = _grid(dict(zip(s.adm[a], Y2[a])), Y2[a].shape[1], s, np.complex128)
        g = _fft(G, axis=0)                                          # O7 DFT along lambda
        for pi in pis:
            kind, theta, _, b = s.paths[pi]
            if kind == SPIN:
                fh, k = psi_fr_hat(b, theta, s), int(s.kf[b])
            else:
                fh, k = gauss_hat(s.sigma_F, s.N_fr, s.N_fr), (s.log2F if avg else 0)
            U2 = np.abs(_ifft(g * fh[:, None], axis=0))[:: 2 ** k]   # |X * Psi|
            P = phi_T_pool(U2, ka, s)                                # O9 time
            out[pi] = phi_F_pool(P, k, s) if avg else P[: s.n1]      # O9 lambda
    phi_pis = [pi for pi in want if s.paths[pi][0] in (PHI_T_PSI_F, PHI_T_PHI_F)]
    if phi_pis:
        G = _grid({lam: Yphi[lam] for lam in range(s.n1)}, Yphi.shape[1], s, np.float64)
        g = _fft(G, axis=0)
        for pi in phi_pis:
            kind, _, _, b = s.paths[pi]
            if kind == PHI_T_PSI_F:                                  # O8: spin +1 only
                k = int(s.kf[b])
                U2 = np.abs(_ifft(g * psi_fr_hat(b, +1, s)[:, None], axis=0))[:: 2 ** k]
                P = phi_T_pool(U2, s.log2T, s)
                out[pi] = phi_F_pool(P, k, s) if avg else P[: s.n1]
            else:                                                    # phi_t x phi_f: no modulus
                k = s.log2F if avg else 0
                V = _ifft(g * gauss_hat(s.sigma_F, s.N_fr, s.N_fr)[:, None], axis=0).real
                V = V[:: 2 ** k][: s.lam_out]
                out[pi] = V[:, time_frames(s)]
    return out


def jtfs_forward(x: np.ndarray, p: Params, paths=None, s: Schedule | None = None):
    """Forward JTFS of one signal x (N,) in fp64.

    Returns dict(S0=(frames,), S1=(n1, frames), S2=(P, lam_out, frames)).
    With `paths` (indices into schedule(p).paths) only those S2 maps are
    computed; the others are NaN."""
    s = s or schedule(p)
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (p.N,):
        raise ValueError(f"x must have shape ({p.N},)")
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite input")
    S0, S1, Yphi, _, Y2 = first_order(x, s)
    maps = joint_stage(Y2, Yphi, s, paths)
    S2 = np.full((len(s.paths), s.lam_out, s.n_frames), np.nan)
    for pi, m in maps.items():
        S2[pi] = m
    return dict(S0=S0, S1=S1, S2=S2)


def time_scattering(x: np.ndarray, p: Params, s: Schedule | None = None):
    """Second-order time scattering (Scattering1D): "applying only a
    1-D temporal wavelet filterbank to the first-order scalogram",
    i.e. S2_t[lambda, alpha] = (|U1_lambda * psi_alpha| * phi_T) at the retained
    frames, without any convolution along lambda (compare Eq. (3)).

    Readings: the same banks, critical subsampling (R5), padding
    (R6) and admissible pairs j1(lambda) < j2(alpha) (R7) as the JTFS of Eq. (3),
    so |U1 * psi_alpha| is |Y2_alpha| of first_order(); rows ordered alpha-major
    then lambda (schedule order).  Returns dict(S0=(frames,), S1=(n1, frames),
    S2=(n2, frames)) with n2 = sum_alpha |adm(alpha)|."""
    s = s or schedule(p)
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (p.N,):
        raise ValueError(f"x must have shape ({p.N},)")
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite input")
    S0, S1, _, _, Y2 = first_order(x, s)
    rows = [phi_T_pool(np.abs(Y2[a]), s.k_alpha[a], s) for a in s.alphas]
    S2 = np.concatenate(rows, axis=0) if rows else np.zeros((0, s.n_frames))
    return dict(S0=S0, S1=S1, S2=S2)


def unpack_layout(s: Schedule):
    """Offsets of the packed out_3D record: [S0 | S1 (n1 x fr) | S2 (P x lam_out x fr)]."""
    fr = s.n_frames
    o_s1 = fr
    o_s2 = o_s1 + s.n1 * fr
    total = o_s2 + len(s.paths) * s.lam_out * fr
    return dict(S0=0, S1=o_s1, S2=o_s2, total=total)


def pack(res: dict) -> np.ndarray:
    """O12: out_3D flattened row-major (reading R-O11/O12)."""
    return np.concatenate([res["S0"].ravel(), res["S1"].ravel(), res["S2"].ravel()])


# ----------------------------------------------------------------------------
# NEXT-4: scale-rate map export and mu-log compression
# ----------------------------------------------------------------------------
def u2_map_shape(s: Schedule, pi: int):
    """(rows, cols) of u2_map for path pi (a SPIN or PSI_T_PHI_F path)."""
    kind, _, a, b = s.paths[pi]
    if kind == SPIN:
        k = int(s.kf[b])
    elif kind == PSI_T_PHI_F:
        k = s.log2F if s.p.average_fr else 0
    else:
        raise ValueError("u2_map exists only for the psi_t paths (spinned, psi_t x phi_f)")
    ka = s.k_alpha[a]
    return -(-s.n1 // 2 ** k), -(-s.p.N // 2 ** ka)


def u2_map(x: np.ndarray, p: Params, pi: int, s: Schedule | None = None) -> np.ndarray:
    """Scale-rate visualisation of Fig. 1: |X * Psi_{alpha,beta,theta}|,
    the joint wavelet modulus BEFORE the lowpass Phi (Eq. (3) without its last
    convolution), on the whole time and log-frequency axes.

    Readings (R21): the map is U2 of step O7 on its critical grid --
    rows r' of the lambda axis decimated by 2^k (k = k_f(beta) in Eq. (3) mode,
    log2 F for psi_t x phi_f, 0 in Eq. (4) mode), restricted to the rows over the
    scalogram, r' 2^k < n1; columns n of the alpha grid (exponent k_alpha)
    restricted to the unpadded signal, n in U(k_alpha) = [ceil(pad_left / 2^k_alpha),
    + ceil(N / 2^k_alpha)).  Returns float64 (rows, cols)."""
    s = s or schedule(p)
    rows, cols = u2_map_shape(s, pi)
    kind, theta, a, b = s.paths[pi]
    x = np.asarray(x, dtype=np.float64)
    _, _, _, _, Y2 = first_order(x, s)
    G = _grid(dict(zip(s.adm[a], Y2[a])), Y2[a].shape[1], s, np.complex128)
    if kind == SPIN:
        fh, k = psi_fr_hat(b, theta, s), int(s.kf[b])
    else:
        fh, k = gauss_hat(s.sigma_F, s.N_fr, s.N_fr), (s.log2F if s.p.average_fr else 0)
    U2 = np.abs(_ifft(_fft(G, axis=0) * fh[:, None], axis=0))[:: 2 ** k]   # O7, |X * Psi|
    c0 = -(-s.pad_left // 2 ** s.k_alpha[a])
    return U2[:rows, c0: c0 + cols]


def mulog_mu(S2: np.ndarray) -> np.ndarray:
    """Eq. (adalog:mu): mu(lambda_2) = (1/N) sum_n iint S x_n(lambda_2,
    lambda, t) dt dlambda over a set of N examples; the integral over the sampled
    (lambda, t) grid is the sum of the map.  S2: (B, P, lam_out, frames)."""
    S2 = np.asarray(S2, dtype=np.float64)
    return S2.sum(axis=(2, 3)).sum(axis=0) / S2.shape[0]


def mulog(S2: np.ndarray, mu: np.ndarray, eps: float = 0.1) -> np.ndarray:
    """Eq. (adalog): S~(lambda_2, lambda, t) = log(1 + S / (eps mu(lambda_2))),
    eps = 0.1 per path.  Reading R22: applied to every second-order map
    lambda_2 (the S2 paths); S0 / S1 are left as they are (the convnet
    treats first order separately).  A path with mu = 0 (all-zero maps) maps to 0."""
    S2 = np.asarray(S2, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    den = eps * mu[None, :, None, None]
    safe = np.where(den > 0, den, 1.0)
    return np.where(den > 0, np.log1p(S2 / safe), 0.0)
