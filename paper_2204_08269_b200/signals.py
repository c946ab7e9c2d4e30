"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY code shared by the oracle-side tests and the GPU path:
it holds input recipes and none of the JTFS arithmetic.

* ``am_chirp``    -- Eq. (5) AM/FM exponential chirp (Sec. 3.2);
* ``chirp_grid``  -- the 16^3 geometric grid of (f_c, f_m, gamma);
* ``notes``       -- instrument-like notes (Medley-solos-DB shaped);
* ``bird_texture``-- bird-call-like texture (Fig. 1 c/d, Sec. 5);
* ``white``       -- N(0, 1) noise (throughput sweep).
All return float32 arrays; the same array feeds the oracle and the GPU.
"""
from __future__ import annotations

import numpy as np


def am_chirp(N: int, fs: float, f_c: float, f_m: float, gamma: float,
             w: float = 2.0) -> np.ndarray:
    """Eq. (5): g(t) = phi_w(gamma t) sin(2 pi f_m t) sin(2 pi f_c / (gamma ln 2) 2^{gamma t}).

    phi_w(u) = exp(-u^2 / (2 (w/4)^2)) (reading R17), t = 0 at mid-signal;
    instantaneous frequency f_c 2^{gamma t}, essential duration w / gamma."""
    t = (np.arange(N) - N / 2) / fs
    env = np.exp(-((gamma * t) ** 2) / (2.0 * (w / 4.0) ** 2))
    car = np.sin(2 * np.pi * f_c / (gamma * np.log(2.0)) * 2.0 ** (gamma * t))
    return (env * np.sin(2 * np.pi * f_m * t) * car).astype(np.float32)


def chirp_grid(N: int = 2 ** 13, fs: float = 8192.0, n: int = 16):
    """Eq. (5) over the geometric 16^3 grid: f_c 512..1024 Hz,
    f_m 4..32 Hz, gamma 0.5..4 oct/s; f_c-major order.  Deterministic."""
    fc = 512.0 * 2.0 ** (np.arange(n) / (n - 1))
    fm = 4.0 * 8.0 ** (np.arange(n) / (n - 1))
    gm = 0.5 * 8.0 ** (np.arange(n) / (n - 1))
    params, sig = [], []
    for a in fc:
        for b in fm:
            for c in gm:
                params.append((a, b, c))
                sig.append(am_chirp(N, fs, a, b, c))
    return np.array(params), np.stack(sig)


def _pink(rng, N):
    spec = rng.standard_normal(N // 2 + 1) + 1j * rng.standard_normal(N // 2 + 1)
    f = np.arange(N // 2 + 1, dtype=np.float64)
    f[0] = 1.0
    y = np.fft.irfft(spec / np.sqrt(f), n=N)
    return y / (np.sqrt(np.mean(y ** 2)) + 1e-30)


def note(N: int = 2 ** 16, fs: float = 22050.0, seed: int = 1000) -> np.ndarray:
    """One synthetic instrument note: harmonic series with 1/h e^{-bh} roll-off,
    ADSR envelope, vibrato, 20 % glissandi (Fig. 1b), -40 dB pink noise, peak 0.9."""
    rng = np.random.default_rng(seed)
    t = np.arange(N) / fs
    f0 = 55.0 * 32.0 ** rng.uniform()
    b = rng.uniform(0.0, 0.3)
    nh = int(max(1, min(20, np.floor(0.45 * fs / f0))))
    vib_f, vib_c = rng.uniform(4, 7), rng.uniform(0, 30)
    gliss = rng.uniform(-1, 1) if rng.uniform() < 0.2 else 0.0
    inst = f0 * 2.0 ** (gliss * t + vib_c / 1200.0 * np.sin(2 * np.pi * vib_f * t))
    phase = 2 * np.pi * np.cumsum(inst) / fs
    y = np.zeros(N)
    for h in range(1, nh + 1):
        ok = (h * inst) < 0.45 * fs
        y += ok * np.sin(h * phase + rng.uniform(0, 2 * np.pi)) / h * np.exp(-b * h)
    att, rel = rng.uniform(0.01, 0.1), rng.uniform(0.1, 0.5)
    dur = N / fs
    env = np.clip(t / att, 0, 1) * np.clip((dur - t) / rel, 0, 1) * (0.7 + 0.3 * np.exp(-3 * t))
    y = y * env
    y = y / (np.max(np.abs(y)) + 1e-30)
    y = y + 0.01 * _pink(rng, N)
    return (0.9 * y / np.max(np.abs(y))).astype(np.float32)


def note_glissando(seed: int) -> float:
    """The glissando rate (octaves/s, 0 = none) that note(seed=seed) draws -- the same
    draws in the same order as note(), so tests can pick glissandi (Fig. 1b)."""
    rng = np.random.default_rng(seed)
    rng.uniform(), rng.uniform(), rng.uniform(4, 7), rng.uniform(0, 30)
    return rng.uniform(-1, 1) if rng.uniform() < 0.2 else 0.0


def notes(B: int, N: int = 2 ** 16, fs: float = 22050.0, seed0: int = 1000) -> np.ndarray:
    """Config c3 batch: seeds seed0 + i."""
    return np.stack([note(N, fs, seed0 + i) for i in range(B)])


def bird_texture(N: int = 2 ** 17, fs: float = 22050.0, seed: int = 7) -> np.ndarray:
    """Config c4: 10-14 calls of 50-300 ms, up/down FM sweeps 2->6 kHz with 2-3
    partials, 20-60 Hz AM, random onsets, -30 dB noise."""
    rng = np.random.default_rng(seed)
    y = np.zeros(N)
    for _ in range(rng.integers(10, 15)):
        L = int(rng.uniform(0.05, 0.3) * fs)
        on = rng.integers(0, N - L)
        tt = np.arange(L) / fs
        f_a, f_b = rng.uniform(2000, 6000, size=2)
        inst = f_a + (f_b - f_a) * tt / tt[-1]
        ph = 2 * np.pi * np.cumsum(inst) / fs
        am = 0.5 * (1 + np.sin(2 * np.pi * rng.uniform(20, 60) * tt))
        win = np.sin(np.pi * np.arange(L) / L) ** 2
        call = sum(np.sin(k * ph) / k for k in range(1, rng.integers(2, 4) + 1)
                   if k * max(f_a, f_b) < 0.45 * fs)
        y[on:on + L] += win * am * call
    y = y / (np.max(np.abs(y)) + 1e-30)
    y = y + 10 ** (-30 / 20) * rng.standard_normal(N)
    return (0.9 * y / np.max(np.abs(y))).astype(np.float32)


def white(B: int, N: int, seed: int = 0) -> np.ndarray:
    """Config c5: white N(0, 1) float32."""
    return np.random.default_rng(seed).standard_normal((B, N)).astype(np.float32)
