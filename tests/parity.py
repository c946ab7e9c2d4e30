"""Per-path parity metric (fixed before any GPU measurement).

e_{b,p} = ||S_gpu - S_ora||_2 / max(||S_ora||_2, eta * RMS_p' ||S_ora_{b,p'}||_2),  eta = 1e-3
over paths p = S0, each S1 row, each S2 map.  Pass iff max e <= 1e-4.
The floor exists because fp32 roundoff from a signal's large paths (~1e-7 of
them) cannot be held to 1e-4 *relative* on paths 1e-4 times smaller.
"""
import numpy as np

TOL = 1e-4
ETA = 1e-3


def path_blocks(s0, s1, s2):
    """List of per-path arrays in output order for one signal."""
    return [np.asarray(s0)] + [np.asarray(r) for r in s1] + [np.asarray(m) for m in s2]


def path_errors(gpu_blocks, ora_blocks, paths=None):
    idx = range(len(ora_blocks)) if paths is None else paths
    norms = np.array([np.linalg.norm(ora_blocks[i]) for i in range(len(ora_blocks))
                      if np.all(np.isfinite(ora_blocks[i]))])
    floor = ETA * np.sqrt(np.mean(norms ** 2))
    errs = []
    for i in idx:
        o = np.asarray(ora_blocks[i], dtype=np.float64)
        g = np.asarray(gpu_blocks[i], dtype=np.float64)
        errs.append(np.linalg.norm(g - o) / max(np.linalg.norm(o), floor))
    return np.array(errs)
