"""Per-path parity metric (fixed before any GPU measurement).

e_{b,p} = ||S_gpu - S_ora||_2 / max(||S_ora||_2, eta * RMS_p' ||S_ora_{b,p'}||_2),  eta = 1e-3
over paths p = S0, each S1 row, each S2 map.  Pass iff max e <= 1e-4.
The floor exists because fp32 roundoff from a signal's large paths (~1e-7 of
them) cannot be held to 1e-4 *relative* on paths 1e-4 times smaller.
Blocks may be complex (stage taps such as Y2 rows): norms are taken of the complex
values, so the imaginary parts count.
"""
import numpy as np

TOL = 1e-4
ETA = 1e-3


def path_blocks(s0, s1, s2):
    """List of per-path arrays in output order for one signal."""
    return [np.asarray(s0)] + [np.asarray(r) for r in s1] + [np.asarray(m) for m in s2]


def _as64(a):
    a = np.asarray(a)
    return a.astype(np.complex128) if np.iscomplexobj(a) else a.astype(np.float64)


def path_errors(gpu_blocks, ora_blocks, paths=None):
    idx = range(len(ora_blocks)) if paths is None else paths
    norms = np.array([np.linalg.norm(_as64(ora_blocks[i])) for i in range(len(ora_blocks))
                      if np.all(np.isfinite(ora_blocks[i]))])
    floor = ETA * np.sqrt(np.mean(norms ** 2))
    errs = []
    for i in idx:
        o = _as64(ora_blocks[i])
        g = _as64(gpu_blocks[i])
        assert g.shape == o.shape, (i, g.shape, o.shape)
        errs.append(np.linalg.norm(g - o) / max(np.linalg.norm(o), floor))
    return np.array(errs)


def unfloored_errors(gpu_blocks, ora_blocks):
    """Plain relative errors of the paths ABOVE the floor ("also report
    un-floored errors for paths above the floor")."""
    norms = np.array([np.linalg.norm(_as64(b)) for b in ora_blocks])
    floor = ETA * np.sqrt(np.mean(norms ** 2))
    out = []
    for g, o, n in zip(gpu_blocks, ora_blocks, norms):
        if n > floor:
            out.append(np.linalg.norm(_as64(g) - _as64(o)) / n)
    return np.array(out)
