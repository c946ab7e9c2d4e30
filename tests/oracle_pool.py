"""Runs fp64 oracle forwards (oracle/jtfs_oracle.py) in a pool of single-threaded
worker processes, one signal per task, so the full-path parity tests at the bench's
sizes finish in minutes.  Test infrastructure only (the oracle never runs on the
product path)."""
from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np

_POOL = None


def _job(args):
    okw, x, paths = args
    from oracle import jtfs_oracle as O
    O.set_workers(1)
    r = O.jtfs_forward(np.asarray(x, dtype=np.float64), O.Params(**okw), paths=paths)
    return r["S0"], r["S1"], r["S2"]


def pool():
    global _POOL
    if _POOL is None:
        _POOL = cf.ProcessPoolExecutor(max_workers=max(1, os.cpu_count() or 1),
                                       mp_context=mp.get_context("spawn"))
    return _POOL


def submit(okw: dict, x, paths=None):
    """Future of (S0, S1, S2) of the oracle on one fp32 signal x (promoted to fp64)."""
    return pool().submit(_job, (dict(okw), np.asarray(x, dtype=np.float32), paths))
