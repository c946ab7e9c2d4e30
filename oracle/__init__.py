"""fp64 CPU oracle for the forward JTFS operator of arXiv 2204.08269.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library, its
Python binding, the multi-GPU driver) may import, call, link or execute this
package.  The only permitted callers are ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs.

The oracle shares no code with the GPU path: it is written from PAPER.md
Eqs. (1)-(4) and the readings listed in DESIGN.md §3 (taken from
SURVEY.md §8(c)), in plain numpy/scipy fp64, step by step.
"""
from .jtfs_oracle import (  # noqa: F401
    Params, Schedule, schedule, morlet_bank, morlet_hat, gauss_hat,
    jtfs_forward, pack, unpack_layout, set_workers, first_order, joint_stage,
)
