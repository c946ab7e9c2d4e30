"""Full-path parity at the benchmarked sizes: every S0,
S1 and S2 path of the GPU forward against the fp64 oracle, at the bench's launch
configuration (the GPU record comes from the same batched forward bench.py times).

  c3  BASELINE configs[2] (P:241 setting with T = 2^13): the bench's first 16 notes
      (seeds 1000-1015, glissandi at 1001 / 1011 / 1015) + the rising glissando 1021,
      out of the 256-note forward -- Eq. (3), spin
  c4  BASELINE configs[3]: one bird texture (seed 7), N = 2^17, J = 13, all 150 paths
  c2  BASELINE configs[1]: 256 chirps of the 16^3 grid (every 16th) out of the 4096-chirp
      forward, Eq. (4)
  §4.2 preset (P:241, 44 x 32 per path): 2 notes, all 173 paths
Bar: per-path floored relative L2 <= 1e-4 (tests/parity.py).
"""
import numpy as np
import pytest

from paper_2204_08269_b200 import signals

from . import oracle_pool
from .parity import TOL, path_blocks, path_errors, unfloored_errors

pytestmark = pytest.mark.gpu

C3 = dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
C4 = dict(N=2 ** 17, J=13, Q=16, J_fr=5, T=2 ** 13, F=4)
C2 = dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False)
P42 = dict(N=2 ** 16, J=13, Q=16, J_fr=6, T=2 ** 11, F=4)

C3_IDX = list(range(16)) + [21]          # indices into notes(256, seed0=1000)
C2_IDX = list(range(0, 4096, 16))        # 256 of the 16^3 grid


@pytest.fixture(scope="module")
def inputs():
    return dict(c3=signals.notes(256, seed0=1000), c4=signals.bird_texture(seed=7)[None, :].copy(),
                c2=signals.chirp_grid()[1], p42=signals.notes(2, seed0=2000))


@pytest.fixture(scope="module")
def futures(inputs):
    """Every oracle job of this module, submitted at once (the slow c4 job first)."""
    f = {"c4": [oracle_pool.submit(C4, inputs["c4"][0])]}
    f["c3"] = [oracle_pool.submit(C3, inputs["c3"][i]) for i in C3_IDX]
    f["p42"] = [oracle_pool.submit(P42, inputs["p42"][i]) for i in range(2)]
    f["c2"] = [oracle_pool.submit(C2, inputs["c2"][i]) for i in C2_IDX]
    return f


@pytest.fixture(scope="module")
def jt():
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    return jtfs


def _gpu(jt, kw, X, flags=0):
    import torch
    plan = jt.Plan(**kw, flags=flags)
    out = plan.forward(torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda())
    torch.cuda.synchronize()
    return plan, out.cpu().numpy().astype(np.float64)


def _check(plan, rows, futs, name):
    worst, worst_unf, n_paths = 0.0, 0.0, 0
    for row, fu in zip(rows, futs):
        S0, S1, S2 = fu.result()
        g = path_blocks(*plan.unpack(row))
        o = path_blocks(S0, S1, S2)
        e = path_errors(g, o)
        worst = max(worst, float(e.max()))
        worst_unf = max(worst_unf, float(unfloored_errors(g, o).max()))
        n_paths = len(o)
        assert e.max() <= TOL, (name, float(e.max()), int(np.argmax(e)))
    print(f"\n{name}: {len(rows)} signals x {n_paths} paths, max floored e = {worst:.2e}, "
          f"max un-floored e (paths above the floor) = {worst_unf:.2e}")


def test_c3_all_paths_17_notes(jt, inputs, futures):
    plan, out = _gpu(jt, C3, inputs["c3"])          # the bench's 256-note launch
    _check(plan, out[C3_IDX], futures["c3"], "c3")


def test_c4_bird_texture_all_paths(jt, inputs, futures):
    plan, out = _gpu(jt, C4, inputs["c4"], flags=jt.JTFS_LATENCY)   # bench --workload c4 plan
    _check(plan, out, futures["c4"], "c4")


def test_c2_256_grid_chirps_all_paths(jt, inputs, futures):
    plan, out = _gpu(jt, C2, inputs["c2"])          # the bench's 4096-chirp launch
    _check(plan, out[C2_IDX], futures["c2"], "c2")


def test_paper_preset_all_paths(jt, inputs, futures):
    plan, out = _gpu(jt, P42, inputs["p42"])
    assert (plan.layout.lambda_out, plan.layout.n_frames) == (44, 32)
    _check(plan, out, futures["p42"], "sec4.2 preset")
