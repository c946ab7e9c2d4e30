"""Path-sharded forward (jtfs_forward_units / jtfs_reduce_pack) on the GPU.

The ranks of a path-sharded run are simulated in one process (one GPU runs each
rank's unit list in turn; the partial buffers are then summed as
shard.exchange_partials would): the result must be byte-identical to
jtfs_forward, for c3 (batch plan) and c4 (single long signal, JTFS_LATENCY),
and c4 must meet the parity bar against the fp64 oracle.
"""
import numpy as np
import pytest

from oracle import jtfs_oracle as O
from paper_2204_08269_b200 import shard, signals

from .parity import TOL, path_blocks, path_errors

pytestmark = pytest.mark.gpu

C3 = dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
C4 = dict(N=2 ** 17, J=13, Q=16, J_fr=5, T=2 ** 13, F=4)


@pytest.fixture(scope="module")
def jt():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a visible CUDA device")
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    return jtfs


def _sharded(plan, x, world):
    import torch
    units = plan.units()
    parts = shard.lpt_assign([u["cost"] for u in units], world)
    B = x.shape[0]
    total = torch.zeros(B, plan.partials_size, dtype=torch.float32, device="cuda")
    out = torch.empty(B, plan.floats_per_signal, dtype=torch.float32, device="cuda")
    for r in reversed(range(world)):            # rank 0 last: its workspace feeds reduce_pack
        p = torch.empty_like(total)
        o = torch.empty_like(out)
        plan.forward_units(x, parts[r], p, o)
        total += p                              # disjoint slices: exact
        if r == 0:
            out.copy_(o)
    plan.reduce_pack(total, out)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("world", [1, 3])
def test_c3_sharded_equals_forward(jt, world):
    import torch
    plan = jt.Plan(**C3)
    x = torch.from_numpy(signals.notes(2, seed0=1200)).cuda()
    ref = plan.forward(x).cpu().numpy()
    got = _sharded(plan, x, world).cpu().numpy()
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


def test_c4_single_long_signal_sharded(jt):
    import torch
    plan = jt.Plan(**C4, flags=jt.JTFS_LATENCY)
    X = signals.bird_texture(seed=7)[None, :]
    x = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda()
    ref = plan.forward(x)
    torch.cuda.synchronize()
    got = _sharded(plan, x, 8)
    assert np.array_equal(ref.cpu().numpy().view(np.uint32), got.cpu().numpy().view(np.uint32))
    # parity of the c4 forward against the oracle on a sample of paths
    prm = O.Params(**C4)
    s = O.schedule(prm)
    P = len(s.paths)
    sample = sorted({0, 7, 60, 66, P - 20, P - 8, P - 2, P - 1})
    O.set_workers(8)
    ora = O.jtfs_forward(X[0].astype(np.float64), prm, paths=sample, s=s)
    s0, s1, s2 = plan.unpack(got[0].cpu().numpy().astype(np.float64))
    n_first = 1 + s.n1
    sel = list(range(n_first)) + [n_first + p for p in sample]
    e = path_errors(path_blocks(s0, s1, s2), path_blocks(ora["S0"], ora["S1"], ora["S2"]), sel)
    assert e.max() <= TOL, float(e.max())


def test_forward_units_rejects_bad_lists(jt):
    import torch
    plan = jt.Plan(**C3)
    x = torch.zeros(1, C3["N"], device="cuda")
    p = torch.empty(1, plan.partials_size, device="cuda")
    o = torch.empty(1, plan.floats_per_signal, device="cuda")
    n = len(plan.units())
    for bad in ([n], [-1], [0, 0]):
        with pytest.raises(jt.JTFSError) as e:
            plan.forward_units(x, bad, p, o)
        assert e.value.status == jt.JTFS_ERR_INVALID_ARG
