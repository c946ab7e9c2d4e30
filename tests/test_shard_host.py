"""Host logic of the path-sharded forward (paper_2204_08269_b200/shard.py), on CPU.

The CUDA work of `forward_units` / `reduce_pack` is covered by
tests/test_gpu_shard.py; here: the unit table of a host-only plan (c4 config), the
deterministic contiguous (and LPT) assignments, the partial ranges units own, and the
point-to-point exchange of the owned ranges over a world_size-2 gloo group (exact copies).
"""
import os
import socket

import numpy as np
import pytest

from paper_2204_08269_b200 import shard

C4 = dict(N=2 ** 17, J=13, Q=16, J_fr=5, T=2 ** 13, F=4)


@pytest.fixture(scope="module")
def jt():
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    return jtfs


def test_unit_table_tiles_every_alpha(jt):
    plan = jt.Plan(**C4, device=-1, flags=jt.JTFS_LATENCY)
    units = plan.units()
    assert len(units) > 148                      # enough units for one signal to fill the GPU
    by_alpha = {}
    for u in units:
        by_alpha.setdefault(u["alpha"], []).append(u)
        assert u["cost"] > 0 and u["ncols"] > 0
    assert sorted(by_alpha) == list(range(plan.layout.n_alpha))
    for a, us in by_alpha.items():
        cols = sorted((u["col0"], u["ncols"]) for u in us)
        assert cols[0][0] == 0
        for (c0, n0), (c1, _) in zip(cols, cols[1:]):
            assert c1 == c0 + n0                 # contiguous, non-overlapping chunks
    # the batch plan of the same config uses coarser chunks
    assert len(jt.Plan(**C4, device=-1).units()) <= len(units)
    # a host-only plan refuses to compute (no CPU fallback)
    import ctypes as C
    ids = (C.c_int32 * 1)(0)
    st = jt.library().jtfs_forward_units(plan.handle, None, 1, ids, 1, None, None, None, 0, None)
    assert st == jt.JTFS_ERR_UNSUPPORTED


def test_lpt_assignment():
    rng = np.random.default_rng(3)
    costs = rng.uniform(1, 100, 257).tolist()
    for world in (1, 2, 3, 8):
        parts = shard.lpt_assign(costs, world)
        assert parts == shard.lpt_assign(costs, world)           # deterministic
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(costs)))                   # a partition
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(costs)             # LPT bound
    with pytest.raises(ValueError):
        shard.lpt_assign(costs, 0)


def test_contiguous_assignment_and_owned_ranges(jt):
    plan = jt.Plan(**C4, device=-1, flags=jt.JTFS_LATENCY)
    costs = [u["cost"] for u in plan.units()]
    rng = np.random.default_rng(4)
    for cs in (costs, rng.uniform(1, 100, 257).tolist()):
        for world in (1, 2, 3, 8):
            parts = shard.contiguous_assign(cs, world)
            assert parts == shard.contiguous_assign(cs, world) and len(parts) == world
            assert parts[0][0] == 0 and parts[-1][1] == len(cs)
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))      # contiguous partition
            loads = [sum(cs[a:b]) for a, b in parts]
            assert max(loads) <= sum(cs) / world + max(cs) + 1e-9          # within one unit of the mean
    # unit ranges tile the partials buffer in unit order, disjoint
    prev_end = None
    for u in range(len(costs)):
        b, e = plan.unit_partials_range(u)
        assert e > b and (prev_end is None or b >= prev_end)
        prev_end = e
    assert prev_end <= plan.partials_size


def _fill(n, ranges):
    buf = np.zeros(n, dtype=np.float32)
    for b, e in ranges:
        k = np.arange(b, e)
        buf[b:e] = (np.sin(k * 0.37) * 10.0 ** ((k % 7) - 3)).astype(np.float32)
    return buf


def _worker(rank, world, port, n, ranges, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for B in (1, 2):
            t = torch.from_numpy(np.stack([_fill(n, [ranges[rank]])] * B))
            shard.exchange_partials(t, ranges, dst=0)
            if rank == 0:
                q.put((B, t.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_exchange_partials_gloo_world2(jt):
    import torch.multiprocessing as mp
    plan = jt.Plan(**C4, device=-1, flags=jt.JTFS_LATENCY)
    costs = [u["cost"] for u in plan.units()]
    parts = shard.contiguous_assign(costs, 2)
    ranges = [shard.owned_range(plan, a, b) for a, b in parts]
    n = plan.partials_size
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, ranges, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _fill(n, ranges)
    for B in (1, 2):
        assert got[B] == np.stack([want] * B).tobytes()             # byte-identical to one rank


def test_batch_slice_partitions():
    for B in (0, 1, 7, 256, 4097):
        for world in (1, 2, 3, 8):
            sl = [shard.batch_slice(B, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            sizes = [b - a for a, b in sl]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.batch_slice(4, 2, 2)


def _gather_worker(rank, world, port, B, fps, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b0, b1 = shard.batch_slice(B, world, rank)
        full = torch.arange(B * fps, dtype=torch.float32).reshape(B, fps)
        got = shard.gather_outputs(full[b0:b1].clone(), B)
        q.put((rank, got.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 8])
def test_gather_outputs_gloo_world2(B):
    # the optional all_gather of the batch-sharded records (ragged split)
    import torch.multiprocessing as mp
    fps = 5
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, B, fps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(B * fps, dtype=np.float32).tobytes()
    assert res[0] == want and res[1] == want


class _MockPlan:
    """Stands in for Plan in the host test of the batch-sharded forward: a deterministic
    per-signal map (the sharding is plumbing; the CUDA forward is tested on the GPU)."""
    floats_per_signal = 3

    def forward(self, x, stream=None):
        import torch
        return torch.stack([x.sum(1), x[:, 0] * 2, x[:, -1] - 1], dim=1)


def _bs_worker(rank, world, port, B, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = torch.arange(B * 4, dtype=torch.float32).reshape(B, 4)
        got = shard.forward_batch_sharded(_MockPlan(), x, gather=True)
        q.put((rank, got.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [5, 8])
def test_forward_batch_sharded_with_gather_gloo_world2(B):
    import torch
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bs_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = torch.arange(B * 4, dtype=torch.float32).reshape(B, 4)
    want = _MockPlan().forward(x).numpy().tobytes()
    assert res[0] == want and res[1] == want
