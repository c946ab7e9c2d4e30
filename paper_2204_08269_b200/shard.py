"""Path sharding of one JTFS forward over several GPUs.

For a single long signal (config c4) the batch does not shard, but the joint
stage does: its phi_T-pooled output (Eq. (3)) is a sum over
time of per-(alpha, time chunk) contributions.  KD's work units are those
(alpha, chunk) pairs (`Plan.units()`), ordered like the partials buffer they
write; each rank

  1. owns one contiguous range of unit ids (`contiguous_assign`: the optimal
     contiguous split of the modelled unit costs), hence one contiguous float range
     of the partials buffer;
  2. runs the replicated first stages (Eqs. (1)-(2): KA..KC, S0/S1) and KD for its
     units (`Plan.forward_unitset`: a unit set bound once, no host sync);
  3. sends exactly its range to rank 0 (NCCL point-to-point), which receives each
     rank's range in place -- no arithmetic on the exchange, so the result is
     byte-identical to `Plan.forward` on one GPU for any rank count;
  4. rank 0 finishes Eq. (3) (phi_F pooling, phi paths, packing) with
     `Plan.reduce_pack`.
This module is plumbing only: all arithmetic of the path runs in libjtfs.so.
"""
from __future__ import annotations


def lpt_assign(costs, world: int):
    """Deterministic LPT: units sorted by (-cost, id), each to the least-loaded rank
    (ties -> lowest rank).  Returns per-rank ascending unit-id lists."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    load = [0.0] * world
    parts = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        parts[r].append(i)
        load[r] += float(costs[i])
    return [sorted(p) for p in parts]


def contiguous_assign(costs, world: int):
    """Split unit ids 0..n-1 into `world` contiguous ranges minimising the largest range
    cost (binary search on the bound + greedy fill; deterministic).  Returns per-rank
    (first, last + 1) id ranges (possibly empty)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    c = [float(v) for v in costs]

    def fill(bound):
        parts, start, acc = [], 0, 0.0
        for i, v in enumerate(c):
            if acc + v > bound and i > start:
                parts.append((start, i))
                start, acc = i, 0.0
            acc += v
        parts.append((start, len(c)))
        return parts

    lo, hi = max(c, default=0.0), sum(c)
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if len(fill(mid)) <= world:
            hi = mid
        else:
            lo = mid
    parts = fill(hi)
    while len(parts) < world:
        parts.append((len(c), len(c)))
    return parts


def owned_range(plan, first: int, last: int):
    """[begin, end) floats of one signal's partials written by units first..last-1."""
    if last <= first:
        return 0, 0
    return plan.unit_partials_range(first)[0], plan.unit_partials_range(last - 1)[1]


def exchange_partials(partials, ranges, group=None, dst: int = 0):
    """Every rank sends its own contiguous partials range ranges[rank] = (b, e) (floats
    per signal) to `dst`, which receives each into place: an exact copy, no reduction
    (every float is written by exactly one rank's units)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    reqs = []
    if rank == dst:
        for r in range(world):
            b, e = ranges[r]
            if r != dst and e > b:
                buf = partials[:, b:e].contiguous() if partials.shape[0] > 1 else partials[0, b:e]
                reqs.append((dist.irecv(buf, src=dist.get_global_rank(group, r) if group else r, group=group), buf, b, e))
        for q, buf, b, e in reqs:
            q.wait()
            if partials.shape[0] > 1:
                partials[:, b:e] = buf.view(partials.shape[0], e - b)
    else:
        b, e = ranges[rank]
        if e > b:
            buf = partials[:, b:e].contiguous() if partials.shape[0] > 1 else partials[0, b:e]
            dist.send(buf, dst=dist.get_global_rank(group, dst) if group else dst, group=group)
    return partials


_SHARDS = {}


def _shard_of(plan, world: int, rank: int):
    """(unit set bound for this rank, owned partial ranges of every rank), computed once per
    (plan, world, rank): the host-side assignment is not on the per-forward path."""
    key = (id(plan), world, rank)
    hit = _SHARDS.get(key)
    if hit is None or hit[0].plan is not plan:
        parts = contiguous_assign([u["cost"] for u in plan.units()], world)
        first, last = parts[rank]
        hit = (plan.unitset(range(first, last)), [owned_range(plan, a, b) for a, b in parts])
        _SHARDS[key] = hit
    return hit


def forward_sharded(plan, x, group=None, stream=None):
    """Path-sharded forward of x (CUDA float32 [B, N], B <= the plan's micro-batch)
    over the ranks of `group`.  Returns the packed output on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    uset, ranges = _shard_of(plan, world, rank)
    B = x.shape[0]
    # every step (KD, the NCCL exchange, KE) is ordered on ONE stream: torch's
    # point-to-point ops run on the current stream, so a caller's stream becomes it here
    with torch.cuda.stream(stream) if stream is not None else _nullctx():
        partials = torch.empty(B, plan.partials_size, dtype=torch.float32, device=x.device)
        out = torch.empty(B, plan.floats_per_signal, dtype=torch.float32, device=x.device)
        plan.forward_unitset(x, uset, partials, out)
        if world > 1:
            exchange_partials(partials, ranges, group=group, dst=0)
        if rank != 0:
            return None
        plan.reduce_pack(partials, out)
    return out


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ---- batch sharding (configs c3 / c5): signals are independent ----
def batch_slice(B: int, world: int, rank: int):
    """Contiguous signal range [b0, b1) of `rank`: the first B % world ranks get one extra."""
    if world < 1 or not 0 <= rank < world or B < 0:
        raise ValueError("bad batch split")
    q, r = divmod(B, world)
    b0 = rank * q + min(rank, r)
    return b0, b0 + q + (1 if rank < r else 0)


def gather_outputs(local_out, B: int, group=None):
    """The optional collective of the batch-sharded path: all ranks' fp32 records
    (rank r holds batch_slice(B, world, r)) gathered into one [B, floats] tensor on every
    rank with all_gather_into_tensor (ranks' slices padded to the largest one)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local_out
    rank = dist.get_rank(group)
    fps = local_out.shape[1]
    cnt = max(b1 - b0 for b0, b1 in (batch_slice(B, world, r) for r in range(world)))
    send = torch.zeros(cnt, fps, dtype=local_out.dtype, device=local_out.device)
    b0, b1 = batch_slice(B, world, rank)
    send[: b1 - b0] = local_out
    recv = torch.empty(world * cnt, fps, dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    parts = []
    for r in range(world):
        a, b = batch_slice(B, world, r)
        parts.append(recv[r * cnt: r * cnt + (b - a)])
    return torch.cat(parts, dim=0)


def forward_batch_sharded(plan, x_full, group=None, gather: bool = True, stream=None):
    """Batch-sharded forward: rank r transforms its contiguous slice of x_full (CUDA
    float32 [B, N]) with no data-path collective; with `gather` the records are
    all-gathered (one NCCL all_gather_into_tensor).  Outputs are byte-identical to a
    single-GPU forward (the per-signal computation does not depend on B or the split)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b0, b1 = batch_slice(x_full.shape[0], world, rank)
    with torch.cuda.stream(stream) if stream is not None else _nullctx():  # forward and gather on one stream
        out = plan.forward(x_full[b0:b1].contiguous())
        return gather_outputs(out, x_full.shape[0], group) if gather else out
