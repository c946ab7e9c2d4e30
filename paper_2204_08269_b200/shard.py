"""Path sharding of one JTFS forward over several GPUs.

For a single long signal (config c4) the batch does not shard, but the joint
stage does: its phi_T-pooled output (Eq. (3)) is a sum over
time of per-(alpha, time chunk) contributions.  KD's work units are those
(alpha, chunk) pairs (`Plan.units()`); each rank

  1. runs the replicated first stages (Eqs. (1)-(2): KA..KC, S0/S1) and KD for
     the units assigned to it (`Plan.forward_units`), whose partial slices are
     disjoint from every other rank's (the rest of its buffer is zero);
  2. contributes its partial buffer to a SUM reduction to rank 0 -- every slice
     is nonzero on exactly one rank, so x + 0 + ... + 0 = x exactly and the
     result does not depend on the reduction order or on the number of ranks;
  3. rank 0 finishes Eq. (3) (phi_F pooling, phi paths, packing) with
     `Plan.reduce_pack`.

The result is byte-identical to `Plan.forward` on one GPU.  Units are assigned by
a deterministic longest-processing-time greedy on the plan's modelled unit cost.
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


def exchange_partials(partials, group=None, dst: int = 0):
    """Sum the ranks' disjoint partial buffers onto `dst` (in place there).

    Exact because each slice is nonzero on exactly one rank."""
    import torch.distributed as dist
    dist.reduce(partials, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return partials


def forward_sharded(plan, x, group=None, stream=None):
    """Path-sharded forward of x (CUDA float32 [B, N], B <= the plan's micro-batch)
    over the ranks of `group`.  Returns the packed output on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    units = plan.units()
    mine = lpt_assign([u["cost"] for u in units], world)[rank]
    B = x.shape[0]
    # every step (KD, the NCCL reduce, KE) is ordered on ONE stream: torch's collectives
    # run on the current stream, so a caller's stream becomes the current one here
    with torch.cuda.stream(stream) if stream is not None else _nullctx():
        partials = torch.empty(B, plan.partials_size, dtype=torch.float32, device=x.device)
        out = torch.empty(B, plan.floats_per_signal, dtype=torch.float32, device=x.device)
        plan.forward_units(x, mine, partials, out)
        if world > 1:
            exchange_partials(partials, group=group, dst=0)
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
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    import torch
    b0, b1 = batch_slice(x_full.shape[0], world, rank)
    with torch.cuda.stream(stream) if stream is not None else _nullctx():  # forward and gather on one stream
        out = plan.forward(x_full[b0:b1].contiguous())
        return gather_outputs(out, x_full.shape[0], group) if gather else out
