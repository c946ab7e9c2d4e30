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
    partials = torch.empty(B, plan.partials_size, dtype=torch.float32, device=x.device)
    out = torch.empty(B, plan.floats_per_signal, dtype=torch.float32, device=x.device)
    plan.forward_units(x, mine, partials, out, stream=stream)
    if world > 1:
        exchange_partials(partials, group=group, dst=0)
    if rank != 0:
        return None
    plan.reduce_pack(partials, out, stream=stream)
    return out
