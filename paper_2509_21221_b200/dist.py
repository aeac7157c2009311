"""Multi-GPU: instance sharding + one NCCL gather of per-instance results.

Instances are independent, so rank r owns a contiguous global id range and builds its own shard
(the caller's seeded generator: no input transfer).  The only collective is an all-gather of the
packed per-instance results after the solve; nothing runs inside the solver loops.  The RNG of
the rounds is keyed on the global instance id (inst_base), so every instance's result is
independent of the GPU count -- the gathered results equal a single-GPU run of the same ids.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

RESULT_FIELDS = ("flow_value", "total_cost", "augmentations", "status", "rounds_run", "dec_flow", "dec_cost",
                 "dangling")


def shard_range(total: int, world: int, rank: int):
    """Contiguous, balanced [lo, hi) instance range of `rank`."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_results(sol, rr) -> torch.Tensor:
    """[B][8] int64: F, cost, A, status, rounds, F_dec, cost_dec, dangling."""
    cols = [sol.flow_value, sol.total_cost, sol.augmentations, sol.status, rr.rounds_run, rr.dec_flow, rr.dec_cost,
            rr.dangling]
    return torch.stack([c.to(torch.int64) for c in cols], dim=1)


def gather_packed(local: torch.Tensor, world: int, group=None, counts=None) -> torch.Tensor:
    """All ranks' rows in rank order, [sum_r B_r][C].  Shards may differ in size (B % world != 0):
    every rank pads to the largest shard for one all_gather_into_tensor and the padding is cut
    out again.  `counts` (rows per rank) may be given when every rank knows them (shard_range);
    otherwise they are exchanged first (one tiny all_gather)."""
    local = local.contiguous()
    if world <= 1:
        return local
    if counts is None:
        c = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
        allc = torch.empty(world, dtype=torch.int64, device=local.device)
        dist.all_gather_into_tensor(allc, c, group=group)
        counts = [int(x) for x in allc.tolist()]
    mx = max(counts)
    pad = torch.zeros((mx, local.shape[1]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * mx, local.shape[1]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * mx: r * mx + counts[r]] for r in range(world)])


def gather_results(sol, rr, world: int, group=None, counts=None):
    """All ranks' packed results, [total][8] in global id order (None on a single GPU: nothing
    to exchange)."""
    if world <= 1:
        return None
    return gather_packed(pack_results(sol, rr), world, group, counts)


def totals(gathered: torch.Tensor) -> dict:
    """Objective totals over all instances (flow, cost, decentralized flow and cost)."""
    s = gathered.sum(dim=0)
    return {k: int(s[i]) for i, k in enumerate(RESULT_FIELDS)}


def solve_sharded(make_shard, total: int, max_rounds: int, *, rank: int | None = None, world: int | None = None,
                  group=None, churn=None, **flow_kw):
    """One sharded pass of the hot path (SURVEY.md 1c layer 5, 3 #5): this rank's contiguous share
    of `total` instances is built by `make_shard(lo, hi)` -> (cap, src, snk, link, supply, alive)
    device tensors (the caller's seeded generator, keyed on global ids), solved exactly
    (solve_batch) and by the decentralized rounds (max_rounds), and the packed results of all
    ranks are gathered in global id order.  `churn(flow, lo, hi)` (optional) runs between the
    pre-churn rounds and the step (the churn protocol of SURVEY.md 8(d)): with it, the step is
    pre-churn rounds -> churn -> cold solve -> repair rounds, else cold solve + rounds.
    Returns (packed [total][8] on every rank -- or this rank's [B][8] when world == 1, the Flow)."""
    from .flow import Flow
    if world is None:
        world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if world > 1 else 0
    lo, hi = shard_range(total, world, rank)
    cap, src, snk, link, supply, alive = make_shard(lo, hi)
    fl = Flow(cap, src, snk, link, supply, alive=alive, inst_base=lo, **flow_kw)
    if churn is not None:
        fl.decentralized_rounds(max_rounds)
        churn(fl, lo, hi)
    sol = fl.solve_batch()
    rr = fl.decentralized_rounds(max_rounds)
    counts = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
    local = pack_results(sol, rr)
    return (gather_packed(local, world, group, counts) if world > 1 else local), fl
