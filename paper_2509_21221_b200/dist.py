"""Multi-GPU: instance sharding + one NCCL gather of per-instance results.

Instances are independent, so rank r owns the contiguous global id range [r*B, (r+1)*B) and
generates its own shard from the seeded generator (no input transfer).  The only collective is
an all_gather_into_tensor of the packed per-instance results after the solve; nothing runs
inside the solver loops.  The RNG of the rounds is keyed on the global instance id
(inst_base), so every instance's result is independent of the GPU count.
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


def gather_results(sol, rr, world: int, group=None):
    """All ranks' packed results, [world*B][8] (None on a single GPU: nothing to exchange)."""
    if world <= 1:
        return None
    local = pack_results(sol, rr).contiguous()
    out = torch.empty((world * local.shape[0], local.shape[1]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out


def totals(gathered: torch.Tensor) -> dict:
    """Objective totals over all instances (flow, cost, decentralized flow and cost)."""
    s = gathered.sum(dim=0)
    return {k: int(s[i]) for i, k in enumerate(RESULT_FIELDS)}
