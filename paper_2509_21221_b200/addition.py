"""Batched node-addition optimizer over the C-ABI.

PAPER.md:446-449: "the optimal choice of node addition is determined by running the minimum cost
flow algorithm for each combination of S candidate nodes added to each of the S stages"; the
improvement of a placement is (cost_now - cost_after) / cost_now.  The S!
placements are built on the device (gwtf_addition_build), solved as one batch by the exact
solver (gwtf_flow_solve_batch, unchanged) and reduced on the device (gwtf_addition_select).
Baselines: capacity-first (candidates by capacity, highest first,
matched with the stages ranked by utilization, highest first) and a seeded random placement.
"""
from __future__ import annotations

import math

import torch

from . import _lib
from ._lib import check, lib
from .flow import Flow


def num_placements(S: int) -> int:
    return math.factorial(S)


def placement(index: int, S: int) -> list:
    """perm[s] = candidate placed in stage s for placement `index` (lexicographic rank)."""
    pool = list(range(S))
    perm = []
    for s in range(S):
        f = math.factorial(S - 1 - s)
        d, index = divmod(index, f)
        perm.append(pool.pop(d))
    return perm


def placement_index(perm) -> int:
    """Lexicographic rank of a permutation (inverse of placement())."""
    pool = sorted(perm)
    idx = 0
    for s, c in enumerate(perm):
        d = pool.index(c)
        idx += d * math.factorial(len(perm) - 1 - s)
        pool.pop(d)
    return idx


def _p(t):
    return None if t is None else t.data_ptr()


def optimal_addition(cap, src_cost, snk_cost, link_cost, cand_cap, cand_in, cand_out, cand_cc, supply: int, *,
                     max_cap: int, chunk: int = 65536, stream=None):
    """All S! placements of the S candidates (device tensors, layouts of include/gwtf.h
    gwtf_addition_build), solved exactly.  Returns dict(best_index, perm, F, cost, all_F, all_cost)."""
    S, n = cap.shape
    dev = cap.device
    total = num_placements(S)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    all_F = torch.empty(total, dtype=torch.int64, device=dev)
    all_cost = torch.empty(total, dtype=torch.int64, device=dev)
    n1 = n + 1
    for first in range(0, total, chunk):
        count = min(chunk, total - first)
        cap_o = torch.empty((count, S, n1), dtype=torch.int32, device=dev)
        src_o = torch.empty((count, n1), dtype=torch.int32, device=dev)
        snk_o = torch.empty((count, n1), dtype=torch.int32, device=dev)
        link_o = torch.empty((count, max(S - 1, 0), n1, n1), dtype=torch.int32, device=dev)
        check("gwtf_addition_build", lib().gwtf_addition_build(
            S, n, _p(cap), _p(src_cost), _p(snk_cost), _p(link_cost), _p(cand_cap), _p(cand_in), _p(cand_out),
            _p(cand_cc), first, count, _p(cap_o), _p(src_o), _p(snk_o), _p(link_o), st.cuda_stream))
        fl = Flow(cap_o, src_o, snk_o, link_o, torch.full((count,), supply, dtype=torch.int64, device=dev),
                  max_cap=max_cap, stream=st)
        sol = fl.solve_batch()
        all_F[first:first + count] = sol.flow_value
        all_cost[first:first + count] = sol.total_cost
        fl.close()
    best = torch.empty(1, dtype=torch.int64, device=dev)
    check("gwtf_addition_select", lib().gwtf_addition_select(total, _p(all_F), _p(all_cost), _p(best),
                                                              st.cuda_stream))
    st.synchronize()
    b = int(best.item())
    return {"best_index": b, "perm": placement(b, S), "F": int(all_F[b].item()), "cost": int(all_cost[b].item()),
            "all_F": all_F, "all_cost": all_cost}


def capacity_first(cand_cap, stage_cap, flow_value: int) -> list:
    """candidates sorted by capacity, highest first (ties: lower id), matched
    positionally with the stages ranked by utilization F / capacity, highest first (ties: lower
    stage).  Returns perm[s] = candidate joining stage s."""
    S = len(stage_cap)
    cands = sorted(range(S), key=lambda c: (-int(cand_cap[c]), c))
    util = [(flow_value / int(stage_cap[s]) if int(stage_cap[s]) > 0 else float("inf")) for s in range(S)]
    stages = sorted(range(S), key=lambda s: (-util[s], s))
    perm = [0] * S
    for c, s in zip(cands, stages):
        perm[s] = c
    return perm


def random_placement(S: int, seed: int) -> list:
    g = torch.Generator().manual_seed(seed)
    return torch.randperm(S, generator=g).tolist()


def improvement(cost_now: float, cost_after: float) -> float:
    """(cost_now - cost_after) / cost_now."""
    return (cost_now - cost_after) / cost_now
