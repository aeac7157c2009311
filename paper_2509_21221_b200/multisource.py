"""Multi-data-node flows (exact-solve part) over the C-ABI.

PAPER.md:203 and the flow-test settings 5-6 have several data nodes, each of which
must get its own microbatches back.  SPEC.md:215 decomposes this heuristically: one single-commodity
problem per data node, in data-node order, each over the node capacities the earlier ones left.
Every step of the method runs in the library's kernels: the exact solves (gwtf_flow_solve_batch) and the
residual capacities (gwtf_flow_residual_caps); this module sequences the calls and keeps per-data-node
totals (torch additions of the per-call outputs).  Two readings of "round-robin order": whole data nodes
one after another (multi_source_ssp), or one microbatch per data node per turn (multi_source_ssp_unit).
"""
from __future__ import annotations

import torch

from .flow import Flow


def multi_source_ssp(cap, alive, link_cost, src_costs, snk_costs, supplies, *, max_cap: int, stream=None):
    """cap/alive [B][S][n], link_cost [B][S-1][n][n], src_costs/snk_costs: K tensors [B][n] (one per
    data node), supplies: K tensors [B] (int64).  Returns K (flow_value, total_cost, node_flow) triples."""
    out = []
    cap_k, alive_k = cap, alive
    for src, snk, M in zip(src_costs, snk_costs, supplies):
        fl = Flow(cap_k, src, snk, link_cost, M, max_cap=max_cap, alive=alive_k, stream=stream)
        sol = fl.solve_batch()
        nf, _, _, _ = fl.get_assignment(dense_arcs=False)
        cap_k, alive_k = fl.residual_caps(), None
        out.append((sol.flow_value, sol.total_cost, nf))
        fl.close()
    return out


def multi_source_ssp_unit(cap, alive, link_cost, src_costs, snk_costs, supplies, *, max_cap: int, stream=None):
    """Round-robin by microbatch: the data nodes take turns routing one microbatch each (a supply-1
    exact solve over the capacities left so far) until none can; same outputs as multi_source_ssp.
    Instances whose data node k is done get supply 0 in its later turns."""
    K = len(src_costs)
    B = cap.shape[0]
    dev = cap.device
    cap_r, alive_r = cap, alive  # the first solve applies the alive mask; residual caps include it
    F = [torch.zeros(B, dtype=torch.int64, device=dev) for _ in range(K)]
    C = [torch.zeros(B, dtype=torch.int64, device=dev) for _ in range(K)]
    NF = [torch.zeros_like(cap) for _ in range(K)]
    active = [torch.ones(B, dtype=torch.bool, device=dev) & (supplies[k] > 0) for k in range(K)]
    while any(bool(a.any()) for a in active):
        for k in range(K):
            if not bool(active[k].any()):
                continue
            fl = Flow(cap_r, src_costs[k], snk_costs[k], link_cost, active[k].to(torch.int64), max_cap=max_cap,
                      alive=alive_r, stream=stream)
            sol = fl.solve_batch()
            nf, _, _, _ = fl.get_assignment(dense_arcs=False)
            cap_r, alive_r = fl.residual_caps(), None
            fl.close()
            routed = sol.flow_value > 0
            F[k] += sol.flow_value
            C[k] += sol.total_cost
            NF[k] += nf
            active[k] = active[k] & routed & (F[k] < supplies[k])
    return [(F[k], C[k], NF[k]) for k in range(K)]


def mc_rounds(cap, alive, link_cost, src_costs, snk_costs, supplies, *, max_cap: int, max_rounds: int, seed=0,
              inst_base=0, T0=1.7, alpha=0.95, objective=0, steady_window=5, deny_after=3, digests=False,
              state=False, start_state=None, round0=0, stream=None):
    """Multi-data-node decentralized rounds (gwtf_mc_rounds): K data
    nodes with src_costs / snk_costs (K tensors [B][n] int32) and supplies (K tensors [B] int64) on the
    shared relays and links; rounds from the empty state.  Returns a dict: rounds [B], F_dec / cost_dec
    [K][B], dangling [B], digests [B][max_rounds] (if asked), up / down / tag [B][S][n][max_cap] (if
    state)."""
    import ctypes

    from ._lib import check, lib
    B, S, n = cap.shape
    K = len(supplies)
    dev = cap.device
    src = torch.stack(list(src_costs)).to(torch.int32).contiguous()
    snk = torch.stack(list(snk_costs)).to(torch.int32).contiguous()
    sup = torch.stack(list(supplies)).to(torch.int64).contiguous()
    out = dict(rounds=torch.empty(B, dtype=torch.int32, device=dev),
               F_dec=torch.empty((K, B), dtype=torch.int64, device=dev),
               cost_dec=torch.empty((K, B), dtype=torch.int64, device=dev),
               dangling=torch.empty(B, dtype=torch.int32, device=dev))
    if digests:
        out["digests"] = torch.zeros((B, max(max_rounds, 1)), dtype=torch.int64, device=dev)
    Mmax = max(1, int(sup.max()))
    if state or start_state is not None:
        for k in ("up", "down", "tag"):
            out[k] = torch.empty((B, S, n, max_cap), dtype=torch.int32, device=dev)
        for k in ("src_down", "snk_up"):
            out[k] = torch.empty((B, K, Mmax), dtype=torch.int32, device=dev)
        if start_state is not None:  # the starting state (copied in; the arrays receive the final state)
            for k in ("up", "down", "tag", "src_down", "snk_up"):
                out[k].copy_(start_state[k].reshape(out[k].shape))
    p = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    link = link_cost.contiguous() if S > 1 else None
    check("gwtf_mc_rounds", lib().gwtf_mc_rounds(
        B, S, n, max_cap, K, p(cap.contiguous()), p(alive.contiguous() if alive is not None else None), p(link),
        p(src), p(snk), p(sup), seed, inst_base, T0, alpha, objective, steady_window, deny_after, max_rounds,
        p(out["rounds"]), p(out["F_dec"]), p(out["cost_dec"]), p(out["dangling"]), p(out.get("digests")),
        p(out.get("up")), p(out.get("down")), p(out.get("tag")), p(out.get("src_down")), p(out.get("snk_up")),
        1 if start_state is not None else 0, int(round0), ctypes.c_void_p(st.cuda_stream)))
    return out
