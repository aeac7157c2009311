"""Hand-derived pin cases shared by the oracle pins (tests/test_oracle_pins.py, CPU) and the GPU
parity tests (tests/test_gpu_pins.py).  Every expected value below is derived by hand in the
docstring or comment next to it, from DESIGN.md 2.2-2.3 (the readings of PAPER.md:241-269) -- none
was produced by running the oracle or the CUDA path.

Pointer encoding: relay slot = gid * max_cap + j, NONE = -1, data-node slot k = -2 - k
(SRC k on an up pointer, SNK k on a down pointer)."""
from __future__ import annotations

import numpy as np

ABSENT = np.iinfo(np.int32).max
NONE = -1


def D(k):
    """data-node slot k as a pointer (SRC k for up, SNK k for down)"""
    return -2 - k


def state(S, n, MC, M, slots, src_down, snk_up, kacc=None, deny=None, quiet=0, rnd=0):
    """Round state in the export layouts from {slot id: (up, down)}; unlisted slots are FREE."""
    up = np.full(S * n * MC, NONE, np.int32)
    dn = np.full(S * n * MC, NONE, np.int32)
    for p, (u, d) in slots.items():
        up[p], dn[p] = u, d
    return dict(up=up.reshape(S, n, MC), down=dn.reshape(S, n, MC),
                src_down=np.asarray(src_down, np.int32), snk_up=np.asarray(snk_up, np.int32),
                kacc=np.zeros((S, n), np.int32) if kacc is None else np.asarray(kacc, np.int32).reshape(S, n),
                deny=np.zeros((S, n), np.int32) if deny is None else np.asarray(deny, np.int32).reshape(S, n),
                quiet=quiet, round=rnd)


# --------------------------------------------------------------------------- instances (dicts)
def inst(S, n, MC, M, cap, src, snk, link, alive=None):
    return dict(S=S, n=n, max_cap=MC, M=M, cap=np.asarray(cap, np.int32).reshape(S, n),
                src=np.asarray(src, np.int32), snk=np.asarray(snk, np.int32),
                link=np.asarray(link, np.int32).reshape(max(S - 1, 0), n, n),
                alive=np.ones((S, n), np.uint8) if alive is None else np.asarray(alive, np.uint8).reshape(S, n))


def link_from(S, n, arcs):
    """link[s][v][u] = d((s,u) -> (s+1,v)) from {(s, u, v): cost}; everything else ABSENT."""
    L = np.full((max(S - 1, 0), n, n), ABSENT, np.int32)
    for (s, u, v), c in arcs.items():
        L[s, v, u] = c
    return L


# ===================================================================== SSP canonical ties (C2)
def ssp_tie_position():
    """S=2, n=2, caps 1, M=1, every cost 0 except links = 1.  All four s*-t* paths cost 1 with the
    same 5 hops; the canonical rule (lowest (layer, position) tight predecessor, walking back from
    t*) picks out_{1,0}, then in_{1,0}, then out_{0,0} over out_{0,1}, then in_{0,0}:
    path s* -> (0,0) -> (1,0) -> t*.  F = 1, cost = 1, A = 1; node flow [[1,0],[1,0]], f(0->0) = 1.
    (Highest-index ties would give [[0,1],[0,1]].)"""
    I = inst(2, 2, 1, 1, [1, 1, 1, 1], [0, 0], [0, 0], np.ones((1, 2, 2), np.int32))
    exp = dict(F=1, cost=1, A=1, node_flow=[[1, 0], [1, 0]], src_flow=[1, 0], snk_flow=[1, 0],
               arc=[(0, 0, 0, 1)])  # (s, u, v, f)
    return I, exp


def ssp_tie_hops():
    """S=2, n=2, caps 1, M=2, src = snk = 0, d(0->0)=1, d(0->1)=2, d(1->0)=2, d(1->1)=3.
    Aug 1: keys in_0 = (0,1), out_0 = (0,2); in_{1,0} = (1,3) via out_{0,0}, in_{1,1} = (2,3) via
      out_{0,0}; t* = (1,5) via out_{1,0}.  Path s*-(0,0)-(1,0)-t*, delta 1, cost 1.
    Aug 2: (0,0) and (1,0) are saturated.  in_{1,0} = (2,3) via out_{0,1}; out_{0,0} = in_{1,0}
      + (-1, 1) = (1,4) (reverse arc); in_{1,1} = min((0,2)+(3,1) via out_{0,1}, (1,4)+(2,1) via
      out_{0,0}) = min((3,3), (3,5)) = (3,3): the COST ties at 3 and the hop count decides;
      t* = (3,5) via out_{1,1}.  Path s*-(0,1)-(1,1)-t*, cost 3.
    F = 2, cost = 4, A = 2, f(0->0) = f(1->1) = 1.  Cost-only keys with the lowest-position rule
    would take out_{0,0} at in_{1,1} and route s*-(0,1)-(1,0)~(0,0)-(1,1)-t* (same cost 3), ending
    with f(1->0) = f(0->1) = 1 instead."""
    link = link_from(2, 2, {(0, 0, 0): 1, (0, 0, 1): 2, (0, 1, 0): 2, (0, 1, 1): 3})
    I = inst(2, 2, 1, 2, [1, 1, 1, 1], [0, 0], [0, 0], link)
    exp = dict(F=2, cost=4, A=2, node_flow=[[1, 1], [1, 1]], src_flow=[1, 1], snk_flow=[1, 1],
               arc=[(0, 0, 0, 1), (0, 1, 1, 1)])
    return I, exp


def ssp_tie_cancel():
    """S=2, n=2, caps 1, M=2, src = snk = 0, d(0->0)=1, d(1->0)=1, d(0->1)=1, d(1->1)=10.
    Aug 1: in_{1,0} = (1,3) (out_{0,0} and out_{0,1} tie; lowest position out_{0,0}); in_{1,1} =
      (1,3) via out_{0,0}; t* = (1,5), out_{1,0} and out_{1,1} tie -> out_{1,0}.
      Path s*-(0,0)-(1,0)-t*, cost 1.
    Aug 2: in_{1,0} = (1,3) via out_{0,1}; out_{0,0} = (1,3) + (-1,1) = (0,4) over the reverse arc;
      in_{1,1} = min((0,4)+(1,1), (0,2)+(10,1)) = (1,5) via out_{0,0}; t* = (1,7) via out_{1,1}.
      Path s*-(0,1)-(1,0)~(0,0)-(1,1)-t*: it cancels f(0->0); cost 1 - 1 + 1 = 1, delta 1.
    F = 2, cost = 2, A = 2, f(0->0) = 0, f(1->0) = f(0->1) = 1."""
    link = link_from(2, 2, {(0, 0, 0): 1, (0, 1, 0): 1, (0, 0, 1): 1, (0, 1, 1): 10})
    I = inst(2, 2, 1, 2, [1, 1, 1, 1], [0, 0], [0, 0], link)
    exp = dict(F=2, cost=2, A=2, node_flow=[[1, 1], [1, 1]], src_flow=[1, 1], snk_flow=[1, 1],
               arc=[(0, 1, 0, 1), (0, 0, 1, 1)])
    return I, exp


def ssp_bottleneck():
    """S=2, n=1, caps [2, 3], M=5, src 1, d = 2, snk 4: one augmentation of delta = min(M - F = 5,
    residual 2, 3) = 2.  F = 2, cost = 2 * 7 = 14, A = 1 (A < F)."""
    I = inst(2, 1, 3, 5, [2, 3], [1], [4], [[[2]]])
    exp = dict(F=2, cost=14, A=1, node_flow=[[2], [2]], src_flow=[2], snk_flow=[2], arc=[(0, 0, 0, 2)])
    return I, exp


SSP_CASES = {"position": ssp_tie_position, "hops": ssp_tie_hops, "cancel": ssp_tie_cancel,
             "bottleneck": ssp_bottleneck}


def arc_dense(I, arcs):
    a = np.zeros((max(I["S"] - 1, 0), I["n"], I["n"]), np.int32)
    for s, u, v, f in arcs:
        a[s, v, u] = f
    return a


# ===================================================================== DENY (DESIGN 2.3 R4-R6)
def deny_case():
    """S=3, n=2, caps 1, M=2, T0 = 0 (no uphill move).  gids: a0=0 a1=1 (stage 0), b0=2 b1=3,
    c0=4 c1=5 (dead).  Links a0->b0 = a1->b1 = 1, a0->b1 = a1->b0 absent, b0->c0 = b1->c0 = 1,
    b*->c1 = 1; src = snk = 1.
    Start (round 40): SRC0 -> a0 -> b0 (IN), SRC1 -> a1 -> b1 (IN), c0 OUT -> SNK0.

    Every peer draw is forced (n = 2, one slot each); every move below is ruled out by an absent
    link, a peer without PAIRED slots, j1 == j2, or a dead peer -- so the trace is RNG-free.
      r40: b0 and b1 both request c0's one OUT slot (adv 1); b0 (lower gid) is granted, b1 is
           REJECTED -- a requester, so not idle, so deny[b1] stays 0.  F_dec 1.
      r41: c0 has no OUT: b1 finds no target, is idle with IN -> deny[b1] = 1.
      r42: deny[b1] = 2.
      r43: deny[b1] = 3 = deny_after -> DENY: b1's slot FREE, a1's slot PAIRED -> IN
           (up SRC1 kept, down cleared), deny[b1] = 0.
      r44: a1 (IN) finds no target (b1 advertises nothing, a1->b0 absent): deny[a1] = 1.
      r45: deny[a1] = 2.
      r46: DENY by a1: a1's slot FREE, SRC1 unpaired, deny[a1] = 0.
      r47-r51: quiet 1..5 -> stop after r51 (12 rounds from r40).
    Final: F_dec 1 (SRC0-a0-b0-c0-SNK0, cost 1+1+1+1 = 4), dangling 0."""
    n, MC = 2, 1
    arcs = {(0, 0, 0): 1, (0, 1, 1): 1, (1, 0, 0): 1, (1, 1, 0): 1, (1, 0, 1): 1, (1, 1, 1): 1}
    I = inst(3, n, MC, 2, [1] * 6, [1, 1], [1, 1], link_from(3, n, arcs), alive=[1, 1, 1, 1, 1, 0])
    st0 = state(3, n, MC, 2, {0: (D(0), 2), 1: (D(1), 3), 2: (0, NONE), 3: (1, NONE), 4: (NONE, D(0))},
                src_down=[0, 1], snk_up=[4, NONE], rnd=40)
    # expected (slot 0..5 (up, down), src_down, snk_up, deny) after each round r40, r41, ...
    a = {0: (D(0), 2), 1: (D(1), 3), 2: (0, 4), 3: (1, NONE), 4: (2, D(0))}
    after = {
        40: (a, [0, 1], [4, NONE], [0, 0, 0, 0, 0, 0]),
        41: (a, [0, 1], [4, NONE], [0, 0, 0, 1, 0, 0]),
        42: (a, [0, 1], [4, NONE], [0, 0, 0, 2, 0, 0]),
        43: ({0: (D(0), 2), 1: (D(1), NONE), 2: (0, 4), 4: (2, D(0))}, [0, 1], [4, NONE], [0] * 6),
        44: ({0: (D(0), 2), 1: (D(1), NONE), 2: (0, 4), 4: (2, D(0))}, [0, 1], [4, NONE], [0, 1, 0, 0, 0, 0]),
        45: ({0: (D(0), 2), 1: (D(1), NONE), 2: (0, 4), 4: (2, D(0))}, [0, 1], [4, NONE], [0, 2, 0, 0, 0, 0]),
        46: ({0: (D(0), 2), 2: (0, 4), 4: (2, D(0))}, [0, NONE], [4, NONE], [0] * 6),
    }
    final = dict(rounds=12, F_dec=1, cost_dec=4, dangling=0, round=52)
    return I, st0, after, final, dict(T0=0.0, seed=11, inst_id=0)


# ===================================================================== R0a self-pairing
def selfpair_case():
    """S=3, n=2, M=2, T0 = 0.  gids a0=0 a1=1, b0=2 (cap 4) b1=3, c0=4 c1=5; caps 1 otherwise;
    max_cap 4, so slot ids are gid*4+j.  Links a0->b0 = a1->b0 = 1, b0->c0 = 5, b0->c1 = 2, every
    link into or out of b1 absent (a*->b1, b1->c*); src = snk = 1.
    Start (round 7): b0 holds s0 OUT (-> c0, cost to sink 5+1 = 6), s1 IN (from a0), s2 OUT
    (-> c1, cost 2+1 = 3), s3 IN (from a1); c0, c1 paired to SNK0 / SNK1; a0, a1 from SRC0 / SRC1.
      r7:  R0a -- b0's LOWEST IN slot s1 takes the downstream of its MIN-COST OUT slot s2 (c1, cost
           3 < 6); s2 becomes FREE ("unless it had already unpaired inflow it can connect it
           to").  R1: b0 (IN s3) finds no target (c0, c1 advertise nothing); b1 has no links.
           R4: b0 idle with IN -> deny[b0] = 1; every other move is ruled out (j1 == j2 for a0/a1
           and c0/c1, absent a->b1 links for b1's Redirect).
      r8:  R0a again: s3 takes s0's downstream c0, s0 becomes FREE.  b0's deny stays 1 (no IN).
      r9-r13: quiet 1..5 -> stop (7 rounds from r7).
    Final F_dec 2: SRC0-a0-b0-c1-SNK1 (1+1+2+1 = 5) + SRC1-a1-b0-c0-SNK0 (1+1+5+1 = 8) = 13.
    (Highest-cost first would link s1 to c0 in r7; highest IN first would link s3 in r7.)"""
    n, MC = 2, 4
    arcs = {(0, 0, 0): 1, (0, 1, 0): 1, (1, 0, 0): 5, (1, 0, 1): 2}
    I = inst(3, n, MC, 2, [1, 1, 4, 1, 1, 1], [1, 1], [1, 1], link_from(3, n, arcs))
    a0, a1, c0, c1 = 0, 4, 16, 20
    b = lambda j: 8 + j  # noqa: E731
    st0 = state(3, n, MC, 2, {a0: (D(0), b(1)), a1: (D(1), b(3)), b(0): (NONE, c0), b(1): (a0, NONE),
                              b(2): (NONE, c1), b(3): (a1, NONE), c0: (b(0), D(0)), c1: (b(2), D(1))},
                src_down=[a0, a1], snk_up=[c0, c1], rnd=7)
    after = {
        7: ({a0: (D(0), b(1)), a1: (D(1), b(3)), b(0): (NONE, c0), b(1): (a0, c1), b(3): (a1, NONE),
             c0: (b(0), D(0)), c1: (b(1), D(1))}, [a0, a1], [c0, c1], [0, 0, 1, 0, 0, 0]),
        8: ({a0: (D(0), b(1)), a1: (D(1), b(3)), b(1): (a0, c1), b(3): (a1, c0),
             c0: (b(3), D(0)), c1: (b(1), D(1))}, [a0, a1], [c0, c1], [0, 0, 1, 0, 0, 0]),
    }
    final = dict(rounds=7, F_dec=2, cost_dec=13, dangling=0, round=14)
    return I, st0, after, final, dict(T0=0.0, seed=3, inst_id=0)


# ===================================================================== annealing draw
# h(seed, inst, round, gid, stream) of DESIGN.md 2.3 at the inputs the annealing trace uses:
# inst 0, round 100, stream 3 (the accept draw), gid 0 and 1 -- computed by hand from the
# splitmix64 finalizer (whose outputs are pinned against the published SplitMix64 sequence in
# test_oracle_pins.test_mix64_published_sequence).  The decision compares h >> 32 with
# thr[0][1] = 2385022711 = floor(exp(-1/1.7) * 2^32) (pinned by the table test).
THR_0_1 = 2385022711
ANNEAL_DRAWS = {
    # seed: (h(gid 0, stream 3), h(gid 1, stream 3), outcome)
    6: (0x87f660b0485fa814, 0x82876c035ebbe063, "gid0"),   # 2281070768 < thr: n1's swap commits
    19: (0x8f4436ac9dba2237, 0x58cb0b478370003c, "gid1"),  # 2403612332 >= thr (by 0.8%); n3: 1489701703 <
    2: (0xf784f419f74f750c, 0xe7ea5ac77eefa86f, "none"),   # 4152685593, 3890895559: both reject
}


def anneal_case(seed):
    """PAPER.md:256's instance at the SUM optimum, SUM objective, T0 = 1.7, alpha 0.95:
    n1=gid0 -> n2=gid2 (d 3), n3=gid1 -> n4=gid3 (d 8); the swap n1->n4 (6), n3->n2 (6) has
    delta = +1 for both n1 and n3 (an uphill move).  One round from round 100: no requests (all
    slots PAIRED); n2/n4 cannot Change (j1 == j2 = D); n1 and n3 each propose the swap iff their
    draw (h(gid, 3) >> 32) < thr[kacc=0][1]; both touch the same four slots, so the lower gid
    proposing wins the reservation.  The committed swap gives cost_dec 12 and kacc[winner] = 1;
    with no proposal the state stays at cost 11 and quiet counts 1."""
    link = np.zeros((1, 2, 2), np.int32)
    link[0, 0, 0], link[0, 0, 1], link[0, 1, 0], link[0, 1, 1] = 3, 6, 6, 8  # [v][u]
    I = inst(2, 2, 1, 2, [1, 1, 1, 1], [0, 0], [0, 0], link)
    st0 = state(2, 2, 1, 2, {0: (D(0), 2), 1: (D(1), 3), 2: (0, D(0)), 3: (1, D(1))},
                src_down=[0, 1], snk_up=[2, 3], rnd=100)
    outcome = ANNEAL_DRAWS[seed][2]
    if outcome == "none":
        exp = ({0: (D(0), 2), 1: (D(1), 3), 2: (0, D(0)), 3: (1, D(1))}, [0, 0, 0, 0], 11)
    else:
        k = [1, 0, 0, 0] if outcome == "gid0" else [0, 1, 0, 0]
        exp = ({0: (D(0), 3), 1: (D(1), 2), 2: (1, D(0)), 3: (0, D(1))}, k, 12)
    return I, st0, exp, dict(T0=1.7, alpha=0.95, seed=seed, inst_id=0)


def expected_state(S, n, MC, M, slots, src_down, snk_up, deny=None, kacc=None):
    st = state(S, n, MC, M, slots, src_down, snk_up, kacc=kacc, deny=deny)
    return st
