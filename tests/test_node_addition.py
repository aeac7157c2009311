"""Node addition:
the oracle's exhaustive optimizer pinned against an independent construction solved by networkx,
the baselines' host logic, and (-m gpu) the batched GPU optimizer against the oracle."""
import itertools

import numpy as np
import pytest
import torch

import gen
import oracle
from oracle import ABSENT

from paper_2509_21221_b200 import addition


def _nx_placement(I, cand, perm):
    """(F, cost) of the base + candidates perm[s] -> stage s, built directly as a networkx graph
    (independent of oracle.placed_instance)."""
    nx = pytest.importorskip("networkx")
    S, n = I.S, I.n
    G = nx.DiGraph()
    G.add_edge("s", "D", capacity=I.M, weight=0)
    ce = I.cap_eff()
    nodes = [[("b", s, i) for i in range(n)] + [("c", s, perm[s])] for s in range(S)]
    caps = [[int(ce[s, i]) for i in range(n)] + [int(cand["cap"][perm[s]])] for s in range(S)]
    for s in range(S):
        for k, x in enumerate(nodes[s]):
            G.add_edge(("in",) + x, ("out",) + x, capacity=caps[s][k], weight=0)
    for i in range(n):
        if I.src[i] != ABSENT:
            G.add_edge("D", ("in", "b", 0, i), weight=int(I.src[i]))
        if I.snk[i] != ABSENT:
            G.add_edge(("out", "b", S - 1, i), "t", weight=int(I.snk[i]))
    G.add_edge("D", ("in", "c", 0, perm[0]), weight=int(cand["cin"][perm[0]][0][0]))
    G.add_edge(("out", "c", S - 1, perm[S - 1]), "t", weight=int(cand["cout"][perm[S - 1]][S - 1][0]))
    for s in range(S - 1):
        for v in range(n):
            for u in range(n):
                if I.link[s, v, u] != ABSENT:
                    G.add_edge(("out", "b", s, u), ("in", "b", s + 1, v), weight=int(I.link[s, v, u]))
        c0, c1 = perm[s], perm[s + 1]
        for v in range(n):
            G.add_edge(("out", "c", s, c0), ("in", "b", s + 1, v), weight=int(cand["cout"][c0][s][v]))
        for u in range(n):
            G.add_edge(("out", "b", s, u), ("in", "c", s + 1, c1), weight=int(cand["cin"][c1][s + 1][u]))
        G.add_edge(("out", "c", s, c0), ("in", "c", s + 1, c1), weight=int(cand["cc"][c0][c1]))
    fl = nx.max_flow_min_cost(G, "s", "t")
    return sum(fl["s"].values()), nx.cost_of_flow(G, fl)


@pytest.mark.parametrize("seed", range(6))
def test_oracle_optimal_addition_vs_networkx(seed):
    """argmin over all 3! = 6 (and 4! = 24) placements equals an independent
    re-enumeration (networkx min-cost max-flow on a directly built graph)."""
    S = 3 if seed < 4 else 4
    cfg = gen.CONFIGS["addition"].with_(S=S, n=3, M=12)
    bt = gen.generate(cfg, seed, 1)
    I = oracle.instance_from_batch(bt, 0)
    cand = gen.generate_candidates(cfg, seed)
    best, perm, F, C = oracle.optimal_addition(I, cand)
    assert len(F) == len(C) == len(list(itertools.permutations(range(S))))
    perms = list(itertools.permutations(range(S)))
    ref = [_nx_placement(I, cand, p) for p in perms]
    assert [(int(f), int(c)) for f, c in zip(F, C)] == ref
    key = [(-f, c, k) for k, (f, c) in enumerate(ref)]
    assert best == min(key)[2] and perm == perms[best]


def test_oracle_addition_degenerate():
    """Zero-capacity candidates change nothing: every placement has the base (F, cost) and the
    first (lexicographic) placement wins the tie."""
    cfg = gen.CONFIGS["addition"].with_(S=3, n=3, M=9)
    bt = gen.generate(cfg, 1, 1)
    I = oracle.instance_from_batch(bt, 0)
    cand = gen.generate_candidates(cfg, 1)
    cand["cap"][:] = 0
    best, perm, F, C = oracle.optimal_addition(I, cand)
    base = oracle.ssp(I)
    assert best == 0 and tuple(perm) == (0, 1, 2)
    assert (F == base.F).all() and (C == base.cost).all()


def test_improvement_formula():
    """SPEC.md:699-701 examples."""
    assert oracle.improvement(10, 8) == pytest.approx(0.2)
    assert oracle.improvement(10, 10) == 0
    assert oracle.improvement(8, 10) == pytest.approx(-0.25)
    assert addition.improvement(10, 8) == pytest.approx(0.2)


def test_placement_ranks():
    for S in range(1, 7):
        for k, p in enumerate(itertools.permutations(range(S))):
            assert addition.placement(k, S) == list(p) and addition.placement_index(p) == k


def test_capacity_first_rule():
    """highest capacity to the highest-utilization stage, second to second;
    capacity ties -> lower candidate id, utilization ties -> lower stage."""
    # stage capacities 10, 4, 8 with F = 4: utilizations 0.4, 1.0, 0.5 -> ranked [1, 2, 0]
    perm = addition.capacity_first([5, 2, 7], [10, 4, 8], 4)
    assert perm == [1, 2, 0]  # cand 2 (cap 7) -> stage 1, cand 0 (5) -> stage 2, cand 1 (2) -> stage 0
    assert addition.capacity_first([3, 3], [5, 5], 2) == [0, 1]


@pytest.mark.gpu
@pytest.mark.parametrize("S,inst", [(3, 0), (4, 1), (5, 2), (5, 3)])
def test_gpu_optimal_addition_parity(S, inst):
    """Every placement's (F, cost) and the chosen placement equal the oracle's exhaustive run."""
    cfg = gen.CONFIGS["addition"].with_(S=S)
    bt = gen.generate(cfg, inst, 1)
    I = oracle.instance_from_batch(bt, 0)
    cand = gen.generate_candidates(cfg, inst)
    best, perm, F, C = oracle.optimal_addition(I, cand)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    r = addition.optimal_addition(d(I.cap_eff()), d(I.src), d(I.snk), d(I.link), d(cand["cap"]), d(cand["cin"]),
                                  d(cand["cout"]), d(cand["cc"]), I.M, max_cap=cfg.max_cap, chunk=37)
    assert np.array_equal(r["all_F"].cpu().numpy(), F) and np.array_equal(r["all_cost"].cpu().numpy(), C)
    assert r["best_index"] == best and r["perm"] == list(perm)


@pytest.mark.gpu
def test_gpu_optimal_addition_full_setting_sampled():
    """Setting 1 at full size (8 stages, 40,320 placements): sampled placements and the chosen one
    against the oracle solved one at a time."""
    cfg = gen.CONFIGS["addition"]
    bt = gen.generate(cfg, 0, 1)
    I = oracle.instance_from_batch(bt, 0)
    cand = gen.generate_candidates(cfg, 0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    r = addition.optimal_addition(d(I.cap_eff()), d(I.src), d(I.snk), d(I.link), d(cand["cap"]), d(cand["cin"]),
                                  d(cand["cout"]), d(cand["cc"]), I.M, max_cap=cfg.max_cap)
    F, C = r["all_F"].cpu().numpy(), r["all_cost"].cpu().numpy()
    rng = np.random.default_rng(5)
    for k in list(rng.integers(0, len(F), 40)) + [r["best_index"]]:
        o = oracle.ssp(oracle.placed_instance(I, cand, addition.placement(int(k), cfg.S)))
        assert (int(F[k]), int(C[k])) == (o.F, o.cost), k
    key = np.lexsort((np.arange(len(F)), C, -F))
    assert int(key[0]) == r["best_index"]
