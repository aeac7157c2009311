"""Pins of the oracle's exact solve against what the paper and the
mathematics fix -- worked examples, brute force, closed forms, an independent network
simplex, scipy HiGHS LP, networkx, and certificates.  CPU only."""
import os

import numpy as np
import pytest

import gen
import oracle
from oracle import ABSENT, Instance

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


def golden(kind):
    out = []
    for line in open(GOLD):
        line = line.split("#")[0].split()
        if line and line[0] == kind:
            out.append(line[1:])
    return out


def rand_instance(rng, S, n, M, cap_hi=3, cost_hi=20, dead_p=0.0, absent_p=0.0, cost_lo=1, zero_cost=False):
    cap = rng.integers(1, cap_hi + 1, (S, n))
    lo = 0 if zero_cost else cost_lo
    src = rng.integers(lo, cost_hi + 1, n)
    snk = rng.integers(lo, cost_hi + 1, n)
    link = rng.integers(lo, cost_hi + 1, (max(S - 1, 0), n, n))
    link = np.where(rng.random(link.shape) < absent_p, ABSENT, link)
    src = np.where(rng.random(n) < absent_p / 2, ABSENT, src)
    snk = np.where(rng.random(n) < absent_p / 2, ABSENT, snk)
    alive = (rng.random((S, n)) >= dead_p).astype(np.uint8)
    return Instance(S, n, cap_hi, M, cap, src, snk, link, alive)


# ---------------------------------------------------------------- worked examples
def test_eq1_spec_examples():
    for c_i, c_j, lij, lji, bij, bji, size, want in (map(int, r) for r in golden("eq1")):
        # one-node stages: D (loc 0) -> relay (loc 1); use the src arc (c_D = 0) and a 2-stage link
        comp = np.array([[c_i], [c_j]], np.int32)
        loc = np.array([[0], [1]], np.int32)
        lat = np.array([[0, lij], [lji, 0]], np.int32)
        bw = np.array([[1, bij], [bji, 1]], np.int32)
        _, _, link = oracle.eq1(2, 1, 2, comp, loc, 0, lat, bw, size)
        assert link[0, 0, 0] == want


def test_eq1_symmetry_and_data_node():
    """Eq. 1 is symmetric under swapping i and j; the data node has c_D = 0."""
    rng = np.random.default_rng(1)
    L = 4
    lat = rng.integers(1, 150, (L, L)).astype(np.int32)
    bw = rng.integers(50, 500, (L, L)).astype(np.int32)
    comp = rng.integers(50, 200, (2, 3)).astype(np.int32)
    loc = rng.integers(0, L, (2, 3)).astype(np.int32)
    src, snk, link = oracle.eq1(2, 3, L, comp, loc, 2, lat, bw, 1000)
    # swap stage roles: the reversed 2-stage instance gives the transposed tile
    src2, snk2, link2 = oracle.eq1(2, 3, L, comp[::-1].copy(), loc[::-1].copy(), 2, lat, bw, 1000)
    assert np.array_equal(link[0], link2[0].T)
    assert np.array_equal(src, snk2) and np.array_equal(snk, src2)
    # real-valued Eq. 1, doubled, vs the integer form: differs only by the floor
    for v in range(3):
        for u in range(3):
            a, b = loc[0, u], loc[1, v]
            d = (comp[0, u] + comp[1, v]) / 2 + (lat[a, b] + lat[b, a]) / 2 + 2 * 1000 / (bw[a, b] + bw[b, a])
            assert 0 <= 2 * d - link[0, v, u] < 1


def test_ssp_spec_examples():
    for r in golden("ssp"):
        S, n, M = map(int, r[:3])
        vals = list(map(int, r[3:]))
        cap = np.array(vals[: S * n]).reshape(S, n)
        src = np.array(vals[S * n: S * n + n])
        snk = np.array(vals[S * n + n: S * n + 2 * n])
        F, cost = vals[-2:]
        I = Instance(S, n, 3, M, cap, src, snk, np.zeros((0, n, n)))
        res = oracle.ssp(I)
        assert (res.F, res.cost) == (F, cost)
        assert oracle.network_simplex(I) == (F, cost)


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(60))
def test_ssp_vs_brute_force_tiny(seed):
    rng = np.random.default_rng(seed)
    I = rand_instance(rng, 3, 3, int(rng.integers(1, 9)), dead_p=0.15 if seed % 3 == 0 else 0,
                      absent_p=0.2 if seed % 4 == 1 else 0, zero_cost=seed % 5 == 2)
    res = oracle.ssp(I)
    assert (res.F, res.cost) == oracle.brute_force(I)


def test_ssp_vs_brute_force_generated_tiny():
    bt = gen.generate(gen.CONFIGS["tiny"], 0, 40)
    for b in range(40):
        I = oracle.instance_from_batch(bt, b)
        res = oracle.ssp(I)
        assert (res.F, res.cost) == oracle.brute_force(I)


# ---------------------------------------------------------------- network simplex / LP / networkx
@pytest.mark.parametrize("shape", [(2, 4, 6), (3, 5, 10), (4, 3, 7), (5, 6, 12), (1, 5, 9), (6, 4, 30)])
def test_ssp_vs_network_simplex(shape):
    S, n, M = shape
    for seed in range(25):
        rng = np.random.default_rng(1000 * S + seed)
        I = rand_instance(rng, S, n, M, cap_hi=4, dead_p=0.15 * (seed % 2), absent_p=0.25 * (seed % 3 == 0),
                          zero_cost=seed % 4 == 3)
        res = oracle.ssp(I)
        assert (res.F, res.cost) == oracle.network_simplex(I), (shape, seed)


def test_ssp_vs_network_simplex_configs():
    for name, B in (("gpt", 12), ("flow1", 10), ("flow3", 10), ("flow4", 10)):
        cfg = gen.CONFIGS[name]
        bt = gen.generate(cfg, 0, B)
        if cfg.cost_kind == gen.COST_EQ1:
            src, snk, link = oracle.eq1_batch(bt)
        else:
            src, snk, link = bt.src, bt.snk, bt.link
        for b in range(B):
            I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
            res = oracle.ssp(I)
            assert (res.F, res.cost) == oracle.network_simplex(I), (name, b)


def _lp(I: Instance):
    """Min-cost max-flow as two LPs with scipy HiGHS (node-arc incidence is totally unimodular)."""
    from scipy.optimize import linprog
    S, n = I.S, I.n
    arcs = []  # (tail, head, cost, cap)
    node = lambda kind, s, i: 2 + 2 * (s * n + i) + kind  # 0 in, 1 out  # noqa: E731
    ce = I.cap_eff()
    for i in range(n):
        if I.src[i] != ABSENT:
            arcs.append((0, node(0, 0, i), I.src[i], None))
        if I.snk[i] != ABSENT:
            arcs.append((node(1, S - 1, i), 1, I.snk[i], None))
    for s in range(S):
        for i in range(n):
            arcs.append((node(0, s, i), node(1, s, i), 0, int(ce[s, i])))
    for s in range(S - 1):
        for v in range(n):
            for u in range(n):
                if I.link[s, v, u] != ABSENT:
                    arcs.append((node(1, s, u), node(0, s + 1, v), int(I.link[s, v, u]), None))
    N = 2 + 2 * S * n
    E = len(arcs)
    Aeq = np.zeros((N - 2, E + 1))
    for e, (t, h, _, _) in enumerate(arcs):
        if t >= 2:
            Aeq[t - 2, e] -= 1
        if h >= 2:
            Aeq[h - 2, e] += 1
    # variable E = total flow F; s* emits F, which must be <= M
    src_row = np.zeros(E + 1)
    for e, (t, _, _, _) in enumerate(arcs):
        if t == 0:
            src_row[e] = 1
    src_row[E] = -1
    Aeq = np.vstack([Aeq, src_row])
    beq = np.zeros(Aeq.shape[0])
    bounds = [(0, c) for (_, _, _, c) in arcs] + [(0, I.M)]
    c1 = np.zeros(E + 1)
    c1[E] = -1
    r1 = linprog(c1, A_eq=Aeq, b_eq=beq, bounds=bounds, method="highs")
    F = round(-r1.fun)
    bounds[-1] = (F, F)
    c2 = np.array([a[2] for a in arcs] + [0], float)
    r2 = linprog(c2, A_eq=Aeq, b_eq=beq, bounds=bounds, method="highs")
    return F, round(r2.fun)


def test_ssp_vs_highs_lp():
    for seed in range(40):
        rng = np.random.default_rng(7000 + seed)
        S, n = int(rng.integers(1, 5)), int(rng.integers(1, 6))
        I = rand_instance(rng, S, n, int(rng.integers(1, 15)), cap_hi=4, dead_p=0.1, absent_p=0.15)
        res = oracle.ssp(I)
        assert (res.F, res.cost) == _lp(I), seed


def test_ssp_vs_networkx():
    nx = pytest.importorskip("networkx")
    for seed in range(40):
        rng = np.random.default_rng(9000 + seed)
        S, n = int(rng.integers(1, 5)), int(rng.integers(1, 6))
        I = rand_instance(rng, S, n, int(rng.integers(1, 15)), cap_hi=4, dead_p=0.1, absent_p=0.15, zero_cost=True)
        G = nx.DiGraph()
        ce = I.cap_eff()
        G.add_edge("s", "D", capacity=I.M, weight=0)
        for i in range(n):
            if I.src[i] != ABSENT:
                G.add_edge("D", ("in", 0, i), weight=int(I.src[i]))
            if I.snk[i] != ABSENT:
                G.add_edge(("out", S - 1, i), "t", weight=int(I.snk[i]))
        for s in range(S):
            for i in range(n):
                G.add_edge(("in", s, i), ("out", s, i), capacity=int(ce[s, i]), weight=0)
        for s in range(S - 1):
            for v in range(n):
                for u in range(n):
                    if I.link[s, v, u] != ABSENT:
                        G.add_edge(("out", s, u), ("in", s + 1, v), weight=int(I.link[s, v, u]))
        if "t" not in G:
            F, cost = 0, 0
        else:
            fl = nx.max_flow_min_cost(G, "s", "t")
            F = sum(fl["s"].values())
            cost = nx.cost_of_flow(G, fl)
        res = oracle.ssp(I)
        assert (res.F, res.cost) == (F, cost), seed


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("seed", range(30))
def test_closed_form_max_flow_complete_links(seed):
    """With complete inter-stage links, F* = min(M, min_s sum_i cap_eff[s][i])."""
    rng = np.random.default_rng(seed)
    S, n = int(rng.integers(1, 7)), int(rng.integers(1, 8))
    I = rand_instance(rng, S, n, int(rng.integers(1, 40)), cap_hi=5, dead_p=0.2)
    want = min(I.M, int(I.cap_eff().sum(axis=1).min()))
    assert oracle.ssp(I).F == want


@pytest.mark.parametrize("seed", range(30))
def test_closed_form_separable_costs(seed):
    """d(u,v) = x_u + y_v (Eq. 1 with lambda = size = 0 is this with x = y = c): every path of the
    flow pays its node weights, and the stage-wise greedy is optimal."""
    rng = np.random.default_rng(100 + seed)
    S, n = int(rng.integers(1, 6)), int(rng.integers(1, 7))
    x = rng.integers(0, 30, (S, n))
    y = rng.integers(0, 30, (S, n))
    cD_out, cD_in = int(rng.integers(0, 10)), int(rng.integers(0, 10))
    src = cD_out + y[0]
    snk = x[S - 1] + cD_in
    link = np.zeros((max(S - 1, 0), n, n), np.int64)
    for s in range(S - 1):
        link[s] = x[s][None, :] + y[s + 1][:, None]  # [v][u]
    cap = rng.integers(1, 5, (S, n))
    alive = (rng.random((S, n)) >= 0.2).astype(np.uint8)
    M = int(rng.integers(1, 30))
    I = Instance(S, n, 5, M, cap, src, snk, link, alive)
    ce = I.cap_eff()
    F = min(M, int(ce.sum(axis=1).min()))
    want = (cD_out + cD_in) * F
    for s in range(S):
        w = np.repeat(x[s] + y[s], ce[s])
        want += int(np.sort(w)[:F].sum())
    res = oracle.ssp(I)
    assert (res.F, res.cost) == (F, want)


def test_closed_form_uniform_costs():
    """All arcs cost d: every path has S+1 arcs, cost* = F (S+1) d."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        S, n, d = int(rng.integers(1, 6)), int(rng.integers(1, 6)), int(rng.integers(0, 9))
        cap = rng.integers(1, 4, (S, n))
        I = Instance(S, n, 3, int(rng.integers(1, 20)), cap, np.full(n, d), np.full(n, d), np.full((max(S - 1, 0), n, n), d))
        res = oracle.ssp(I)
        assert res.cost == res.F * (S + 1) * d


def test_closed_form_assignment():
    """S=2, unit capacities, M = n: cost* = sum(src) + sum(snk) + LAP(C) (scipy linear_sum_assignment)."""
    from scipy.optimize import linear_sum_assignment
    rng = np.random.default_rng(6)
    for _ in range(20):
        n = int(rng.integers(1, 8))
        link = rng.integers(0, 50, (1, n, n))
        src, snk = rng.integers(0, 20, n), rng.integers(0, 20, n)
        I = Instance(2, n, 1, n, np.ones((2, n)), src, snk, link)
        r, c = linear_sum_assignment(link[0])
        res = oracle.ssp(I)
        assert (res.F, res.cost) == (n, int(src.sum() + snk.sum() + link[0][r, c].sum()))


# ---------------------------------------------------------------- certificates and structure
def test_certificates_generated_configs():
    for name, B in (("tiny", 50), ("gpt", 20), ("llama", 3), ("churn", 2), ("flow2", 10)):
        cfg = gen.CONFIGS[name]
        bt = gen.generate(cfg, 0, B)
        if cfg.cost_kind == gen.COST_EQ1:
            src, snk, link = oracle.eq1_batch(bt)
        else:
            src, snk, link = bt.src, bt.snk, bt.link
        for b in range(B):
            I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
            r = oracle.ssp(I)
            assert oracle.certify(I, r.F, r.cost, r.node_flow, r.src_flow, r.snk_flow, r.arc_flow) == 0, (name, b)
            assert r.F == min(I.M, int(I.cap_eff().sum(axis=1).min())) or (link[b] == ABSENT).any()


def test_certificate_rejects_corruptions():
    """The certificate is a real check: it rejects a suboptimal, a non-maximal and a non-conserving flow."""
    rng = np.random.default_rng(11)
    I = rand_instance(rng, 3, 4, 6)
    r = oracle.ssp(I)
    assert oracle.certify(I, r.F, r.cost, r.node_flow, r.src_flow, r.snk_flow, r.arc_flow) == 0
    bad = r.arc_flow.copy()
    s, v, u = np.argwhere(bad > 0)[0]
    bad[s, v, u] -= 1
    assert oracle.certify(I, r.F, r.cost, r.node_flow, r.src_flow, r.snk_flow, bad) != 0
    # a max flow rerouted onto a strictly worse path: swap one unit to the most expensive parallel arc
    z = lambda *a: oracle.certify(I, *a)  # noqa: E731
    assert z(r.F, r.cost + 1, r.node_flow, r.src_flow, r.snk_flow, r.arc_flow) != 0
    # half flow is not maximum
    I2 = Instance(1, 2, 1, 2, np.ones((1, 2)), np.array([1, 1]), np.array([1, 1]), np.zeros((0, 2, 2)))
    assert oracle.certify(I2, 1, 2, np.array([[1, 0]]), np.array([1, 0]), np.array([1, 0]), np.zeros((0, 2, 2))) == 7


def test_suboptimal_detected_by_certificate():
    """A feasible max flow that is not min cost fails the optimality (negative cycle) check."""
    link = np.array([[[1, 10], [10, 1]]])  # [v][u]: u0->v0 1, u1->v1 1, crosses 10
    I = Instance(2, 2, 1, 2, np.ones((2, 2)), np.zeros(2), np.zeros(2), link)
    cross = np.array([[[0, 1], [1, 0]]])
    ones = np.ones((2, 2))
    assert oracle.certify(I, 2, 20, ones, np.ones(2), np.ones(2), cross) == 8
    assert oracle.certify(I, 2, 2, ones, np.ones(2), np.ones(2), np.array([[[1, 0], [0, 1]]])) == 0


def test_cost_curve_convex_and_augmentations():
    """cost(F') over F' = 0..F* is convex and piecewise linear (SSP path costs are non-decreasing)."""
    for seed in range(15):
        rng = np.random.default_rng(300 + seed)
        I = rand_instance(rng, 4, 4, 12, cap_hi=3)
        r = oracle.ssp(I, curve=True)
        inc = np.diff(r.curve)
        assert (np.diff(inc) >= 0).all()
        assert r.curve[-1] == r.cost
        assert 1 <= r.A <= max(r.F, 1) or r.F == 0


def test_zero_and_degenerate():
    # empty stage (all dead) -> flow 0 (not an error: SURVEY 8(b) errors)
    I = Instance(3, 2, 2, 5, np.full((3, 2), 2), np.ones(2), np.ones(2), np.ones((2, 2, 2)),
                 np.array([[1, 1], [0, 0], [1, 1]], np.uint8))
    r = oracle.ssp(I)
    assert (r.F, r.cost, r.A) == (0, 0, 0)
    # M = 0
    I = Instance(2, 2, 2, 0, np.full((2, 2), 2), np.ones(2), np.ones(2), np.ones((1, 2, 2)))
    assert (oracle.ssp(I).F, oracle.network_simplex(I)) == (0, (0, 0))
    # all links absent
    I = Instance(2, 2, 2, 3, np.full((2, 2), 2), np.ones(2), np.ones(2), np.full((1, 2, 2), ABSENT))
    assert oracle.ssp(I).F == 0 and oracle.network_simplex(I) == (0, 0)


def test_ssp_needs_reverse_arcs():
    """An instance where the second augmenting path must cancel flow on a first-path arc:
    greedy path-by-path routing is suboptimal, SSP (with residual reverse arcs) is optimal."""
    # stage 0: a0,a1; stage 1: b0,b1.  a0->b0 = 1, a0->b1 = 5, a1->b0 = 5, a1->b1 = 100
    link = np.array([[[1, 5], [5, 100]]])  # [v][u]
    I = Instance(2, 2, 1, 2, np.ones((2, 2)), np.zeros(2), np.zeros(2), link)
    r = oracle.ssp(I)
    assert (r.F, r.cost) == (2, 10)
    assert r.arc_flow[0, 0, 0] == 0  # the first (cost 1) arc was cancelled by the second path
    assert oracle.brute_force(I) == (2, 10)
