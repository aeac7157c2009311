"""Pins of the oracle's warm-start rerouting (PAPER.md:188 reroute after a
failure, :274-288 crash handling).  The optimum's (F, cost) is unique, so the warm result must
equal what the independent network simplex and brute force find on the churned instance, and
its assignment must pass the certificate (conservation, capacity, maximality, no negative
residual cycle).  CPU only."""
import numpy as np
import pytest

import oracle
from oracle import ABSENT, Instance
from tests.test_oracle_ssp import rand_instance


def churned(rng, I, kill_p=0.25, absent_p=0.1, recost_p=0.1, revive=True):
    alive = I.alive.copy()
    kill = rng.random(alive.shape) < kill_p
    alive[kill] = 0
    if revive:  # joins: some dead relays come back
        alive[(I.alive == 0) & (rng.random(alive.shape) < 0.5)] = 1
    link = I.link.copy()
    live_links = link != ABSENT
    link[(rng.random(link.shape) < absent_p) & live_links] = ABSENT
    rec = (rng.random(link.shape) < recost_p) & (link != ABSENT)
    link[rec] = rng.integers(1, 40, int(rec.sum()))
    src = I.src.copy()
    src[(rng.random(I.n) < absent_p) & (src != ABSENT)] = ABSENT
    return Instance(I.S, I.n, I.max_cap, I.M, I.cap, src, I.snk.copy(), link, alive)


def check(I0, I1, brute=False):
    base = oracle.ssp(I0)
    r, st = oracle.warm_reroute(I0, base, I1)
    F_ns, c_ns = oracle.network_simplex(I1)
    assert (r.F, r.cost) == (F_ns, c_ns)
    assert oracle.certify(I1, r.F, r.cost, r.node_flow, r.src_flow, r.snk_flow, r.arc_flow) == 0
    if brute:
        assert (r.F, r.cost) == oracle.brute_force(I1)
    return base, r, st


def test_warm_no_churn_is_identity():
    """No churn: nothing stripped, no cycle (the base flow is optimal), no augmentation; same flow."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        I = rand_instance(rng, 4, 5, 12, cap_hi=4)
        base, r, st = check(I, I)
        assert st == {"stripped": 0, "cycles": 0, "augment": 0}
        assert np.array_equal(r.node_flow, base.node_flow) and np.array_equal(r.arc_flow, base.arc_flow)


def test_warm_matches_brute_force_tiny():
    rng = np.random.default_rng(12)
    for _ in range(40):
        I = rand_instance(rng, 3, 3, int(rng.integers(1, 9)), cap_hi=3, dead_p=0.1, absent_p=0.1)
        check(I, churned(rng, I), brute=True)


@pytest.mark.parametrize("S,n,M", [(4, 6, 16), (6, 8, 40), (8, 12, 64)])
def test_warm_matches_network_simplex(S, n, M):
    rng = np.random.default_rng(100 + S)
    stripped = cycles = 0
    for _ in range(12):
        I = rand_instance(rng, S, n, M, cap_hi=5, cost_hi=30, absent_p=0.05)
        _, _, st = check(I, churned(rng, I))
        stripped += st["stripped"]
        cycles += st["cycles"]
    assert stripped > 0  # the churn really removed carried flow


def test_warm_needs_cycle_cancelling():
    """Hand-built: 2 stages x 2 relays, M = 2, base optimum routes 0->0 and 1->1 (cost 1 each).
    Churn removes link 1->1 and re-costs 0->0 to 30 and 0->1 to 2.  The kept unit on 0->0 (now 30)
    is not min-cost for F = 1 (0->1 costs 2): a negative residual cycle exists and must be
    cancelled; the re-solve then adds 1->0 (10).  Optimum 2 + 10 = 12 (brute force agrees)."""
    S, n, M = 2, 2, 2
    cap = np.array([[1, 1], [1, 2]])
    src = np.array([0, 0]); snk = np.array([0, 0])
    link = np.array([[[1, 10], [10, 1]]])  # link[0][v][u]
    I0 = Instance(S, n, 2, M, cap, src, snk, link)
    link1 = link.copy(); link1[0, 1, 1] = ABSENT; link1[0, 1, 0] = 2; link1[0, 0, 0] = 30
    I1 = Instance(S, n, 2, M, cap, src, snk, link1)
    _, r, st = check(I0, I1, brute=True)
    assert st["cycles"] >= 1 and r.cost == 12 and r.F == 2
