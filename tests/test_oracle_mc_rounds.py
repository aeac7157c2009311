"""Pins of the multi-data-node rounds oracle (MC-SYNC), CPU only:
a hand-derived trace with two data nodes ("each data node ... its own flow back"), the
reduction to the pinned single-commodity rounds at K = 1 (state equal round by round), and the
invariants every round on flow-test settings 5 and 6: capacity, pairing
bijectivity, every chain of SRC_k made of slots tagged k and ending at SNK_k."""
import numpy as np
import pytest

import gen
import oracle
from oracle import ABSENT, Instance

NONE = -1


def two_node_instance():
    """S=2, n=2, caps 1; stage 0 = {a0, a1}, stage 1 = {b0, b1}; links a0->b0 = 10, a0->b1 = 1,
    a1->b0 = 1, a1->b1 = 10; data node D0: src [1, 50], snk [1, 50]; D1: src [50, 1], snk [50, 1];
    one microbatch each."""
    link = np.array([[[10, 1], [1, 10]]], np.int32)  # [s][v][u]
    I = Instance(2, 2, 1, 1, np.ones((2, 2)), np.zeros(2), np.zeros(2), link)
    return I, [[1, 50], [50, 1]], [[1, 50], [50, 1]], [1, 1]


def test_mc_hand_trace_two_data_nodes():
    """Round 1: b0 and b1 (stable, last stage) each take the cheaper data-node sink: b0 -> SNK_0
    (snk 1 < 50), b1 -> SNK_1; both become OUT with tags 0 / 1.  Round 2: a0 (stable) takes the
    cheapest (target, data node) pair: b1 for D1 (1 + 1 = 2) over b0 for D0 (10 + 1); a1 takes b0
    for D0 (1 + 1); their slots become OUT with tags 1 / 0.  Round 3: each data node requests only
    advertisers of its own tag: D0 pairs a1 (50 + 2 = 52), D1 pairs a0 (52).  The Change a0 <-> a1
    would mix the data nodes (tags 1 and 0): never proposed.  Rounds 4-8 are quiet: (F, cost) =
    ([1, 1], [52, 52]) after 8 rounds, although D0-a0-b0-D0 and D1-a1-b1-D1 would cost 12 each --
    the greedy requests are myopic (the paper's flows approximate the optimum)."""
    I, srcs, snks, M = two_node_instance()
    R = oracle.McRounds(I, srcs, snks, M, T0=0.0, seed=5)
    R.run(1)
    st = R.export()
    assert list(st["down"].ravel()) == [NONE, NONE, -2, -3] and list(st["tag"].ravel()) == [-1, -1, 0, 1]
    assert list(st["snk_up"].ravel()) == [2, 3]
    R.run(1)
    st = R.export()
    assert list(st["down"].ravel()) == [3, 2, -2, -3] and list(st["tag"].ravel()) == [1, 0, 0, 1]
    r = R.run(1)
    st = R.export()
    assert list(st["src_down"].ravel()) == [1, 0]
    assert list(r["F_dec"]) == [1, 1] and list(r["cost_dec"]) == [52, 52] and r["dangling"] == 0
    r = R.run(100)
    assert r["rounds"] == 5 and list(r["cost_dec"]) == [52, 52] and R.export()["round"] == 8


@pytest.mark.parametrize("name", ["flow1", "flow3", "tiny", "gpt"])
def test_mc_single_data_node_is_the_pinned_rounds(name):
    """K = 1: MC-SYNC is GWTF-SYNC (every rule reduces to the single-commodity one; pointer
    encodings coincide), so the full state must equal the pinned oracle's after every round."""
    cfg = gen.CONFIGS[name]
    bt = gen.generate(cfg, 0, 3)
    src, snk, link = oracle.eq1_batch(bt) if cfg.cost_kind == gen.COST_EQ1 else (bt.src, bt.snk, bt.link)
    for b in range(3):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        R1 = oracle.Rounds(I, seed=7, inst_id=b)
        Rk = oracle.McRounds(I, [I.src], [I.snk], [I.M], seed=7, inst_id=b)
        for _ in range(min(cfg.max_rounds, 80)):
            a = R1.run(1)
            c = Rk.run(1)
            assert (a["F_dec"], a["cost_dec"], a["dangling"]) == (int(c["F_dec"][0]), int(c["cost_dec"][0]), c["dangling"])
            s1, sk = R1.export(), Rk.export()
            for key in ("up", "down", "kacc", "deny"):
                assert np.array_equal(s1[key], sk[key]), key
            assert np.array_equal(s1["src_down"], sk["src_down"][0]) and np.array_equal(s1["snk_up"], sk["snk_up"][0])


def _check_mc_invariants(I, st, K, Mmax, M):
    S, n, MC = I.S, I.n, I.max_cap
    ce = I.cap_eff()
    up, dn, tg = st["up"].reshape(-1), st["down"].reshape(-1), st["tag"].reshape(-1)
    for p in range(S * n * MC):
        v, j = divmod(p, MC)
        s, i = divmod(v, n)
        if j >= ce[s, i]:
            assert up[p] == NONE and dn[p] == NONE
            continue
        if dn[p] >= 0:
            assert up[dn[p]] == p and tg[dn[p]] == tg[p]
        elif dn[p] <= -2:
            k, x = divmod(-2 - dn[p], Mmax)
            assert s == S - 1 and st["snk_up"][k, x] == p and tg[p] == k
        if up[p] >= 0:
            assert dn[up[p]] == p and tg[up[p]] == tg[p]
        elif up[p] <= -2:
            k, x = divmod(-2 - up[p], Mmax)
            assert s == 0 and st["src_down"][k, x] == p and tg[p] == k
    for k in range(K):  # unused data-node slots stay empty
        assert (st["src_down"][k, M[k]:] == NONE).all() and (st["snk_up"][k, M[k]:] == NONE).all()


@pytest.mark.parametrize("name", ["flow5", "flow6"])
def test_mc_invariants_flow_settings_5_6(name):
    cfg = gen.CONFIGS[name]
    K = cfg.extra["data_nodes"]
    bt = gen.generate(cfg, 0, 4)
    xs, xk = gen.generate_data_nodes(cfg, 0, 4, K)
    for b in range(4):
        I = oracle.instance_from_batch(bt, b)
        srcs = [bt.src[b]] + [xs[k][b] for k in range(K - 1)]
        snks = [bt.snk[b]] + [xk[k][b] for k in range(K - 1)]
        Ms = [cfg.M // K] * K
        R = oracle.McRounds(I, srcs, snks, Ms, seed=3, inst_id=b)
        for _ in range(120):
            r = R.run(1)
            st = R.export()
            _check_mc_invariants(I, st, K, max(Ms), Ms)
            assert R.digest() == R.digest()
        # every data node's routed flow is feasible for it alone: at most the single-commodity max flow
        for k in range(K):
            Ik = Instance(I.S, I.n, I.max_cap, Ms[k], I.cap, srcs[k], snks[k], I.link, I.alive)
            assert r["F_dec"][k] <= oracle.ssp(Ik).F
        # and together at most what the shared relays can carry
        assert r["F_dec"].sum() <= oracle.ssp(Instance(I.S, I.n, I.max_cap, sum(Ms), I.cap, srcs[0], snks[0],
                                                        I.link, I.alive)).F


def in_slot_case():
    """S=2, n=2, caps 1, K=2, one microbatch each; every link 1, src_k = [1, 1], snk_0 = [10, 10],
    snk_1 = [1, 1] (D1's sink is the cheaper one from both last-stage relays).  Start (round 20):
    SRC_0 -> a0 -> b0, and b0's slot is IN (tag 0: its chain came from D0, its downstream is gone);
    everything else empty.
      r20: b0 holds unpaired inflow of D0, so it may only ask D0's sink -- 10, although D1's costs 1
           (each data node gets its own flow back); b1 (stable) takes the cheaper D1-sink.
      r21: a1 (stable) pairs with b1's tag-1 outflow (1 + 1 = 2).
      r22: D1 pairs a1 (1 + 2 = 3).  Change a0 <-> a1 or b0 <-> b1 would mix D0's and D1's chains.
      r23-r27 quiet: (F, cost) = ([1, 1], [12, 3]) after 8 rounds.
    (A requester holding an IN slot asking any data node would send D0's chain to D1's sink.)"""
    from tests.pin_cases import D, NONE as N_, state
    I = Instance(2, 2, 1, 1, np.ones((2, 2)), np.zeros(2), np.zeros(2), np.ones((1, 2, 2), np.int32))
    st = state(2, 2, 1, 1, {0: (D(0), 2), 2: (0, N_)}, src_down=[[0], [N_]], snk_up=[[N_], [N_]], rnd=20)
    st["tag"] = np.array([0, -1, 0, -1], np.int32).reshape(2, 2, 1)
    return I, [[1, 1], [1, 1]], [[10, 10], [1, 1]], [1, 1], st


def test_mc_in_slot_asks_its_own_data_node():
    I, srcs, snks, M, st0 = in_slot_case()
    R = oracle.McRounds(I, srcs, snks, M, T0=0.0, seed=4)
    R.import_state(st0)
    R.run(1)
    st = R.export()
    assert list(st["down"].ravel()) == [2, NONE, -2, -3] and list(st["tag"].ravel()) == [0, -1, 0, 1]
    r = R.run(100)
    assert r["rounds"] == 7 and list(r["F_dec"]) == [1, 1] and list(r["cost_dec"]) == [12, 3]
    assert R.export()["round"] == 28
    bad = {k: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v) for k, v in st0.items()}
    bad["tag"].reshape(-1)[2] = 1  # b0's slot tagged 1 under a0's tag-0 slot: not a valid tagged pairing
    with pytest.raises(ValueError):
        oracle.McRounds(I, srcs, snks, M, T0=0.0).import_state(bad)
