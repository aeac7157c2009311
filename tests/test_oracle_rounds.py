"""Pins of the oracle's decentralized rounds -- hand-derived traces of the
paper's worked examples (PAPER.md:256 Change, :258 Redirect), annealing thresholds
(PAPER.md:259 with SPEC.md:288-289/:307/:316), invariants and quality bounds
(SPEC.md:736).  CPU only."""
import os

import numpy as np
import pytest

import gen
import oracle
from oracle import ABSENT, Instance, OBJ_MINIMAX, OBJ_SUM

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")
NONE = -1


def golden(kind):
    return [l.split("#")[0].split()[1:] for l in open(GOLD) if l.split("#")[0].split()[:1] == [kind]]


# ------------------------------------------------------------------ annealing thresholds
def test_anneal_table_spec_examples():
    tbl, width, K = oracle.anneal_table(1.7, 0.95)
    for T0, alpha, delta, u, accept in golden("anneal"):
        t, _, _ = oracle.anneal_table(float(T0), float(alpha))
        h32 = int(float(u) * (1 << 32))  # the draw (h >> 32) that corresponds to U(0,1) = u
        assert (h32 < int(t[0, int(delta)])) == bool(int(accept))
    assert (width, K) == (38, 71)           # exp(-38/1.7) < 2^-32 <= exp(-37/1.7); 1.7*0.95^71*22.18 < 1
    assert tbl[0, 2] == 1324418311 and tbl[0, 1] == 2385022711
    # T = T0 alpha^k: monotone in k and in delta, and zero at the table edges
    assert (np.diff(tbl[:, 1:].astype(np.int64), axis=0) <= 0).all()
    assert (np.diff(tbl[:, 1:].astype(np.int64), axis=1) <= 0).all()
    assert tbl[K, 1] == 0 and tbl[K - 1, 1] > 0
    t0, w0, K0 = oracle.anneal_table(0.0, 0.95)  # annealing off
    assert (w0, K0) == (1, 0) and not t0.any()


# ------------------------------------------------------------------ hand traces
def run_digest_trace(I, rounds, **kw):
    R = oracle.Rounds(I, **kw)
    out = []
    for _ in range(rounds):
        st = R.run(1)
        out.append((st, R.export()))
    return R, out


def test_trace_spec_example_one_stage():
    """SPEC.md:187 instance, round by round: R1 both relays pair with D-sink; R2 D pairs A
    (cost 4 = 2+2); R3 D pairs B -> (2, 10); then W=5 quiet rounds."""
    I = Instance(1, 2, 1, 2, np.ones((1, 2)), np.array([2, 3]), np.array([2, 3]), np.zeros((0, 2, 2)))
    R = oracle.Rounds(I, seed=123, T0=1.7)
    r1 = R.run(1)
    st = R.export()
    assert list(st["down"].ravel()) == [-2, -3] and list(st["snk_up"]) == [0, 1] and r1["F_dec"] == 0
    r2 = R.run(1)
    st = R.export()
    assert list(st["src_down"]) == [0, NONE] and (r2["F_dec"], r2["cost_dec"]) == (1, 4)
    r3 = R.run(1)
    assert (r3["F_dec"], r3["cost_dec"]) == (2, 10)
    rest = R.run(100)
    assert rest["rounds"] == 5 and (rest["F_dec"], rest["cost_dec"]) == (2, 10)
    assert oracle.ssp(I).cost == 10


def change_instance():
    # stage 0 = {n1 (0), n3 (1)}, stage 1 = {n2 (0), n4 (1)}; d(n1,n2)=3, d(n3,n4)=8, d(n1,n4)=6, d(n3,n2)=6
    link = np.zeros((1, 2, 2), np.int32)
    link[0, 0, 0], link[0, 0, 1], link[0, 1, 0], link[0, 1, 1] = 3, 6, 6, 8  # [v][u]
    return Instance(2, 2, 1, 2, np.ones((2, 2)), np.zeros(2), np.zeros(2), link)


@pytest.mark.parametrize("seed", [0, 1, 99])
def test_trace_change_example_minimax(seed):
    """PAPER.md:256 embedded in a whole instance, MINIMAX, annealing off.  The trace
    is RNG-independent (n = 2 forces the peer, one PAIRED slot each forces the slots)."""
    I = change_instance()
    R = oracle.Rounds(I, seed=seed, T0=0.0, objective=OBJ_MINIMAX)
    R.run(1)  # R1: n2, n4 pair with D-sink
    st = R.export()
    assert list(st["down"][1, :, 0]) == [-2, -3]
    R.run(1)  # R2: n1 -> n2 granted, n3 -> n2 rejected (lower gid wins)
    st = R.export()
    assert st["down"][0, 0, 0] == 2 * 1 + 0 and st["down"][0, 1, 0] == NONE
    r = R.run(1)  # R3: n3 -> n4; D pairs n1 (F = 1, cost 3)
    assert (r["F_dec"], r["cost_dec"]) == (1, 3)
    r = R.run(1)  # R4: D pairs n3 (cost 11); n1 and n3 both propose the swap (max 8 -> 6); n1 wins
    st = R.export()
    assert (r["F_dec"], r["cost_dec"]) == (2, 12)
    assert st["down"][0, 0, 0] == 3 and st["down"][0, 1, 0] == 2  # n1 -> n4, n3 -> n2
    assert list(st["kacc"][0]) == [1, 0]
    r = R.run(100)
    assert r["rounds"] == 5 and (r["F_dec"], r["cost_dec"]) == (2, 12)  # stops after round 9
    assert R.export()["round"] == 9


def test_trace_change_example_sum():
    """Same instance, SUM objective: the swap has delta = +1 and annealing is off -> rejected;
    the result is the SSP optimum (2, 11).  Pins that MINIMAX mode is not SUM-optimal."""
    I = change_instance()
    R = oracle.Rounds(I, seed=5, T0=0.0, objective=OBJ_SUM)
    r = R.run(1000)
    assert (r["F_dec"], r["cost_dec"]) == (2, 11) and R.export()["round"] == 9
    s = oracle.ssp(I)
    assert (s.F, s.cost) == (2, 11)


def redirect_instance():
    # stage 0 = {a, dead}, stage 1 = {b (0), x (1)}, stage 2 = {c, dead}; d(a,b)=5 d(b,c)=6 d(a,x)=4 d(x,c)=5
    link = np.full((2, 2, 2), ABSENT, np.int32)
    link[0, 0, 0], link[0, 1, 0] = 5, 4   # a -> b, a -> x
    link[1, 0, 0], link[1, 0, 1] = 6, 5   # b -> c, x -> c
    alive = np.array([[1, 0], [1, 1], [1, 0]], np.uint8)
    return Instance(3, 2, 1, 1, np.ones((3, 2)), np.zeros(2), np.zeros(2), link, alive)


def test_trace_redirect_example():
    """PAPER.md:258 embedded, SUM, annealing off.  Pins the phase order: x proposes the
    Redirect (11 -> 9) in the same round as the grant a -> b it acts on (R4 reads the post-R3 state)."""
    I = redirect_instance()
    R = oracle.Rounds(I, seed=7, T0=0.0)
    R.run(1)  # c pairs D-sink
    R.run(1)  # b and x request c; b wins
    st = R.export()
    assert st["down"][1, 0, 0] == 2 * 2 + 0 and st["down"][1, 1, 0] == NONE
    R.run(1)  # a -> b granted; x redirects a -> x -> c in the same round; b freed
    st = R.export()
    x_slot = 3 * 1 + 0  # gid 3 (stage 1, idx 1), slot 0
    assert st["down"][0, 0, 0] == x_slot and st["up"][1, 0, 0] == NONE and st["down"][1, 0, 0] == NONE
    assert st["kacc"][1, 1] == 1
    r = R.run(1)  # D pairs a -> (1, 9)
    assert (r["F_dec"], r["cost_dec"]) == (1, 9)
    r = R.run(100)
    assert r["rounds"] == 5 and (r["F_dec"], r["cost_dec"]) == (1, 9) and R.export()["round"] == 9
    assert oracle.ssp(I).cost == 9


# ------------------------------------------------------------------ invariants
def check_invariants(I: Instance, st: dict):
    """Capacity and pairing bijectivity of a round state."""
    S, n, MC, M = I.S, I.n, I.max_cap, I.M
    ce = I.cap_eff()
    up, dn = st["up"], st["down"]
    for s in range(S):
        for i in range(n):
            for j in range(MC):
                u, d = up[s, i, j], dn[s, i, j]
                if j >= ce[s, i]:
                    assert u == NONE and d == NONE
                    continue
                p = (s * n + i) * MC + j
                if d >= 0:
                    ds, di, dj = d // (n * MC), (d // MC) % n, d % MC
                    assert ds == s + 1 and up[ds, di, dj] == p
                    assert I.link[s, di, i] != ABSENT
                elif d <= -2:
                    assert s == S - 1 and st["snk_up"][-2 - d] == p and I.snk[i] != ABSENT
                if u >= 0:
                    us, ui, uj = u // (n * MC), (u // MC) % n, u % MC
                    assert us == s - 1 and dn[us, ui, uj] == p
                elif u <= -2:
                    assert s == 0 and st["src_down"][-2 - u] == p and I.src[i] != ABSENT
    for k in range(M):
        if st["src_down"][k] >= 0:
            d = st["src_down"][k]
            assert up.reshape(-1)[d] == -2 - k
        if st["snk_up"][k] >= 0:
            u = st["snk_up"][k]
            assert dn.reshape(-1)[u] == -2 - k


def flow_of_state(I, st):
    """Flow f(i,j) induced by the complete chains of a state (for SPEC.md:330 conservation)."""
    S, n, MC = I.S, I.n, I.max_cap
    dn = st["down"].reshape(-1)
    F, cost = 0, 0
    for k in range(I.M):
        p = st["src_down"][k]
        if p < 0:
            continue
        c = int(I.src[(p // MC) % n])
        ok = True
        while p >= 0:
            d = dn[p]
            s, i = p // (n * MC), (p // MC) % n
            if d == NONE:
                ok = False
                break
            c += int(I.snk[i]) if d <= -2 else int(I.link[s, (d // MC) % n, i])
            p = d
        if ok:
            F, cost = F + 1, cost + c
    return F, cost


@pytest.mark.parametrize("name", ["tiny", "flow1", "flow3", "gpt"])
def test_invariants_every_round(name):
    cfg = gen.CONFIGS[name]
    bt = gen.generate(cfg, 0, 6)
    src, snk, link = oracle.eq1_batch(bt) if cfg.cost_kind == gen.COST_EQ1 else (bt.src, bt.snk, bt.link)
    for b in range(6):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        R = oracle.Rounds(I, seed=3, inst_id=b)
        for _ in range(60):
            r = R.run(1)
            st = R.export()
            check_invariants(I, st)
            assert (r["F_dec"], r["cost_dec"]) == flow_of_state(I, st)
            assert R.digest() == oracle.digest_state(st, I.S, I.n, I.max_cap, I.M)


def test_determinism_and_seed_dependence():
    cfg = gen.CONFIGS["flow1"]
    bt = gen.generate(cfg, 0, 4)
    for b in range(4):
        I = oracle.instance_from_batch(bt, b)
        d1 = oracle.Rounds(I, seed=1, inst_id=b).run(200, digests=True)["digests"]
        d2 = oracle.Rounds(I, seed=1, inst_id=b).run(200, digests=True)["digests"]
        assert np.array_equal(d1, d2)  # SPEC.md:332 / :743
    I = oracle.instance_from_batch(bt, 0)
    runs = {tuple(oracle.Rounds(I, seed=s).run(300, digests=True)["digests"][-1:]) for s in range(6)}
    assert len(runs) > 1  # the annealing draws matter


def test_quality_bounds_flow_tests():
    """F_dec <= F*, cost_dec >= cost_SSP(F_dec); cost_dec <= 1.5 cost* on >= 80% of seeds."""
    for name in ("flow1", "flow2", "flow3", "flow4"):
        cfg = gen.CONFIGS[name]
        bt = gen.generate(cfg, 0, 10)
        good = 0
        for b in range(10):
            I = oracle.instance_from_batch(bt, b)
            s = oracle.ssp(I, curve=True)
            r = oracle.Rounds(I, seed=9, inst_id=b).run(cfg.max_rounds)
            assert r["F_dec"] <= s.F
            assert r["cost_dec"] >= s.curve[r["F_dec"]]
            good += r["F_dec"] == s.F and r["cost_dec"] <= 1.5 * s.cost
        assert good >= 8, name


# ------------------------------------------------------------------ churn
def test_churn_masks_and_repair():
    cfg = gen.CONFIGS["gpt"]
    bt = gen.generate(cfg, 0, 6)
    src, snk, link = oracle.eq1_batch(bt)
    alive_new, _ = gen.generate_churn(cfg, 0, bt.alive)
    for b in range(6):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        R = oracle.Rounds(I, seed=2, inst_id=b)
        R.run(cfg.max_rounds)
        R.apply_churn(alive_new[b])
        st = R.export()
        Im = R.instance()
        check_invariants(Im, st)
        assert not st["kacc"].any() and not st["deny"].any() and st["quiet"] == 0
        # no pointer survives into a crashed relay
        dead = np.argwhere(alive_new[b] == 0)
        for s, i in dead:
            assert (st["up"][s, i] == NONE).all() and (st["down"][s, i] == NONE).all()
        # post-churn exact solve = the closed form on the masked graph (complete Eq. 1 links)
        Fm = oracle.ssp(Im).F
        assert Fm == min(I.M, int(Im.cap_eff().sum(axis=1).min()))
        r = R.run(cfg.max_rounds)
        check_invariants(Im, R.export())
        assert r["F_dec"] <= Fm


def test_churn_link_drop_and_victim():
    cfg = gen.CONFIGS["churn"].with_(S=4, n=8, M=40)
    bt = gen.generate(cfg, 0, 3)
    alive_new, ld = gen.generate_churn(cfg.with_(linkdrop_p=0.2), 0, bt.alive)
    upd = gen.linkdrop_to_updates(ld)
    for b in range(3):
        I = oracle.instance_from_batch(bt, b)
        R = oracle.Rounds(I, seed=4, inst_id=b)
        R.run(300)
        u = upd[upd[:, 0] == b]
        R.apply_churn(alive_new[b], u)
        Im = R.instance()
        for (_, s, v, w, c) in u:
            assert Im.link[s, v, w] == ABSENT
        check_invariants(Im, R.export())
        R.run(300)
        check_invariants(Im, R.export())
    # victim rule: a relay of the drawn stage that holds a PAIRED slot
    I = oracle.instance_from_batch(bt, 0)
    R = oracle.Rounds(I, seed=4)
    R.run(300)
    v = R.llama_victim(12345 << 32, 777 << 32)
    st = R.export()
    s, i = divmod(v, I.n)
    paired = (st["up"][s, i] != NONE) & (st["down"][s, i] != NONE)
    assert paired.any()
