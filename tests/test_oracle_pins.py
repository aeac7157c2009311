"""Pins of the oracle's remaining definitional parts (VERDICT r1 "What's weak" #1), CPU only:

* the counter RNG of R4: mix64 against the published SplitMix64 sequence, the
  composition of h() and pick() against hand-computed known answers;
* an annealing accept / reject that the draw decides;
* DENY and R0a self-pairing as hand-derived round traces from
  crafted states (tests/pin_cases.py), installed with the oracle's state import;
* the canonical SSP tie-break and augmentation count on hand-worked ties.

Each expected value is derived in tests/pin_cases.py's docstrings, not obtained by running the
oracle; each test fails under the plausible mutation named in its docstring."""
import numpy as np
import pytest

import oracle
from oracle import Instance
from tests import pin_cases as pc


def to_instance(d):
    return Instance(d["S"], d["n"], d["max_cap"], d["M"], d["cap"], d["src"], d["snk"], d["link"], d["alive"])


# ------------------------------------------------------------------ RNG known answers
GAMMA = 0x9E3779B97F4A7C15
# SplitMix64 (Steele, Lea, Flood 2014; Vigna's reference splitmix64.c) seeded with 0 returns
# mix64(k * GAMMA) for k = 1, 2, 3, 4: the published first outputs of the generator.
SPLITMIX64_SEED0 = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]


def test_mix64_published_sequence():
    """The finalizer's constants and shifts (30/27/31, 0xbf58476d1ce4e5b9, 0x94d049bb133111eb)."""
    assert [oracle.mix64(k * GAMMA & (2**64 - 1)) for k in range(1, 5)] == SPLITMIX64_SEED0
    assert oracle.mix64(0) == 0


def _s64(x):
    return x - 2**64 if x >= 2**63 else x


def test_h_composition_known_answers():
    """h = mix(mix(mix(mix(seed) ^ inst) ^ round) ^ (gid*4 + stream)).  With seed = GAMMA,
    inst = out1 ^ 2*GAMMA and round = out2 ^ 3*GAMMA the first three levels walk the published
    sequence (mix(seed) = out1, mix(out1 ^ inst) = out2, mix(out2 ^ round) = out3), so only the
    last level is hand-computed: mix(out3 ^ (4 gid + stream)).  A swapped XOR order (inst and
    round exchanged), a missing level or gid*2 instead of gid*4 all change these values."""
    inst = _s64(SPLITMIX64_SEED0[0] ^ (2 * GAMMA & (2**64 - 1)))
    rnd = _s64(SPLITMIX64_SEED0[1] ^ (3 * GAMMA & (2**64 - 1)))
    assert (inst, rnd) == (-2427902769185081979, -5413622216381820469)
    kat = {(0, 0): 0x7B476C5A5333D0EC, (0, 3): 0x1C2C45AC2DA7E65D, (5, 1): 0x00D743FA52DFA1BB,
           (1000, 2): 0x83BC866BABA2FBE9}
    for (gid, stream), val in kat.items():
        assert oracle.rng_h(GAMMA, inst, rnd, gid, stream) == val
    # the annealing trace's draws (tests/pin_cases.ANNEAL_DRAWS)
    for seed, (h0, h1, _) in pc.ANNEAL_DRAWS.items():
        assert oracle.rng_h(seed, 0, 100, 0, 3) == h0 and oracle.rng_h(seed, 0, 100, 1, 3) == h1


def test_pick_known_answers():
    """pick(x, m) = floor((x >> 32) * m / 2^32) (Lemire's multiply-shift): the high word scaled."""
    assert oracle.pick(0, 7) == 0
    assert oracle.pick(2**63, 10) == 5
    assert oracle.pick(2**64 - 1, 10) == 9
    assert oracle.pick((3 << 32) | 0xFFFFFFFF, 2**31) == 1        # the low word is ignored
    assert oracle.pick(0xC000000000000000, 3) == 2                # 0.75 * 3 = 2.25
    assert oracle.pick(0x5555555600000000, 3) == 1                # just above 1/3


# ------------------------------------------------------------------ annealing decided by the draw
@pytest.mark.parametrize("seed", sorted(pc.ANNEAL_DRAWS))
def test_anneal_draw_decides(seed):
    """PAPER.md:259 with T = 1.7: an uphill Change (delta = +1) commits iff the proposer's
    draw is below thr[0][1].  seed 6: n1 accepts; seed 19: n1's draw is 0.8% above the threshold
    (rejects), n3 accepts; seed 2: both reject.  Fails if the threshold or the draw stream moves."""
    I, st0, (slots, kacc, cost), kw = pc.anneal_case(seed)
    assert (pc.ANNEAL_DRAWS[seed][0] >> 32 < pc.THR_0_1) == (pc.ANNEAL_DRAWS[seed][2] == "gid0")
    R = oracle.Rounds(to_instance(I), **kw)
    R.import_state(st0)
    r = R.run(1)
    st = R.export()
    up = np.full(4, -1, np.int32)
    dn = np.full(4, -1, np.int32)
    for p, (u, d) in slots.items():
        up[p], dn[p] = u, d
    assert np.array_equal(st["up"].ravel(), up) and np.array_equal(st["down"].ravel(), dn)
    assert list(st["kacc"].ravel()) == kacc and r["cost_dec"] == cost and r["F_dec"] == 2


# ------------------------------------------------------------------ crafted-state traces
def _check_state(st, I, slots, src_down, snk_up, deny):
    exp = pc.state(I["S"], I["n"], I["max_cap"], I["M"], slots, src_down, snk_up, deny=deny)
    for k in ("up", "down", "src_down", "snk_up", "deny"):
        assert np.array_equal(np.asarray(st[k]).ravel(), exp[k].ravel()), k


def _trace(case):
    I, st0, after, final, kw = case()
    R = oracle.Rounds(to_instance(I), **kw)
    R.import_state(st0)
    for rnd in sorted(after):
        assert R.export()["round"] == rnd
        R.run(1)
        _check_state(R.export(), I, *after[rnd])
    # the whole trajectory in one call from the start state
    R2 = oracle.Rounds(to_instance(I), **kw)
    R2.import_state(st0)
    r = R2.run(100)
    assert (r["rounds"], r["F_dec"], r["cost_dec"], r["dangling"]) == (final["rounds"], final["F_dec"],
                                                                     final["cost_dec"], final["dangling"])
    assert R2.export()["round"] == final["round"]


def test_deny_trace():
    """PAPER.md:269 DENY, hand-derived (tests/pin_cases.deny_case): a rejected requester does not
    count an idle round; DENY fires on the deny_after-th idle round; the upstream PAIRED slot
    becomes IN (not FREE); the DENY recurses to the source, whose SRC slot becomes unpaired."""
    _trace(pc.deny_case)


def test_selfpair_trace():
    """PAPER.md:253 R0a self-pairing, hand-derived (tests/pin_cases.selfpair_case): the LOWEST IN
    slot takes the downstream of the MIN-COST OUT slot, which becomes FREE; one per round."""
    _trace(pc.selfpair_case)


def test_import_rejects_invalid_states():
    I, st0, _, _, kw = pc.deny_case()
    R = oracle.Rounds(to_instance(I), **kw)
    bad = {k: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v) for k, v in st0.items()}
    bad["down"].reshape(-1)[2] = 5  # b0 -> dead c1's slot, not answered
    with pytest.raises(ValueError):
        R.import_state(bad)
    bad = {k: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v) for k, v in st0.items()}
    bad["src_down"][1] = 0  # two SRC slots claim a0's slot
    with pytest.raises(ValueError):
        R.import_state(bad)
    R.import_state(st0)  # the valid state still imports


# ------------------------------------------------------------------ canonical SSP ties
@pytest.mark.parametrize("name", sorted(pc.SSP_CASES))
def test_ssp_canonical_ties(name):
    """SURVEY C2 / C6 #6 on hand-worked ties (tests/pin_cases.py): lowest-(layer, position)
    predecessors ("position"), the hop count breaking a cost tie ("hops": cost-only keys pick
    the other assignment), a canonical path through a reverse arc ("cancel") and delta > 1
    ("bottleneck": A < F).  Expected F, cost, A and the full assignment."""
    d, exp = pc.SSP_CASES[name]()
    s = oracle.ssp(to_instance(d))
    assert (s.F, s.cost, s.A) == (exp["F"], exp["cost"], exp["A"])
    assert np.array_equal(s.node_flow, np.asarray(exp["node_flow"]))
    assert np.array_equal(s.src_flow, np.asarray(exp["src_flow"]))
    assert np.array_equal(s.snk_flow, np.asarray(exp["snk_flow"]))
    assert np.array_equal(s.arc_flow, pc.arc_dense(d, exp["arc"]))
