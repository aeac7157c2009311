"""Multi-data-node rounds (gwtf_mc_rounds) on the GPU through the
C-ABI against the oracle's McRounds: the hand-derived two-data-node trace, round-by-round digests,
per-data-node (F_dec, cost_dec) and the final state on flow-test settings 5 and 6,
and K = 1 against the single-commodity oracle."""
import numpy as np
import pytest
import torch

import gen
import oracle
from tests.test_oracle_mc_rounds import two_node_instance

pytestmark = pytest.mark.gpu


def _mc(cap, alive, link, srcs, snks, sups, MC, **kw):
    from paper_2509_21221_b200.multisource import mc_rounds
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return mc_rounds(t(cap), t(alive), t(link), [t(s) for s in srcs], [t(s) for s in snks], [t(m) for m in sups],
                     max_cap=MC, **kw)


def test_gpu_mc_hand_trace():
    I, srcs, snks, M = two_node_instance()
    B = 3
    rep = lambda a: np.broadcast_to(np.asarray(a), (B,) + np.asarray(a).shape).copy()  # noqa: E731
    out = _mc(rep(I.cap), rep(I.alive), rep(I.link), [rep(np.asarray(s, np.int32)) for s in srcs],
              [rep(np.asarray(s, np.int32)) for s in snks], [np.full(B, m, np.int64) for m in M], 1,
              max_rounds=100, T0=0.0, seed=5, state=True)
    torch.cuda.synchronize()
    for b in range(B):
        assert int(out["rounds"][b]) == 8
        assert out["F_dec"][:, b].tolist() == [1, 1] and out["cost_dec"][:, b].tolist() == [52, 52]
        assert out["down"][b].reshape(-1).tolist() == [3, 2, -2, -3] and out["tag"][b].reshape(-1).tolist() == [1, 0, 0, 1]


@pytest.mark.parametrize("name,B", [("flow5", 48), ("flow6", 48)])
def test_gpu_mc_rounds_parity(name, B):
    cfg = gen.CONFIGS[name]
    K = cfg.extra["data_nodes"]
    bt = gen.generate(cfg, 0, B)
    xs, xk = gen.generate_data_nodes(cfg, 0, B, K)
    srcs = [bt.src] + [xs[k] for k in range(K - 1)]
    snks = [bt.snk] + [xk[k] for k in range(K - 1)]
    Ms = [cfg.M // K] * K
    sups = [np.full(B, m, np.int64) for m in Ms]
    mr = cfg.max_rounds
    out = _mc(bt.cap, bt.alive, bt.link, srcs, snks, sups, cfg.max_cap, max_rounds=mr, seed=11, inst_base=0,
              digests=True, state=True)
    torch.cuda.synchronize()
    for b in range(B):
        I = oracle.instance_from_batch(bt, b)
        R = oracle.McRounds(I, [s[b] for s in srcs], [s[b] for s in snks], Ms, seed=11, inst_id=b)
        o = R.run(mr, digests=True)
        n_r = int(out["rounds"][b])
        assert n_r == o["rounds"], (name, b)
        got = out["digests"][b, :n_r].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, o["digests"]), (name, b, int(np.argmax(got != o["digests"])))
        assert out["F_dec"][:, b].tolist() == o["F_dec"].tolist() and out["cost_dec"][:, b].tolist() == o["cost_dec"].tolist()
        assert int(out["dangling"][b]) == o["dangling"]
        st = R.export()
        for key in ("up", "down", "tag"):
            assert np.array_equal(out[key][b].cpu().numpy(), st[key]), (name, b, key)


@pytest.mark.parametrize("name", ["flow1", "gpt"])
def test_gpu_mc_single_data_node(name):
    """K = 1 is the single-commodity protocol: the same (rounds, F_dec, cost_dec) as the pinned oracle."""
    cfg = gen.CONFIGS[name]
    B = 16
    bt = gen.generate(cfg, 0, B)
    src, snk, link = oracle.eq1_batch(bt) if cfg.cost_kind == gen.COST_EQ1 else (bt.src, bt.snk, bt.link)
    out = _mc(bt.cap, bt.alive, link, [src], [snk], [bt.supply], cfg.max_cap, max_rounds=cfg.max_rounds, seed=2)
    torch.cuda.synchronize()
    for b in range(B):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        o = oracle.Rounds(I, seed=2, inst_id=b).run(cfg.max_rounds)
        assert (int(out["rounds"][b]), int(out["F_dec"][0, b]), int(out["cost_dec"][0, b])) == (
            o["rounds"], o["F_dec"], o["cost_dec"]), (name, b)


def test_gpu_mc_in_slot_trace():
    """The IN-slot rule on the GPU from the same imported state (tests/test_oracle_mc_rounds.in_slot_case):
    b0's unpaired inflow of D0 goes to D0's sink; (F, cost) = ([1, 1], [12, 3]) after 8 rounds."""
    from tests.test_oracle_mc_rounds import in_slot_case
    I, srcs, snks, M, st0 = in_slot_case()
    B = 2
    rep = lambda a: np.broadcast_to(np.asarray(a), (B,) + np.asarray(a).shape).copy()  # noqa: E731
    start = {k: torch.from_numpy(rep(np.asarray(st0[k], np.int32))).cuda() for k in ("up", "down", "tag", "src_down", "snk_up")}
    out = _mc(rep(I.cap), rep(I.alive), rep(I.link), [rep(np.asarray(s, np.int32)) for s in srcs],
              [rep(np.asarray(s, np.int32)) for s in snks], [np.full(B, m, np.int64) for m in M], 1,
              max_rounds=100, T0=0.0, seed=4, start_state=start, round0=20, state=True)
    torch.cuda.synchronize()
    for b in range(B):
        assert int(out["rounds"][b]) == 8
        assert out["F_dec"][:, b].tolist() == [1, 1] and out["cost_dec"][:, b].tolist() == [12, 3]
        assert out["down"][b].reshape(-1).tolist() == [2, 3, -2, -3] and out["tag"][b].reshape(-1).tolist() == [0, 1, 0, 1]
