"""The hand-derived pin cases (tests/pin_cases.py) on the GPU, through the C-ABI: the canonical
SSP ties (F, cost, A, full assignment), and the crafted-state DENY / self-pairing / annealing
traces installed with gwtf_flow_import_round_state, on the team tier and the cluster tier of
the rounds.  Expected values are the hand-derived literals, the same ones the oracle is pinned
to (tests/test_oracle_pins.py)."""
import numpy as np
import pytest
import torch

from tests import pin_cases as pc

pytestmark = pytest.mark.gpu

REPS = 3  # identical copies of the instance in one batch (inst ids 0..2; the traces are RNG-free)


def _flow(d, B=1, **kw):
    from paper_2509_21221_b200 import Flow
    t = lambda a: torch.from_numpy(np.ascontiguousarray(np.broadcast_to(a, (B,) + a.shape))).cuda()  # noqa: E731
    return Flow(t(d["cap"]), t(d["src"]), t(d["snk"]), t(d["link"]), torch.full((B,), d["M"], dtype=torch.int64,
                device="cuda"), max_cap=d["max_cap"], alive=t(d["alive"]), **kw)


@pytest.mark.parametrize("name", sorted(pc.SSP_CASES))
@pytest.mark.parametrize("tier", ["auto", "global", "cluster"])
def test_gpu_ssp_canonical_ties(name, tier):
    d, exp = pc.SSP_CASES[name]()
    if tier == "cluster" and d["n"] < 2:
        pytest.skip("the cluster tier needs n >= C >= 2")
    fl = _flow(d, B=4, force_global_tier=tier == "global", force_cluster_tier=tier == "cluster")
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    for b in range(4):
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (exp["F"], exp["cost"], exp["A"])
        assert np.array_equal(nf[b], np.asarray(exp["node_flow"])) and np.array_equal(af[b], pc.arc_dense(d, exp["arc"]))
        assert np.array_equal(sf[b], np.asarray(exp["src_flow"])) and np.array_equal(kf[b], np.asarray(exp["snk_flow"]))
    assert (sol.status == 0).all()


def _import(fl, st0, B):
    st = {}
    for k, v in st0.items():
        if k in ("quiet", "round"):
            st[k] = torch.full((B,), int(v), dtype=torch.int64 if k == "round" else torch.int32, device="cuda")
        else:
            a = np.asarray(v, np.int32)
            st[k] = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(a, (B,) + a.shape))).cuda()
    fl.import_round_state(st)


def _check(got, b, d, slots, src_down, snk_up, deny):
    exp = pc.state(d["S"], d["n"], d["max_cap"], d["M"], slots, src_down, snk_up, deny=deny)
    for k in ("up", "down", "src_down", "snk_up", "deny"):
        assert np.array_equal(got[k][b].cpu().numpy().ravel(), exp[k].ravel()), k


@pytest.mark.parametrize("case", ["deny", "selfpair"])
@pytest.mark.parametrize("tier", ["team", "cluster"])
def test_gpu_crafted_traces(case, tier, monkeypatch):
    if tier == "cluster":
        monkeypatch.setenv("GWTF_ROUNDS_GLOBAL", "1")
        monkeypatch.setenv("GWTF_ROUNDS_CLUSTER", "1")
        monkeypatch.setenv("GWTF_ROUNDS_CLUSTER_SIZE", "2")
    d, st0, after, final, kw = (pc.deny_case if case == "deny" else pc.selfpair_case)()
    kw = dict(kw)
    kw["inst_base"] = kw.pop("inst_id")
    fl = _flow(d, B=REPS, **kw)
    _import(fl, st0, REPS)
    for rnd in sorted(after):
        fl.decentralized_rounds(1)
        got = fl.export_round_state()
        for b in range(REPS):
            assert int(got["round"][b]) == rnd + 1
            _check(got, b, d, *after[rnd])
    fl2 = _flow(d, B=REPS, **kw)
    _import(fl2, st0, REPS)
    rr = fl2.decentralized_rounds(100)
    got = fl2.export_round_state()
    for b in range(REPS):
        assert (int(rr.rounds_run[b]), int(rr.dec_flow[b]), int(rr.dec_cost[b]), int(rr.dangling[b])) == (
            final["rounds"], final["F_dec"], final["cost_dec"], final["dangling"])
        assert int(got["round"][b]) == final["round"]


@pytest.mark.parametrize("seed", sorted(pc.ANNEAL_DRAWS))
def test_gpu_anneal_draw_decides(seed):
    d, st0, (slots, kacc, cost), kw = pc.anneal_case(seed)
    kw = dict(kw)
    kw["inst_base"] = kw.pop("inst_id")
    fl = _flow(d, B=1, **kw)
    _import(fl, st0, 1)
    rr = fl.decentralized_rounds(1)
    got = fl.export_round_state()
    _check(got, 0, d, slots, [0, 1], [2, 3], [0] * 4)  # a Change only moves down / up pointers
    assert list(got["kacc"][0].cpu().numpy().ravel()) == kacc
    assert (int(rr.dec_flow[0]), int(rr.dec_cost[0])) == (2, cost)


def test_gpu_import_rejects_invalid_state():
    from paper_2509_21221_b200._lib import GwtfError
    d, st0, _, _, kw = pc.deny_case()
    fl = _flow(d, B=2)
    bad = {k: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v) for k, v in st0.items()}
    bad["down"].reshape(-1)[2] = 5
    with pytest.raises(GwtfError):
        _import(fl, bad, 2)
    got = fl.export_round_state()
    assert (got["up"] == -1).all() and (got["down"] == -1).all()  # reset to empty, not half-imported
    _import(fl, st0, 2)
