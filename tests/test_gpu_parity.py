"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle on the same seeded inputs.

Bar: everything here is integer, so bit-exact -- flow value, cost, augmentation
count, the canonical assignment (node flows, source/sink flows, dense arc flows), every
per-round state digest of the decentralized rounds and the final exported round state."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import gen
import oracle
from tests import harness

pytestmark = pytest.mark.gpu

SSP_CASES = [("tiny", 512), ("gpt", 256), ("llama", 24), ("churn", 6), ("flow1", 64), ("flow2", 64),
             ("flow3", 64), ("flow4", 64)]


def _oracle_ssp(cfg, bt, src, snk, link, b):
    I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
    return oracle.ssp(I)


def _gpu_flow(cfg, inst0, B, **kw):
    from paper_2509_21221_b200 import Flow
    dbt, src, snk, link = harness.device_inputs(cfg, inst0, B)
    return Flow(dbt.cap, src, snk, link, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive, **kw), dbt, src, snk, link


def test_eq1_tiles_parity():
    for name in ("gpt", "llama"):
        cfg = gen.CONFIGS[name]
        bt, src, snk, link = harness.host_inputs(cfg, 100, 16)
        _, dsrc, dsnk, dlink = harness.device_inputs(cfg, 100, 16)
        assert np.array_equal(dsrc.cpu().numpy(), src)
        assert np.array_equal(dsnk.cpu().numpy(), snk)
        assert np.array_equal(dlink.cpu().numpy(), link)


def test_generator_device_twin():
    for name in ("tiny", "gpt", "churn"):
        cfg = gen.CONFIGS[name]
        h = gen.generate(cfg, 7, 9)
        d = gen.generate(cfg, 7, 9, device="cuda")
        for f in ("cap", "alive", "supply", "src", "snk", "link", "comp", "loc", "dloc", "lat", "bw"):
            a = getattr(h, f)
            if a is not None:
                assert np.array_equal(a, getattr(d, f).cpu().numpy()), (name, f)


@pytest.mark.parametrize("name,B", SSP_CASES)
def test_ssp_parity(name, B):
    cfg = gen.CONFIGS[name]
    fl, *_ = _gpu_flow(cfg, 0, B)
    sol = fl.solve_batch()
    nf, sf, kf, af = fl.get_assignment()
    torch.cuda.synchronize()
    assert (sol.status.cpu().numpy() == 0).all()
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    F, C, A = sol.flow_value.cpu().numpy(), sol.total_cost.cpu().numpy(), sol.augmentations.cpu().numpy()
    nf, sf, kf, af = nf.cpu().numpy(), sf.cpu().numpy(), kf.cpu().numpy(), af.cpu().numpy()
    for b in range(B):
        r = _oracle_ssp(cfg, bt, src, snk, link, b)
        assert (F[b], C[b], A[b]) == (r.F, r.cost, r.A), (name, b)
        assert np.array_equal(nf[b], r.node_flow), (name, b)
        assert np.array_equal(sf[b], r.src_flow) and np.array_equal(kf[b], r.snk_flow), (name, b)
        assert np.array_equal(af[b], r.arc_flow), (name, b)


def test_ssp_parity_dead_and_absent():
    """Dead relays, absent links (incl. absent source/sink arcs) and per-instance supply."""
    cfg = gen.CONFIGS["flow1"].with_(alive_p=0.75, absent_p=0.3, cost=(0, 9))
    B = 128
    bt = gen.generate(cfg, 0, B)
    rng = np.random.default_rng(0)
    bt.supply[:] = rng.integers(0, 40, B)
    bt.src[rng.random(bt.src.shape) < 0.2] = gen.ABSENT
    bt.snk[rng.random(bt.snk.shape) < 0.2] = gen.ABSENT
    from paper_2509_21221_b200 import Flow
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    fl = Flow(t(bt.cap), t(bt.src), t(bt.snk), t(bt.link), t(bt.supply), max_cap=cfg.max_cap, alive=t(bt.alive))
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    for b in range(B):
        I = oracle.instance_from_batch(bt, b)
        r = oracle.ssp(I)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), b
        assert np.array_equal(af[b], r.arc_flow) and np.array_equal(nf[b], r.node_flow), b


def test_ssp_global_tier_identical():
    """The same instances through the shared-memory tier and the global-memory tier."""
    cfg = gen.CONFIGS["gpt"]
    a, *_ = _gpu_flow(cfg, 0, 64)
    b, *_ = _gpu_flow(cfg, 0, 64, force_global_tier=True)
    ra, rb = a.solve_batch(), b.solve_batch()
    for x, y in zip(a.get_assignment(), b.get_assignment()):
        assert torch.equal(x, y)
    assert torch.equal(ra.total_cost, rb.total_cost) and torch.equal(ra.augmentations, rb.augmentations)


@pytest.mark.parametrize("name,B", [("tiny", 256), ("flow1", 48), ("flow3", 32), ("flow4", 48), ("gpt", 64)])
def test_rounds_digest_parity(name, B):
    """Round-by-round: the GPU state digest after every round equals the oracle's."""
    cfg = gen.CONFIGS[name]
    fl, *_ = _gpu_flow(cfg, 0, B, seed=17)
    rr = fl.decentralized_rounds(cfg.max_rounds, digests=True)
    st = fl.export_round_state()
    torch.cuda.synchronize()
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    for b in range(B):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        R = oracle.Rounds(I, seed=17, inst_id=b)
        o = R.run(cfg.max_rounds, digests=True)
        n_r = int(rr.rounds_run[b])
        assert n_r == o["rounds"], (name, b)
        got = rr.digests[b, :n_r].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, o["digests"]), (name, b, int(np.argmax(got != o["digests"])))
        assert (int(rr.dec_flow[b]), int(rr.dec_cost[b]), int(rr.dangling[b])) == (o["F_dec"], o["cost_dec"], o["dangling"])
        ost = R.export()
        M = I.M
        assert np.array_equal(st["up"][b].cpu().numpy(), ost["up"]) and np.array_equal(st["down"][b].cpu().numpy(), ost["down"])
        assert np.array_equal(st["src_down"][b, :M].cpu().numpy(), ost["src_down"])
        assert int(st["round"][b]) == ost["round"]


@pytest.mark.parametrize("name,B,C", [("churn", 4, None), ("llama", 3, 4), ("flow3", 8, 2), ("gpt", 6, 16),
                                      ("stress_s", 2, None)])
def test_rounds_cluster_tier_parity(name, B, C, monkeypatch):
    """The rounds on thread-block-cluster teams (C CTAs x 1,024 threads per instance, cluster
    barriers, DSMEM votes): round-by-round digests and final state equal the oracle's."""
    monkeypatch.setenv("GWTF_ROUNDS_GLOBAL", "1")
    monkeypatch.setenv("GWTF_ROUNDS_CLUSTER", "1")
    if C is not None:
        monkeypatch.setenv("GWTF_ROUNDS_CLUSTER_SIZE", str(C))
    cfg = gen.CONFIGS[name]
    fl, *_ = _gpu_flow(cfg, 0, B, seed=17)
    rr = fl.decentralized_rounds(cfg.max_rounds, digests=True)
    st = fl.export_round_state()
    torch.cuda.synchronize()
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    for b in range(B):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        R = oracle.Rounds(I, seed=17, inst_id=b)
        o = R.run(cfg.max_rounds, digests=True)
        n_r = int(rr.rounds_run[b])
        assert n_r == o["rounds"], (name, b)
        got = rr.digests[b, :n_r].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, o["digests"]), (name, b, int(np.argmax(got != o["digests"])))
        assert (int(rr.dec_flow[b]), int(rr.dec_cost[b]), int(rr.dangling[b])) == (o["F_dec"], o["cost_dec"], o["dangling"])
        ost = R.export()
        assert np.array_equal(st["up"][b].cpu().numpy(), ost["up"]) and np.array_equal(st["down"][b].cpu().numpy(), ost["down"])


@pytest.mark.parametrize("objective", [0, 1])
def test_rounds_parity_minimax_and_annealing_off(objective):
    cfg = gen.CONFIGS["flow2"]
    B = 48
    for T0 in (0.0, 25.0):
        fl, *_ = _gpu_flow(cfg, 0, B, seed=5, objective=objective, T0=T0)
        rr = fl.decentralized_rounds(300, digests=True)
        bt, src, snk, link = harness.host_inputs(cfg, 0, B)
        for b in range(B):
            I = oracle.instance_from_batch(bt, b)
            o = oracle.Rounds(I, seed=5, inst_id=b, T0=T0, objective=objective).run(300, digests=True)
            got = rr.digests[b, : o["rounds"]].cpu().numpy().view(np.uint64)
            assert int(rr.rounds_run[b]) == o["rounds"] and np.array_equal(got, o["digests"]), (T0, b)


@pytest.mark.parametrize("name,B", [("gpt", 96), ("llama", 12), ("churn", 4)])
def test_churn_pipeline_parity(name, B):
    """Base rounds to quiescence -> churn -> cold exact solve -> repair rounds."""
    cfg = gen.CONFIGS[name]
    _, pre, sol, rr = harness.gpu_pipeline(cfg, 0, B, seed=3)
    o = harness.oracle_pipeline(cfg, 0, B, seed=3)
    assert np.array_equal(pre.rounds_run.cpu().numpy(), o["pre_rounds"])
    assert np.array_equal(sol.flow_value.cpu().numpy(), o["F"])
    assert np.array_equal(sol.total_cost.cpu().numpy(), o["cost"])
    assert np.array_equal(sol.augmentations.cpu().numpy(), o["A"])
    assert np.array_equal(rr.rounds_run.cpu().numpy(), o["rounds"])
    assert np.array_equal(rr.dec_flow.cpu().numpy(), o["F_dec"])
    assert np.array_equal(rr.dec_cost.cpu().numpy(), o["cost_dec"])
    last = np.array([int(rr.digests[b, int(rr.rounds_run[b]) - 1]) & ((1 << 64) - 1) for b in range(B)], np.uint64)
    assert np.array_equal(last, o["digest"])


def test_hand_traces_on_gpu():
    from tests.test_oracle_rounds import change_instance, redirect_instance
    from paper_2509_21221_b200 import Flow
    for inst, obj, want in ((change_instance(), 1, (2, 12)), (change_instance(), 0, (2, 11)),
                            (redirect_instance(), 0, (1, 9))):
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)[None]).cuda()  # noqa: E731
        fl = Flow(t(inst.cap), t(inst.src), t(inst.snk), t(inst.link), torch.tensor([inst.M], device="cuda"),
                  max_cap=inst.max_cap, alive=t(inst.alive), T0=0.0, objective=obj, seed=99)
        rr = fl.decentralized_rounds(100)
        assert (int(rr.dec_flow[0]), int(rr.dec_cost[0]), int(rr.rounds_run[0])) == (*want, 9)


def test_edge_cases():
    from paper_2509_21221_b200 import Flow
    cases = [  # (S, n, caps, M)
        (1, 1, [[1]], 3), (1, 2, [[0, 0]], 2), (2, 3, [[1, 2, 3], [0, 0, 0]], 5), (3, 1, [[2], [2], [2]], 0),
        (2, 5, [[3] * 5, [3] * 5], 40),
    ]
    for S, n, caps, M in cases:
        rng = np.random.default_rng(S * 10 + n)
        cap = np.array(caps, np.int32)[None]
        src = rng.integers(0, 9, (1, n)).astype(np.int32)
        snk = rng.integers(0, 9, (1, n)).astype(np.int32)
        link = rng.integers(0, 9, (1, max(S - 1, 0), n, n)).astype(np.int32)
        t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        fl = Flow(t(cap), t(src), t(snk), t(link), torch.tensor([M], device="cuda"), max_cap=3)
        sol = fl.solve_batch()
        I = oracle.Instance(S, n, 3, M, cap[0], src[0], snk[0], link[0])
        r = oracle.ssp(I)
        assert (int(sol.flow_value[0]), int(sol.total_cost[0])) == (r.F, r.cost), (S, n)
        rr = fl.decentralized_rounds(50, digests=True)
        o = oracle.Rounds(I).run(50, digests=True)
        assert int(rr.rounds_run[0]) == o["rounds"]
        assert np.array_equal(rr.digests[0, : o["rounds"]].cpu().numpy().view(np.uint64), o["digests"])


def test_host_pointer_mode_matches():
    cfg = gen.CONFIGS["gpt"]
    B = 32
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    from paper_2509_21221_b200 import Flow
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    fh = Flow(pin(bt.cap), pin(src), pin(snk), pin(link), pin(bt.supply), max_cap=cfg.max_cap, alive=pin(bt.alive),
              host=True, seed=1)
    sh = fh.solve_batch()
    rh = fh.decentralized_rounds(cfg.max_rounds)
    fd, *_ = _gpu_flow(cfg, 0, B, seed=1)
    sd = fd.solve_batch()
    rd = fd.decentralized_rounds(cfg.max_rounds)
    torch.cuda.synchronize()
    assert torch.equal(sh.total_cost, sd.total_cost.cpu()) and torch.equal(rh.dec_cost, rd.dec_cost.cpu())


def test_validation_errors():
    from paper_2509_21221_b200 import Flow, GwtfError
    t = lambda a: torch.tensor(a, device="cuda")  # noqa: E731
    cap = t([[[1, 1]]]).int()
    ok = dict(src_cost=t([[1, 1]]).int(), snk_cost=t([[1, 1]]).int(), link_cost=None, supply=t([2]).long())
    with pytest.raises(GwtfError, match="E_INVALID"):
        Flow(cap, **{**ok, "src_cost": t([[-1, 1]]).int()}, max_cap=3)
    with pytest.raises(GwtfError, match="E_INVALID"):
        Flow(cap, **ok, max_cap=33)
    with pytest.raises(GwtfError, match="E_INVALID"):
        Flow(t([[[5, 1]]]).int(), **ok, max_cap=3)
    with pytest.raises(GwtfError, match="E_INVALID"):
        Flow(cap, **{**ok, "supply": t([-1]).long()}, max_cap=3)
    with pytest.raises(GwtfError, match="E_OVERFLOW"):  # (2Sn+2) * maxcost >= 2^42
        n = 2048
        Flow(torch.ones((1, 1, n), dtype=torch.int32, device="cuda"),
             src_cost=torch.full((1, n), 2**30 - 1, dtype=torch.int32, device="cuda"),
             snk_cost=torch.ones((1, n), dtype=torch.int32, device="cuda"), link_cost=None, supply=t([1]).long(),
             max_cap=3)
    fl = Flow(cap, **ok, max_cap=3)
    with pytest.raises(GwtfError, match="E_STATE"):
        fl.get_assignment()
    with pytest.raises(GwtfError, match="E_INVALID"):
        fl.apply_churn(None, t([[5, 0, 0, 0, 1]]).int())


@pytest.mark.parametrize("name,samples", [("gpt", 48), ("llama", 8), ("churn", 6)])
def test_full_size_bench_config_sampled(name, samples):
    """GPT (the bench line), LLaMA and churn (the bench's other_configs) at their full batch sizes and
    launch configurations; sampled instances of the whole churn pipeline vs the oracle."""
    cfg = gen.CONFIGS[name]
    B = cfg.B
    _, pre, sol, rr = harness.gpu_pipeline(cfg, 0, B, seed=0, digests=False)
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(B, samples, replace=False))
    for b in idx:
        o = harness.oracle_pipeline(cfg, int(b), 1, seed=0)
        # instance b of the big batch == instance 0 of a batch starting at global id b
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (
            int(o["F"][0]), int(o["cost"][0]), int(o["A"][0])), b
        assert (int(rr.dec_flow[b]), int(rr.dec_cost[b]), int(rr.rounds_run[b])) == (
            int(o["F_dec"][0]), int(o["cost_dec"][0]), int(o["rounds"][0])), b
    assert (sol.status == 0).all()


@pytest.mark.parametrize("name,B,C", [("gpt", 24, None), ("gpt", 24, 16), ("gpt", 24, 8), ("llama", 6, None),
                                      ("churn", 4, None), ("churn", 4, 16), ("flow3", 16, None), ("churn", 4, "int32"),
                                      ("stress_s", 2, "int32")])
def test_cluster_tier_parity_forced(name, B, C, monkeypatch):
    """Instances forced through the thread-block-cluster tier (HBM-streamed tiles, DSMEM keys), with
    the automatic cluster size, pinned ones (R = n / C destination rows per CTA) and the int32 tile
    stream instead of the 16-bit copy ("int32")."""
    if C == "int32":
        monkeypatch.setenv("GWTF_NO_TILE16", "1")
    elif C is not None:
        monkeypatch.setenv("GWTF_CLUSTER_SIZE", str(C))
    cfg = gen.CONFIGS[name]
    fl, *_ = _gpu_flow(cfg, 0, B, force_cluster_tier=True)
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    for b in range(B):
        r = _oracle_ssp(cfg, bt, src, snk, link, b)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), (name, b)
        assert np.array_equal(nf[b], r.node_flow) and np.array_equal(af[b], r.arc_flow), (name, b)
        assert np.array_equal(sf[b], r.src_flow) and np.array_equal(kf[b], r.snk_flow), (name, b)
    assert (sol.status == 0).all()


def test_cluster_tier_full_width():
    """3 x 1,024 stress distributions: the cluster tier's 1,024-column 8-bit fast path (register keys in
    the permuted conflict-free layout, sparse 8-bit frontier steps of up to 256 columns), full assignment."""
    cfg = gen.CONFIGS["stress_w"]
    B = 2
    fl, *_ = _gpu_flow(cfg, 0, B)
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    for b in range(B):
        r = _oracle_ssp(cfg, bt, src, snk, link, b)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), b
        assert np.array_equal(af[b], r.arc_flow) and np.array_equal(nf[b], r.node_flow), b
        assert np.array_equal(sf[b], r.src_flow) and np.array_equal(kf[b], r.snk_flow), b
    assert (sol.status == 0).all()
    assert fl.stats()["path_nodes"] > 0  # the cluster tier ran (it alone counts traced path nodes)


def test_cluster_tier_stress_hops():
    """64 x 512 stress distributions: >= 17 hop bits in the 32-bit keys, register-resident keys."""
    cfg = gen.CONFIGS["stress_h"]
    B = 2
    fl, *_ = _gpu_flow(cfg, 0, B)
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    for b in range(B):
        r = _oracle_ssp(cfg, bt, src, snk, link, b)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), b
        assert np.array_equal(af[b], r.arc_flow) and np.array_equal(nf[b], r.node_flow), b
    assert (sol.status == 0).all()


def test_cluster_tier_wide_keys():
    """Arc weights too large for the cluster tier's 32-bit relaxation keys (every boundary step
    takes the 64-bit path): link costs scaled by 2^16, still exact."""
    from paper_2509_21221_b200 import Flow
    cfg = gen.CONFIGS["churn"]
    B = 4
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    big = np.where(link == gen.ABSENT, link, link.astype(np.int64) * 65536).astype(np.int32)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    fl = Flow(dev(bt.cap), dev(src), dev(snk), dev(big), dev(bt.supply), max_cap=cfg.max_cap,
              alive=dev(bt.alive), force_cluster_tier=True)
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    for b in range(B):
        r = _oracle_ssp(cfg, bt, src, snk, big, b)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), b
        assert np.array_equal(nf[b], r.node_flow) and np.array_equal(af[b], r.arc_flow), b
    assert (sol.status == 0).all()


def test_cluster_tier_stress_scaled():
    """The stress distributions at 8 x 256 (1.8 MB of tiles per instance): the cluster tier by size."""
    cfg = gen.CONFIGS["stress_s"]
    B = 4
    fl, *_ = _gpu_flow(cfg, 0, B)
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    for b in range(B):
        r = _oracle_ssp(cfg, bt, src, snk, link, b)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), b
        assert np.array_equal(af[b], r.arc_flow) and np.array_equal(nf[b], r.node_flow), b


def test_stress_full_golden():
    """Full-size stress instances (64 x 1,024, M = 4,096) through the cluster tier against the
    oracle's values stored by scripts/stress_golden.py (oracle.ssp: ~1-2 h of CPU each): F, cost,
    augmentations and SHA-256 digests of the canonical assignment."""
    path = os.path.join(os.path.dirname(__file__), "golden", "stress_ssp.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/stress_ssp.json not generated yet")
    gold = json.load(open(path))["instances"]
    cfg = gen.CONFIGS["stress"]
    sha = lambda x: hashlib.sha256(np.ascontiguousarray(x, dtype=np.int32).tobytes()).hexdigest()  # noqa: E731
    for key, g in sorted(gold.items()):
        i = int(key)
        fl, *_ = _gpu_flow(cfg, i, 1)
        sol = fl.solve_batch()
        nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
        assert (int(sol.flow_value[0]), int(sol.total_cost[0]), int(sol.augmentations[0])) == (g["F"], g["cost"], g["A"]), i
        assert sha(nf[0]) == g["node_flow_sha256"] and sha(af[0]) == g["arc_flow_sha256"], i
        assert sha(sf[0]) == g["src_flow_sha256"] and sha(kf[0]) == g["snk_flow_sha256"], i
        fl.close()


def test_stress_rounds_full_golden():
    """Decentralized rounds on full-size stress instances (cluster-team tier), cold, to
    max_rounds = 8,312 or quiescence, against the oracle trajectory stored by
    scripts/stress_rounds_golden.py: rounds run, F_dec, cost_dec, dangling, every 256th per-round
    digest and the SHA-256 of the whole digest sequence."""
    path = os.path.join(os.path.dirname(__file__), "golden", "stress_rounds.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/stress_rounds.json not generated yet")
    gold = json.load(open(path))
    cfg = gen.CONFIGS["stress"]
    for key, g in sorted(gold["instances"].items()):
        i = int(key)
        fl, *_ = _gpu_flow(cfg, i, 1, seed=gold["seed"], inst_base=i)
        rr = fl.decentralized_rounds(gold["max_rounds"], digests=True)
        torch.cuda.synchronize()
        n_r = int(rr.rounds_run[0])
        assert n_r == g["rounds"], i
        assert (int(rr.dec_flow[0]), int(rr.dec_cost[0]), int(rr.dangling[0])) == (g["F_dec"], g["cost_dec"], g["dangling"]), i
        d = np.ascontiguousarray(rr.digests[0, :n_r].cpu().numpy().view(np.uint64))
        assert [str(int(x)) for x in d[::256]] == g["digest_every_256"], i
        assert hashlib.sha256(d.tobytes()).hexdigest() == g["digests_sha256"], i
        fl.close()


@pytest.mark.parametrize("name,B", [("gpt", 256), ("churn", 16)])
def test_solve_and_rounds_matches_serial(name, B):
    """gwtf_flow_solve_and_rounds (solve and rounds on two streams) returns exactly what the two
    serial calls return, after churn, and leaves the same assignment."""
    cfg = gen.CONFIGS[name]
    outs = []
    for concurrent in (False, True):
        fl, dbt, *_ = _gpu_flow(cfg, 0, B, seed=3)
        fl.decentralized_rounds(cfg.max_rounds)
        an, upd = harness.churn_inputs(cfg, 0, dbt.alive, device="cuda")
        fl.apply_churn(an, upd)
        if concurrent:
            sol, rr = fl.solve_and_rounds(cfg.max_rounds)
        else:
            sol = fl.solve_batch()
            rr = fl.decentralized_rounds(cfg.max_rounds)
        nf, sf, kf, af = fl.get_assignment()
        st = fl.export_round_state()
        torch.cuda.synchronize()
        outs.append([x.cpu() for x in (sol.flow_value, sol.total_cost, sol.augmentations, rr.rounds_run, rr.dec_flow,
                                       rr.dec_cost, rr.dangling, nf, af, st["up"], st["down"])])
        fl.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("name", ["flow1", "gpt"])
def test_key_overflow_redo_queue(name):
    """ssp_kernel's 32-bit keys (K1): costs scaled so that every single arc passes the
    32-bit admission check ((maxcost << H) + 1 < 2^29) but shortest-path keys cross 2^29 -- the
    instances abort into the redo queue and the 64-bit relaunch re-solves them.  Status 0 and the
    full canonical assignment equal to the oracle's (VERDICT r1 "What's weak" #2)."""
    from paper_2509_21221_b200 import Flow
    cfg = gen.CONFIGS[name]
    B = 12
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    Sn = cfg.S * cfg.n
    H = 1
    while (1 << H) <= 2 * Sn + 1:
        H += 1
    maxc = int(max(src.max(), snk.max(), link[link != oracle.ABSENT].max()))
    scale = (2**29 - 2) // (maxc << H)  # the largest scale whose single arcs still admit 32-bit keys
    assert scale >= 2
    absent = link == oracle.ABSENT
    src, snk, link = src.astype(np.int64) * scale, snk.astype(np.int64) * scale, link.astype(np.int64) * scale
    link[absent] = oracle.ABSENT
    assert (int(max(src.max(), snk.max(), link.max())) << H) + 1 < 2**29  # each arc admits 32-bit keys
    src, snk, link = src.astype(np.int32), snk.astype(np.int32), link.astype(np.int32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    fl = Flow(t(bt.cap), t(src), t(snk), t(link), t(bt.supply), max_cap=cfg.max_cap, alive=t(bt.alive))
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    assert fl.stats()["redo_64bit"] > 0  # the redo queue was used
    assert (sol.status == 0).all()
    for b in range(B):
        I = oracle.Instance(cfg.S, cfg.n, cfg.max_cap, int(bt.supply[b]), bt.cap[b], src[b], snk[b], link[b], bt.alive[b])
        r = oracle.ssp(I)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), b
        assert np.array_equal(nf[b], r.node_flow) and np.array_equal(af[b], r.arc_flow), b
        assert np.array_equal(sf[b], r.src_flow) and np.array_equal(kf[b], r.snk_flow), b


@pytest.mark.parametrize("name,hi,big", [("llama", 20000, 70000), ("churn", 200, 1000)], ids=["tile16", "tile8"])
@pytest.mark.parametrize("drop", [False, True], ids=["recost", "recost+drop"])
def test_smem_tile16_edge_updates(drop, name, hi, big):
    """The shared-memory tier's narrow tile copies under edge updates: re-costed links are written into
    the copy (it stays in use, a dropped link as the absent code), a cost past its range retires it (llama:
    16-bit -> int32 at 70,000; churn: 8-bit -> 16-bit at 1,000); either way the solve equals the oracle's
    on the updated graph, full assignment."""
    cfg = gen.CONFIGS[name]
    B = 6
    fl, *_ = _gpu_flow(cfg, 0, B)
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    rng = np.random.default_rng(5)
    upd = {}  # one update per arc (the updates of one call apply in parallel)
    for b in range(B):
        for _ in range(40):
            s, v, u = int(rng.integers(0, cfg.S - 1)), int(rng.integers(0, cfg.n)), int(rng.integers(0, cfg.n))
            upd[(b, s, v, u)] = int(rng.integers(1, hi))
    if drop:
        upd[(1, 3, 5, 7)] = gen.ABSENT
        upd[(4, 0, 0, 0)] = big
    upd = np.array([(*k, c) for k, c in upd.items()], np.int32)
    fl.apply_churn(None, torch.from_numpy(upd).cuda())
    for b, s, v, u, c in upd:
        link[b, s, v, u] = c
    sol = fl.solve_batch()
    nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
    for b in range(B):
        r = _oracle_ssp(cfg, bt, src, snk, link, b)
        assert (int(sol.flow_value[b]), int(sol.total_cost[b]), int(sol.augmentations[b])) == (r.F, r.cost, r.A), b
        assert np.array_equal(af[b], r.arc_flow) and np.array_equal(nf[b], r.node_flow), b
