"""GPU parity of warm-start rerouting (gwtf_flow_warm_reroute).

Bar ("parity on (F, cost) only"): the optimum's (F, cost) is unique, so the
warm result must equal, bit for bit, the cold exact solve of the same churned graph (GPU, itself
oracle-parity-tested), the oracle's warm reroute and the oracle's network simplex; its assignment
must pass the oracle's certificate (conservation, capacity, maximality, no negative residual cycle)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from oracle import ABSENT, Instance
from tests import harness

pytestmark = pytest.mark.gpu


def _churn(cfg, bt, seed, kill_p=0.1, drop_p=0.05, recost_p=0.05):
    """Seeded test churn: crash relays, drop links (ABSENT), re-cost links (edge updates)."""
    rng = np.random.default_rng(seed)
    alive = bt.alive.copy()
    alive[rng.random(alive.shape) < kill_p] = 0
    upd = []
    if cfg.S > 1:
        B = alive.shape[0]
        shape = (B, cfg.S - 1, cfg.n, cfg.n)
        x = rng.random(shape)  # disjoint drop / re-cost sets: updates of one call apply in parallel
        drop = np.argwhere(x < drop_p)
        rec = np.argwhere((x >= drop_p) & (x < drop_p + recost_p))
        for b, s, v, u in drop:
            upd.append((b, s, v, u, ABSENT))
        for (b, s, v, u), c in zip(rec, rng.integers(1, 200, len(rec))):
            upd.append((b, s, v, u, int(c)))
    return alive, np.array(upd, np.int32).reshape(-1, 5)


def _host_instance(cfg, bt, src, snk, link, b, alive=None, upd=None):
    lk = link[b].copy()
    if upd is not None:
        for bb, s, v, u, c in upd:
            if bb == b:
                lk[s, v, u] = c
    return Instance(cfg.S, cfg.n, cfg.max_cap, int(bt.supply[b]), bt.cap[b], src[b], snk[b], lk,
                    bt.alive[b] if alive is None else alive[b])


@pytest.mark.parametrize("repair_all", [True, False], ids=["repair", "triage"])
@pytest.mark.parametrize("name,B,samples", [("tiny", 256, 32), ("gpt", 128, 16), ("flow3", 32, 8), ("llama", 8, 4),
                                            ("churn", 4, 2)])
def test_warm_reroute_parity(name, B, samples, repair_all):
    """repair: every instance through the repair kernels (GWTF_WARM_REPAIR_ALL); triage: the default,
    small or heavily damaged instances re-solved cold on the subset."""
    from paper_2509_21221_b200 import Flow
    cfg = gen.CONFIGS[name]
    hbt, hsrc, hsnk, hlink = harness.host_inputs(cfg, 0, B)
    dbt, src, snk, link = harness.device_inputs(cfg, 0, B)
    fl = Flow(dbt.cap, src, snk, link, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive, warm_repair_all=repair_all)
    fl.solve_batch()
    nf, sf, kf, af = fl.get_assignment()
    base = [oracle.SSPResult(0, 0, 0, nf[b].cpu().numpy(), sf[b].cpu().numpy(), kf[b].cpu().numpy(),
                             af[b].cpu().numpy()) for b in range(min(B, samples))]
    alive, upd = _churn(cfg, hbt, seed=7)
    fl.apply_churn(torch.from_numpy(alive).cuda(), torch.from_numpy(upd).cuda() if len(upd) else None)
    F, C, St, Q = fl.warm_reroute(nf, sf, kf, af)
    cold = fl.solve_batch()
    torch.cuda.synchronize()
    assert int(Q.abs().sum()) == 0
    assert torch.equal(F, cold.flow_value) and torch.equal(C, cold.total_cost)
    st = St.cpu().numpy()
    assert st[:, 0].sum() > 0  # the churn really cut carried flow
    ncold = fl.stats()["warm_cold_instances"]
    if not repair_all and (cfg.S - 1) * cfg.n * cfg.n < 4096:
        assert ncold == B  # below the triage's size bound every instance is solved cold
    for b in range(min(B, samples)):
        I0 = _host_instance(cfg, hbt, hsrc, hsnk, hlink, b)
        I1 = _host_instance(cfg, hbt, hsrc, hsnk, hlink, b, alive, upd)
        want = oracle.network_simplex(I1)
        assert (int(F[b]), int(C[b])) == want
        ow, _ = oracle.warm_reroute(I0, base[b], I1)
        assert (ow.F, ow.cost) == want
        assert oracle.certify(I1, int(F[b]), int(C[b]), nf[b].cpu().numpy(), sf[b].cpu().numpy(),
                              kf[b].cpu().numpy(), af[b].cpu().numpy()) == 0


def test_warm_reroute_no_churn_identity():
    from paper_2509_21221_b200 import Flow
    cfg = gen.CONFIGS["gpt"]
    dbt, src, snk, link = harness.device_inputs(cfg, 0, 64)
    fl = Flow(dbt.cap, src, snk, link, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive, warm_repair_all=True)
    sol = fl.solve_batch()
    nf, sf, kf, af = fl.get_assignment()
    nf0, af0 = nf.clone(), af.clone()
    F, C, St, Q = fl.warm_reroute(nf, sf, kf, af)
    torch.cuda.synchronize()
    assert torch.equal(F, sol.flow_value) and torch.equal(C, sol.total_cost)
    assert int(St.abs().sum()) == 0 and int(Q.abs().sum()) == 0
    assert torch.equal(nf, nf0) and torch.equal(af, af0)


def test_warm_reroute_host_pointer_mode():
    from paper_2509_21221_b200 import Flow
    cfg = gen.CONFIGS["tiny"]
    hbt, hsrc, hsnk, hlink = harness.host_inputs(cfg, 0, 64)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    fl = Flow(t(hbt.cap), t(hsrc), t(hsnk), t(hlink), t(hbt.supply), max_cap=cfg.max_cap, alive=t(hbt.alive),
              host=True)
    fl.solve_batch()
    nf, sf, kf, af = fl.get_assignment()
    alive, upd = _churn(cfg, hbt, seed=9, kill_p=0.2)
    fl.apply_churn(t(alive), t(upd) if len(upd) else None)
    F, C, St, Q = fl.warm_reroute(nf, sf, kf, af)
    cold = fl.solve_batch()
    assert torch.equal(F, cold.flow_value) and torch.equal(C, cold.total_cost) and int(Q.abs().sum()) == 0


@pytest.mark.parametrize("repair_all", [False, True])
def test_warm_reroute_cluster_tier(repair_all):
    """The cold subset through the cluster tier (its positive-arc lists and weights redirected to
    scratch, node / src / snk flows straight into the caller's arrays): stress distributions at 8 x 256."""
    from paper_2509_21221_b200 import Flow
    cfg = gen.CONFIGS["stress_s"]
    B = 3
    hbt, hsrc, hsnk, hlink = harness.host_inputs(cfg, 0, B)
    dbt, src, snk, link = harness.device_inputs(cfg, 0, B)
    fl = Flow(dbt.cap, src, snk, link, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive, force_cluster_tier=True,
              warm_repair_all=repair_all)
    fl.solve_batch()
    nf, sf, kf, af = fl.get_assignment()
    alive, upd = _churn(cfg, hbt, seed=11, kill_p=0.05)
    fl.apply_churn(torch.from_numpy(alive).cuda(), torch.from_numpy(upd).cuda() if len(upd) else None)
    F, C, St, Q = fl.warm_reroute(nf, sf, kf, af)
    cold = fl.solve_batch()
    torch.cuda.synchronize()
    assert int(Q.abs().sum()) == 0
    assert torch.equal(F, cold.flow_value) and torch.equal(C, cold.total_cost)
    I1 = _host_instance(cfg, hbt, hsrc, hsnk, hlink, 0, alive, upd)
    assert oracle.certify(I1, int(F[0]), int(C[0]), nf[0].cpu().numpy(), sf[0].cpu().numpy(), kf[0].cpu().numpy(),
                          af[0].cpu().numpy()) == 0
