"""Test/bench harness: moves generated inputs to the device, runs the churn protocol of
SURVEY.md 8(d) through the product binding or through the oracle.  Imports the oracle only
in the oracle_* helpers (test infrastructure)."""
from __future__ import annotations

import numpy as np

import gen

KIND = {"none": 0, "random": 1, "victim": 2}


def host_inputs(cfg, inst0, B):
    """Generated instance batch on the host with oracle-side Eq. 1 tiles (for the oracle)."""
    import oracle
    bt = gen.generate(cfg, inst0, B)
    if cfg.cost_kind == gen.COST_EQ1:
        src, snk, link = oracle.eq1_batch(bt)
    else:
        src, snk, link = bt.src, bt.snk, bt.link
    return bt, src, snk, link


def device_inputs(cfg, inst0, B, device="cuda"):
    """Generated batch on the device; Eq. 1 tiles built by the product's eq1 kernel."""
    import torch
    from paper_2509_21221_b200 import eq1_cost_tiles
    bt = gen.generate(cfg, inst0, B, device=device)
    if cfg.cost_kind == gen.COST_EQ1:
        src, snk, link = eq1_cost_tiles(bt.comp, bt.loc, bt.dloc, bt.lat, bt.bw, cfg.size_kbit)
    else:
        src, snk, link = bt.src, bt.snk, bt.link
    torch.cuda.synchronize()
    return bt, src, snk, link


def churn_inputs(cfg, inst0, alive, device=None):
    """alive_new + edge updates of the 'random' churn protocol."""
    an, ld = gen.generate_churn(cfg, inst0, alive, device=device)
    return an, gen.linkdrop_to_updates(ld)


def gpu_pipeline(cfg, inst0, B, seed=0, digests=True, max_rounds=None, **flow_kw):
    """Base create -> rounds to quiescence -> churn -> cold solve -> repair rounds, on the GPU."""
    import torch
    from paper_2509_21221_b200 import Flow
    bt, src, snk, link = device_inputs(cfg, inst0, B)
    mr = cfg.max_rounds if max_rounds is None else max_rounds
    fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=seed,
              inst_base=inst0, **flow_kw)
    pre = fl.decentralized_rounds(mr)
    if cfg.churn == "random":
        an, upd = churn_inputs(cfg, inst0, bt.alive, device=bt.alive.device)
        fl.apply_churn(an, upd)
    elif cfg.churn == "victim":
        st = fl.export_round_state()
        an = gen.llama_victims(st["up"].cpu().numpy(), st["down"].cpu().numpy(), bt.alive.cpu().numpy(),
                               gen.victim_draws(cfg, inst0, B))
        fl.apply_churn(torch.from_numpy(an).to(bt.alive.device))
    sol = fl.solve_batch()
    rr = fl.decentralized_rounds(mr, digests=digests)
    torch.cuda.synchronize()
    return fl, pre, sol, rr


def oracle_pipeline(cfg, inst0, B, seed=0, threads=None, max_rounds=None):
    import oracle
    bt, src, snk, link = host_inputs(cfg, inst0, B)
    an = upd = vd = None
    if cfg.churn == "random":
        an, upd = churn_inputs(cfg, inst0, bt.alive)
    elif cfg.churn == "victim":
        vd = gen.victim_draws(cfg, inst0, B)
    return oracle.pipeline_batch(cfg, bt.cap, bt.alive, src, snk, link, bt.supply, churn_kind=KIND[cfg.churn],
                                 alive_new=an, updates=upd, victim_draws=vd, seed=seed, inst_base=inst0,
                                 max_rounds=max_rounds, threads=threads)
