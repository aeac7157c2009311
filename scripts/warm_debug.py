"""Warm repair alone (GWTF_WARM_NO_FALLBACK=1): per-status counts and (F, cost) agreement with the cold
solve on one churn event of a config (victim churn for llama).  python scripts/warm_debug.py llama [B]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2509_21221_b200 import Flow  # noqa: E402
from tests import harness  # noqa: E402

name = sys.argv[1]
cfg = gen.CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dev = torch.device("cuda", 0)
bt, src, snk, link = harness.device_inputs(cfg, 0, B, device=dev)
fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
fl.solve_batch()
base = [t.clone() for t in fl.get_assignment()]
if cfg.churn == "victim":
    fl.decentralized_rounds(cfg.max_rounds)
    st = fl.export_round_state()
    an = torch.from_numpy(gen.llama_victims(st["up"].cpu().numpy(), st["down"].cpu().numpy(), bt.alive.cpu().numpy(),
                                            gen.victim_draws(cfg, 0, B))).to(dev)
    upd = None
else:
    an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
fl.apply_churn(an, upd)
F, C, S, Q = fl.warm_reroute(*base)
cold = fl.solve_batch()
torch.cuda.synchronize()
print(name, "status counts", dict(collections.Counter(Q.tolist())))
ok = (Q == 0)
print("ok instances: F/cost mismatches", int(((F != cold.flow_value) | (C != cold.total_cost))[ok].sum()), "of", int(ok.sum()))
print("stats (cut, sat, iters) of ok:", S[ok][:8].tolist())
