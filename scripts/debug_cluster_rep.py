"""Repeats small forced-cluster-tier solves (flow1, gpt, flow3) 80 times against the oracle (races show up as mismatches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from tests import harness
from paper_2509_21221_b200 import Flow
res = []
for name, B in (("flow1", 16), ("gpt", 16), ("flow3", 16)):
    cfg = gen.CONFIGS[name]
    dbt, src, snk, link = harness.device_inputs(cfg, 0, B)
    ok = 0
    for rep in range(5):
        fl = Flow(dbt.cap, src, snk, link, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive, force_cluster_tier=True)
        sol = fl.solve_batch(); torch.cuda.synchronize()
        ok += int((sol.status == 0).sum())
        fl.close()
    res.append(f"{name}: ok {ok}/{5*B}")
print(os.environ.get("GWTF_DEBUG_FLAGS", "0"), " | ".join(res))
