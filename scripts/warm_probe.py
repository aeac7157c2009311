"""Warm-start rerouting (gwtf_flow_warm_reroute) vs the cold exact solve on one churn-protocol
step of a config: device time of each (CUDA events on the handle's stream, after a warm-up),
(F, cost) agreement, and the warm work counters.
  python scripts/warm_probe.py gpt [B] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
from paper_2509_21221_b200 import Flow
from tests import harness

name = sys.argv[1]
cfg = gen.CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) else cfg.B
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = torch.device("cuda", 0)
bt, src, snk, link = harness.device_inputs(cfg, 0, B, device=dev)
st = torch.cuda.Stream(dev)
fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0, stream=st)
fl.solve_batch()
base = [t.clone() for t in fl.get_assignment()]
an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
fl.snapshot()
work = [t.clone() for t in base]
tw, tc = [], []
for r in range(reps + 1):
    fl.restore()
    fl.apply_churn(an, upd)
    for w, b in zip(work, base):
        w.copy_(b)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(st)
    F, C, S, Q = fl.warm_reroute(*work)
    e[1].record(st)
    cold = fl.solve_batch()
    e[2].record(st)
    torch.cuda.synchronize()
    if r:
        tw.append(e[0].elapsed_time(e[1]))
        tc.append(e[1].elapsed_time(e[2]))
out = {"config": name, "B": B, "warm_ms": sorted(tw)[len(tw) // 2], "cold_ms": sorted(tc)[len(tc) // 2],
       "F_mismatch": int((F != cold.flow_value).sum()), "cost_mismatch": int((C != cold.total_cost).sum()),
       "status_nonzero": int((Q != 0).sum()), "units_cut": int(S[:, 0].sum()),
       "cold_subset_per_call": fl.stats()["warm_cold_instances"] // (reps + 1), "cold_augment": int(cold.augmentations.sum())}
print(json.dumps(out))
