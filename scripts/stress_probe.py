"""Stress-shape probe: 64 stages x 1,024 clients, 8 instances, exact solve through the cluster
tier with the supply capped at --supply (bounds the number of augmentations).  Prints the solve
time, augmentations and the algorithmic HBM bytes of the relaxation (E x 4 per augmentation)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2509_21221_b200 import Flow  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--supply", type=int, default=64)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--rounds", type=int, default=0, help="also time decentralized_rounds(max_rounds)")
a = ap.parse_args()
cfg = gen.CONFIGS["stress"]
bt = gen.generate(cfg, 0, a.batch, device="cuda")
bt.supply.fill_(a.supply)
fl = Flow(bt.cap, bt.src, bt.snk, bt.link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive)
del bt.link
torch.cuda.synchronize()
sol = fl.solve_batch()  # warm-up
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(a.reps):
    ev0.record()
    fl.solve_batch(out=sol)
    ev1.record()
    torch.cuda.synchronize()
    ms.append(ev0.elapsed_time(ev1))
A = int(sol.augmentations.sum())
E = (cfg.S - 1) * cfg.n * cfg.n + 2 * cfg.n
alg = A * E * 4
t = min(ms) / 1e3
print(json.dumps({"config": "stress", "B": a.batch, "supply": a.supply, "ms": min(ms), "A_total": A,
                  "F": sol.flow_value.tolist(), "cost": sol.total_cost.tolist(), "status": sol.status.tolist(),
                  "ms_per_aug_per_instance": min(ms) / max(A / a.batch, 1),
                  "algorithmic_GBps": alg / t / 1e9, "stats": fl.stats()}))
if a.rounds:
    ev0.record()
    rr = fl.decentralized_rounds(a.rounds)
    ev1.record()
    torch.cuda.synchronize()
    print(json.dumps({"rounds_ms": ev0.elapsed_time(ev1), "rounds_run": rr.rounds_run.tolist(),
                      "F_dec": rr.dec_flow.tolist(), "cost_dec": rr.dec_cost.tolist()}))
if os.environ.get("GWTF_DEBUG_FLAGS", "0") != "0" and int(os.environ["GWTF_DEBUG_FLAGS"]) & 16:
    raw = fl.stats(raw=True)
    names = ["dense: key gather", "relax(dense, after 1st chunk)", "relax_vote", "tstar", "trev", "backward", "trace", "lookup",
             "augment", "other", "frontier relax", "frontier vote", "dense: wait 1st chunk", "dense: issue + prefetch"]
    cyc = raw[1100:1114].astype(float)
    tot = cyc.sum()
    print("phase cycles (leader thread, all solves, summed over clusters):")
    for nm, c in zip(names, cyc):
        print(f"  {nm:10s} {c:14.0f}  {100 * c / tot:5.1f}%")
if os.environ.get("GWTF_DEBUG_FLAGS", "0") != "0" and int(os.environ["GWTF_DEBUG_FLAGS"]) & 2048:
    raw = fl.stats(raw=True)
    h = raw[1200:1216]
    print("changed columns per non-first relaxation (bucket: 0, 1, 2-3, 4-7, ...):", h.tolist())
