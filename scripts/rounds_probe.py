"""Rounds run per instance in the GPT churn protocol (base convergence and repair), augmentations per solve."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import gen
from tests import harness
from paper_2509_21221_b200 import Flow
cfg = gen.CONFIGS["gpt"]
dev = torch.device("cuda", 0)
bt, src, snk, link = harness.device_inputs(cfg, 0, cfg.B, device=dev)
fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
rr0 = fl.decentralized_rounds(cfg.max_rounds)
an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
fl.apply_churn(an, upd)
sol = fl.solve_batch()
rr = fl.decentralized_rounds(cfg.max_rounds)
torch.cuda.synchronize()
a0 = rr0.rounds_run.cpu().numpy(); a = rr.rounds_run.cpu().numpy()
print("base rounds: mean %.1f max %d; repair rounds: mean %.2f p50 %d p90 %d max %d" % (a0.mean(), a0.max(), a.mean(), np.median(a), np.percentile(a, 90), a.max()))
A = sol.augmentations.cpu().numpy(); print("augmentations mean %.1f max %d" % (A.mean(), A.max()))
print(np.bincount(a)[:40])
