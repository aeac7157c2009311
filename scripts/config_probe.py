"""Per-kernel times of one churn-protocol step for a config (device events, library profiling)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from tests import harness
from paper_2509_21221_b200 import Flow
name = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = gen.CONFIGS[name]
B = B or cfg.B
dev = torch.device("cuda", 0)
bt, src, snk, link = harness.device_inputs(cfg, 0, B, device=dev)
fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
fl.decentralized_rounds(cfg.max_rounds)
an = upd = None
if cfg.churn == "random":
    an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
fl.snapshot()
for rep in range(2):
    fl.restore()
    fl.set_profiling(True)
    if an is not None:
        fl.apply_churn(an, upd)
    sol = fl.solve_batch()
    rr = fl.decentralized_rounds(cfg.max_rounds)
    torch.cuda.synchronize()
    kt = fl.kernel_times()
    fl.set_profiling(False)
print(name, B, fl.stats(), {k: round(v[0], 2) for k, v in kt.items()}, "rounds mean", float(rr.rounds_run.double().mean()),
      "A mean", float(sol.augmentations.double().mean()), "rounds>=max", int((rr.rounds_run >= cfg.max_rounds).sum()))
