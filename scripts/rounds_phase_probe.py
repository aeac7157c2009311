"""Rounds of one churn-protocol step of a config (pre-churn rounds untimed, churn, repair rounds timed)
with the dev-build phase timers (GWTF_DEBUG_FLAGS=16, make DEV=1): leader cycles per phase.
  python scripts/rounds_phase_probe.py gpt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2509_21221_b200 import Flow  # noqa: E402
from tests import harness  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gpt"
cfg = gen.CONFIGS[name]
dev = torch.device("cuda", 0)
bt, src, snk, link = harness.device_inputs(cfg, 0, cfg.B, device=dev)
fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
fl.decentralized_rounds(cfg.max_rounds)
if cfg.churn == "random":
    an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
    fl.apply_churn(an, upd)
fl.snapshot()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for rep in range(3):
    fl.restore()
    torch.cuda.synchronize()
    raw0 = fl.stats(raw=True)
    ev[0].record(fl.stream)
    rr = fl.decentralized_rounds(cfg.max_rounds)
    ev[1].record(fl.stream)
    torch.cuda.synchronize()
    print(f"{name}: repair rounds {ev[0].elapsed_time(ev[1]):.3f} ms, rounds mean {rr.rounds_run.double().mean():.1f} max {int(rr.rounds_run.max())}")
raw = fl.stats(raw=True) - raw0
names = ["start:walk+flush", "r0a-vote", "r0a", "d-scan", "R1", "R2R3", "summ", "R4R5", "R6", "R7"]
cyc = raw[1200:1210].astype(float)
tot = cyc.sum() or 1.0
for nm, c in zip(names, cyc):
    print(f"  {nm:18s} {c:14.0f} {100 * c / tot:5.1f}%")
