"""Stress rounds from the empty state (the bench step's rounds half), dev-build phase timers
(make DEV=1, GWTF_DEBUG_FLAGS=16): leader cycles per round phase.  GWTF_ROUNDS_CLUSTER_SIZE picks
the cluster size (2 = the size used beside the solve).
  python scripts/stress_rounds_phases.py [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2509_21221_b200 import Flow  # noqa: E402

cfg = gen.CONFIGS["stress"]
R = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.max_rounds
bt = gen.generate(cfg, 0, cfg.B, device="cuda")
fl = Flow(bt.cap, bt.src, bt.snk, bt.link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
del bt.link
fl.snapshot()
raw0 = fl.stats(raw=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(fl.stream)
rr = fl.decentralized_rounds(R)
ev[1].record(fl.stream)
torch.cuda.synchronize()
print(f"stress rounds: {ev[0].elapsed_time(ev[1]):.1f} ms, rounds {int(rr.rounds_run.max())}, cluster "
      f"{os.environ.get('GWTF_ROUNDS_CLUSTER_SIZE', 'auto')}")
raw = fl.stats(raw=True) - raw0
names = ["start:walk+flush", "r0a-vote", "r0a", "d-scan", "R1", "R2R3", "summ", "R4R5", "R6", "R7"]
cyc = raw[1200:1210].astype(float)
tot = cyc.sum() or 1.0
for nm, c in zip(names, cyc):
    print(f"  {nm:18s} {c:14.0f} {100 * c / tot:5.1f}%")
