"""Stress-shape decentralized rounds probe: 8 instances of 64 x 1,024, cold start.  Runs --skip
rounds (one launch), then --rounds rounds (a second launch, the one to profile: ncu -k
regex:rounds --launch-skip 1 --launch-count 1), and prints both device times, F_dec and the
per-round time of the second launch."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2509_21221_b200 import Flow  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--skip", type=int, default=0)
ap.add_argument("--rounds", type=int, default=200)
ap.add_argument("--batch", type=int, default=8)
a = ap.parse_args()
cfg = gen.CONFIGS["stress"]
bt = gen.generate(cfg, 0, a.batch, device="cuda")
fl = Flow(bt.cap, bt.src, bt.snk, bt.link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
del bt.link
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record(fl.stream)
r0 = fl.decentralized_rounds(max(a.skip, 1))
ev[1].record(fl.stream)
torch.cuda.synchronize()
raw0 = fl.stats(raw=True)
r1 = fl.decentralized_rounds(a.rounds)
ev[2].record(fl.stream)
torch.cuda.synchronize()
t0, t1 = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
print(json.dumps({"skip_rounds": max(a.skip, 1), "skip_ms": t0, "rounds": r1.rounds_run.tolist(), "ms": t1,
                  "ms_per_round": t1 / max(1, int(r1.rounds_run.max())), "F_dec": r1.dec_flow.tolist(),
                  "cost_dec": r1.dec_cost.tolist(), "dangling": r1.dangling.tolist()}))
if int(os.environ.get("GWTF_DEBUG_FLAGS", "0")) & 16:  # dev build: rounds phase cycles (leader thread)
    raw = fl.stats(raw=True) - raw0  # the second launch only
    names = ["start:walk+flush", "r0a-vote", "r0a", "d-scan", "R1", "R2R3", "summ", "R4R5", "R6", "R7"]
    cyc = raw[1200:1210].astype(float)
    tot = cyc.sum() or 1.0
    print("rounds phase cycles (second launch):")
    for nm, c in zip(names, cyc):
        print(f"  {nm:18s} {c:14.0f} {100 * c / tot:5.1f}%")
    w = raw[1220:1224]
    R = max(1, int(r1.rounds_run.max()))
    print(f"per round (all instances): marks {w[0] / R:.0f}, lowest walkers {w[1] / R:.0f}, up steps {w[2] / R:.0f}, down steps {w[3] / R:.0f}")
