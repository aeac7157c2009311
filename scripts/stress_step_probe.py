"""Stress step variants: solve alone, rounds alone, serial, and concurrent (solve_and_rounds), device
time with CUDA events; GWTF_ROUNDS_CLUSTER_SIZE / GWTF_CLUSTER_SIZE select the cluster sizes.
  python scripts/stress_step_probe.py [solve] [rounds] [serial] [concurrent]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2509_21221_b200 import Flow  # noqa: E402

cfg = gen.CONFIGS["stress"]
bt = gen.generate(cfg, 0, cfg.B, device="cuda")
fl = Flow(bt.cap, bt.src, bt.snk, bt.link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
del bt.link
fl.snapshot()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
res = {"rounds_cluster": os.environ.get("GWTF_ROUNDS_CLUSTER_SIZE"), "ssp_cluster": os.environ.get("GWTF_CLUSTER_SIZE")}


def timed(name, fn):
    fl.restore()
    torch.cuda.synchronize()
    ev[0].record(fl.stream)
    out = fn()
    ev[1].record(fl.stream)
    torch.cuda.synchronize()
    res[name] = ev[0].elapsed_time(ev[1])
    return out


for what in sys.argv[1:] or ["solve", "rounds", "concurrent"]:
    if what == "solve":
        s = timed("solve_ms", lambda: fl.solve_batch())
        res["A"] = int(s.augmentations.sum())
    elif what == "rounds":
        r = timed("rounds_ms", lambda: fl.decentralized_rounds(cfg.max_rounds))
        res["F_dec"] = int(r.dec_flow.sum())
    elif what == "serial":
        timed("serial_ms", lambda: (fl.solve_batch(), fl.decentralized_rounds(cfg.max_rounds)))
    elif what == "concurrent":
        timed("concurrent_ms", lambda: fl.solve_and_rounds(cfg.max_rounds))
print(json.dumps(res), flush=True)
