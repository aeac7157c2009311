"""Phase timing of bench.py's e2e_cold pipeline (create from pinned host buffers, base rounds, churn,
solve, repair rounds, close), several repetitions, to separate allocation cost from kernel time."""
import json
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import gen  # noqa: E402
from paper_2509_21221_b200 import Flow  # noqa: E402
from tests import harness  # noqa: E402


def main():
    cfg = gen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "gpt"]
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    bt, src, snk, link = harness.device_inputs(cfg, 0, B, device="cuda")
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    h = {k: pin(v) for k, v in dict(cap=bt.cap, alive=bt.alive, src=src, snk=snk, link=link, supply=bt.supply).items()}
    a, u = harness.churn_inputs(cfg, 0, bt.alive, device="cuda")
    an, upd = pin(a), (pin(u) if u is not None else None)
    out = []
    for it in range(5):
        ph = {}
        torch.cuda.synchronize()
        t = time.perf_counter()
        f2 = Flow(h["cap"], h["src"], h["snk"], h["link"], h["supply"], max_cap=cfg.max_cap, alive=h["alive"],
                  seed=0, host=True)
        torch.cuda.synchronize(); ph["create"] = time.perf_counter() - t; t = time.perf_counter()
        f2.decentralized_rounds(cfg.max_rounds)
        torch.cuda.synchronize(); ph["base_rounds"] = time.perf_counter() - t; t = time.perf_counter()
        f2.apply_churn(an, upd)
        torch.cuda.synchronize(); ph["churn"] = time.perf_counter() - t; t = time.perf_counter()
        f2.solve_batch()
        torch.cuda.synchronize(); ph["solve"] = time.perf_counter() - t; t = time.perf_counter()
        f2.decentralized_rounds(cfg.max_rounds)
        torch.cuda.synchronize(); ph["repair"] = time.perf_counter() - t; t = time.perf_counter()
        f2.close()
        torch.cuda.synchronize(); ph["close"] = time.perf_counter() - t
        out.append({k: round(v * 1e3, 2) for k, v in ph.items()})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
