import sys, os, json
sys.path.insert(0, "/root/repo")
import torch, numpy as np, gen
from paper_2509_21221_b200 import Flow
from tests import harness
name = sys.argv[1]; cfg = gen.CONFIGS[name]; B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.B
dev = torch.device("cuda", 0)
bt, src, snk, link = harness.device_inputs(cfg, 0, B, device=dev)
fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
fl.solve_batch()
base = [t.clone() for t in fl.get_assignment()]
an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
fl.apply_churn(an, upd)
F, C, S, Q = fl.warm_reroute(*base)
torch.cuda.synchronize()
S = S.cpu().numpy(); f0 = base[1].sum(1).cpu().numpy()
rep = 4 * S[:, 0] <= f0
print("repaired", int(rep.sum()), "of", B)
R = S[rep]
print(json.dumps({"iters_pct": np.percentile(R[:, 2], [50, 90, 99, 100]).tolist(), "cut_pct": np.percentile(R[:, 0], [50, 90, 99, 100]).tolist(),
                  "sat_pct": np.percentile(R[:, 1], [50, 90, 99, 100]).tolist()}))
for k in range(3):
    torch.cuda.synchronize(); e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    w = [t.clone() for t in base]; e[0].record(fl.stream); fl.warm_reroute(*w); e[1].record(fl.stream); torch.cuda.synchronize()
    print("warm ms", e[0].elapsed_time(e[1]))
os.environ["GWTF_PROFILE"] = "1"
