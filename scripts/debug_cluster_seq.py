import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, oracle
from tests import harness
from paper_2509_21221_b200 import Flow
cfg = gen.CONFIGS["gpt"]
b = int(sys.argv[1]) if len(sys.argv) > 1 else 7
dbt, src, snk, link = harness.device_inputs(cfg, b, 1)
fl = Flow(dbt.cap, src, snk, link, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive, force_cluster_tier=True)
sol = fl.solve_batch(); torch.cuda.synchronize()
st = fl.stats(raw=True).astype(np.uint64)
na = int(st[10]); keys = [int(x) for x in st[1000:1000 + na]]
print("inst", b, "status", int(sol.status[0]), "F", int(sol.flow_value[0]), "A", int(sol.augmentations[0]))
print("gpu path costs", [(k >> 20, k & 0xFFFFF) for k in keys])
