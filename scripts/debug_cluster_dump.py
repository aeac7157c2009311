import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from tests import harness
from paper_2509_21221_b200 import Flow
cfg = gen.CONFIGS["gpt"]
B = 1
inst0 = int(os.environ.get("INST", "7"))
dbt, src, snk, link = harness.device_inputs(cfg, inst0, B)
for rep in range(40):
    fl = Flow(dbt.cap, src, snk, link, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive, force_cluster_tier=True)
    sol = fl.solve_batch(); torch.cuda.synchronize()
    break
b = 0
print("rep", rep, "failing instance", b, "statuses", sol.status.tolist())
st = fl.stats(raw=True).astype(np.uint64)
nf, sf, kf, af = [x.cpu().numpy() for x in fl.get_assignment()]
json.dump(dict(inst=b, F=int(sol.flow_value[b]), status=int(sol.status[b]), stats=[int(x) for x in st[:2000]],
               cap=dbt.cap[b:b+1].cpu().numpy().tolist(), alive=dbt.alive[b:b+1].cpu().numpy().tolist(), src=src[b:b+1].cpu().numpy().tolist(),
               snk=snk[b:b+1].cpu().numpy().tolist(), link=link[b:b+1].cpu().numpy().tolist(), g=nf[b:b+1].tolist(), srcf=sf[b:b+1].tolist(), snkf=kf[b:b+1].tolist(),
               arcs=af[b:b+1].tolist()), open("gpurun_out/dump.json", "w"))
print("done", b)
