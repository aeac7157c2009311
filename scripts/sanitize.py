"""One small pass of a kernel family for compute-sanitizer (racecheck / synccheck / memcheck /
initcheck), e.g.  compute-sanitizer --tool racecheck python scripts/sanitize.py ssp gpt
  family: ssp | ssp_cluster | rounds | rounds_cluster | warm | churn;  config: tiny | gpt | stress_s | ...
Parity is checked elsewhere; this only drives each kernel once on a few instances."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from tests import harness  # noqa: E402

fam, name = sys.argv[1], sys.argv[2]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = gen.CONFIGS[name]
if fam == "rounds_cluster":
    os.environ.update(GWTF_ROUNDS_GLOBAL="1", GWTF_ROUNDS_CLUSTER="1")
from paper_2509_21221_b200 import Flow  # noqa: E402

bt, src, snk, link = harness.device_inputs(cfg, 0, B)
fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=1,
          force_cluster_tier=fam == "ssp_cluster")
mr = min(cfg.max_rounds, 200)
if fam in ("ssp", "ssp_cluster"):
    sol = fl.solve_batch()
    print("F", sol.flow_value.tolist(), "status", sol.status.tolist())
elif fam in ("rounds", "rounds_cluster"):
    rr = fl.decentralized_rounds(mr, digests=True)
    print("rounds", rr.rounds_run.tolist(), "F_dec", rr.dec_flow.tolist())
elif fam == "churn":
    fl.decentralized_rounds(mr)
    an, upd = harness.churn_inputs(cfg.with_(crash_p=0.2, rejoin_p=0.2, linkdrop_p=0.05), 0, bt.alive, device=bt.alive.device)
    fl.apply_churn(an, upd)
    st = fl.export_round_state()
    fl.import_round_state(st)
    print("churn ok")
elif fam == "warm":
    fl.solve_batch()
    base = [t.clone() for t in fl.get_assignment()]
    an, upd = harness.churn_inputs(cfg.with_(crash_p=0.2, rejoin_p=0.2), 0, bt.alive, device=bt.alive.device)
    fl.apply_churn(an, upd)
    F, C, S, Q = fl.warm_reroute(*base)
    print("warm F", F.tolist(), "status", Q.tolist())
torch.cuda.synchronize()
print("done")
