"""Oracle values for the full-size stress instances (64 x 1,024, M = 4,096): F, cost, A and
SHA-256 digests of the canonical assignment, written to tests/golden/stress_ssp.json.

Calls only gen/ (inputs) and oracle/ (values); the GPU test tests/test_gpu_parity.py::
test_stress_full_golden compares the CUDA path against this file.  Runtime: ~1-2 h per
instance on one core (Dijkstra over 66 M arcs per augmentation), hence a stored file.

  python scripts/stress_golden.py [--inst 0 1 ...] [--out PATH]
  python scripts/stress_golden.py --merge PART.json ...   (parts written by parallel --out runs)
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--inst", type=int, nargs="+", default=[0])
ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "stress_ssp.json"))
ap.add_argument("--merge", nargs="+", default=None, help="merge part files into the golden file and exit")
a = ap.parse_args()
cfg = gen.CONFIGS["stress"]
out_path = a.out
if a.merge:
    gold = os.path.join(ROOT, "tests", "golden", "stress_ssp.json")
    res = json.load(open(gold))
    for part in a.merge:
        res["instances"].update(json.load(open(part))["instances"])
    res["instances"] = dict(sorted(res["instances"].items(), key=lambda kv: int(kv[0])))
    with open(gold, "w") as f:
        json.dump(res, f, indent=1)
    sys.exit(0)
res = json.load(open(out_path)) if os.path.exists(out_path) else {
    "source": "scripts/stress_golden.py (oracle.ssp on gen.CONFIGS['stress'])", "instances": {}}
for i in a.inst:
    t = time.time()
    bt = gen.generate(cfg, i, 1)
    I = oracle.instance_from_batch(bt, 0, bt.link[0], bt.src[0], bt.snk[0])
    r = oracle.ssp(I)
    sha = lambda x: hashlib.sha256(np.ascontiguousarray(x, dtype=np.int32).tobytes()).hexdigest()  # noqa: E731
    res["instances"][str(i)] = {"F": int(r.F), "cost": int(r.cost), "A": int(r.A),
                                "node_flow_sha256": sha(r.node_flow), "arc_flow_sha256": sha(r.arc_flow),
                                "src_flow_sha256": sha(r.src_flow), "snk_flow_sha256": sha(r.snk_flow),
                                "oracle_seconds": round(time.time() - t, 1)}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(i, res["instances"][str(i)], flush=True)
