"""Oracle trajectory of the decentralized rounds on full-size stress instances (64 x 1,024,
M = 4,096, cold start, max_rounds = 120 + 2M): rounds run, F_dec, cost_dec, dangling, the final
state digest, every 256th per-round digest and the SHA-256 of the whole digest sequence, written
to tests/golden/stress_rounds.json.  Calls only gen/ and oracle/ (seed 17).

  python scripts/stress_rounds_golden.py [--inst 0 ...] [--out PATH]
  python scripts/stress_rounds_golden.py --merge PART.json ...   (parts written by parallel --out runs)
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
ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "stress_rounds.json"))
ap.add_argument("--merge", nargs="+", default=None, help="merge part files into the golden file and exit")
a = ap.parse_args()
cfg = gen.CONFIGS["stress"]
out_path = a.out
if a.merge:
    gold = os.path.join(ROOT, "tests", "golden", "stress_rounds.json")
    res = json.load(open(gold))
    for part in a.merge:
        res["instances"].update(json.load(open(part))["instances"])
    res["instances"] = dict(sorted(res["instances"].items(), key=lambda kv: int(kv[0])))
    with open(gold, "w") as f:
        json.dump(res, f, indent=1)
    sys.exit(0)
res = json.load(open(out_path)) if os.path.exists(out_path) else {
    "source": "scripts/stress_rounds_golden.py (oracle.Rounds on gen.CONFIGS['stress'], seed 17)", "seed": 17,
    "max_rounds": cfg.max_rounds, "instances": {}}
for i in a.inst:
    t = time.time()
    bt = gen.generate(cfg, i, 1)
    I = oracle.instance_from_batch(bt, 0, bt.link[0], bt.src[0], bt.snk[0])
    R = oracle.Rounds(I, seed=17, inst_id=i)
    o = R.run(cfg.max_rounds, digests=True)
    d = np.ascontiguousarray(o["digests"], np.uint64)
    res["instances"][str(i)] = {"rounds": int(o["rounds"]), "F_dec": int(o["F_dec"]), "cost_dec": int(o["cost_dec"]),
                                "dangling": int(o["dangling"]), "final_digest": str(int(d[-1])),
                                "digest_every_256": [str(int(x)) for x in d[::256]],
                                "digests_sha256": hashlib.sha256(d.tobytes()).hexdigest(),
                                "oracle_seconds": round(time.time() - t, 1)}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(i, {k: v for k, v in res["instances"][str(i)].items() if k != "digest_every_256"}, flush=True)
