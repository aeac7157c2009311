"""Multi-GPU parity (SURVEY.md 4 tests/dist, 8(e)): one sharded pass of the churn protocol over
`total` instances on N ranks (torchrun, NCCL), gathered with paper_2509_21221_b200.dist.solve_sharded;
rank 0 then re-solves every instance on one GPU (a single handle over all ids) and checks the
gathered [total][8] results are byte-identical, and checks sampled instances against the oracle.
  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/dist_parity.py gpt 100"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gen  # noqa: E402
from paper_2509_21221_b200 import dist as gdist  # noqa: E402
from tests import harness  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gpt"
total = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = gen.CONFIGS[name]
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)


def make_shard(lo, hi):
    bt, src, snk, link = harness.device_inputs(cfg, lo, hi - lo, device=dev)
    make_shard.alive = bt.alive
    return bt.cap, src, snk, link, bt.supply, bt.alive


def churn(fl, lo, hi):
    if cfg.churn == "random":
        an, upd = harness.churn_inputs(cfg, lo, make_shard.alive, device=dev)
        fl.apply_churn(an, upd)
    elif cfg.churn == "victim":
        st = fl.export_round_state()
        an = gen.llama_victims(st["up"].cpu().numpy(), st["down"].cpu().numpy(), make_shard.alive.cpu().numpy(),
                               gen.victim_draws(cfg, lo, hi - lo))
        fl.apply_churn(torch.from_numpy(an).to(dev))


kw = dict(max_cap=cfg.max_cap, seed=0)
ch = churn if cfg.churn != "none" else None
g, fl = gdist.solve_sharded(make_shard, total, cfg.max_rounds, rank=rank, world=world, churn=ch, **kw)
torch.cuda.synchronize()
if rank == 0:
    ref, _ = gdist.solve_sharded(make_shard, total, cfg.max_rounds, rank=0, world=1, churn=ch, **kw)
    same = bool(torch.equal(g.cpu(), ref.cpu()))
    # sampled instances against the oracle (whole churn step, one instance at a time)
    ids = sorted({0, total - 1, total // 2, *np.random.default_rng(1).integers(0, total, 5).tolist()})
    ok = 0
    import oracle
    for i in ids:
        row = g[i].cpu().numpy()
        if cfg.churn == "none":  # cold: exact solve + rounds from the empty state
            bt, src, snk, link = harness.host_inputs(cfg, i, 1)
            I = oracle.instance_from_batch(bt, 0, link[0], src[0], snk[0])
            s = oracle.ssp(I)
            r = oracle.Rounds(I, seed=0, inst_id=i).run(cfg.max_rounds)
            want = [s.F, s.cost, s.A, 0, r["rounds"], r["F_dec"], r["cost_dec"], r["dangling"]]
        else:  # the churn protocol: pre-churn rounds, churn, cold solve, repair rounds
            o = harness.oracle_pipeline(cfg, i, 1, seed=0)
            want = [int(o["F"][0]), int(o["cost"][0]), int(o["A"][0]), 0, int(o["rounds"][0]), int(o["F_dec"][0]),
                    int(o["cost_dec"][0]), int(o["dangling"][0])]
        ok += [int(x) for x in row] == want
    res = {"config": name, "world": world, "total": total, "shards": [gdist.shard_range(total, world, r) for r in range(world)],
           "gathered_equals_single_gpu": same, "oracle_sampled": len(ids), "oracle_equal": ok,
           "totals": gdist.totals(g)}
    print(json.dumps(res), flush=True)
    if not same or ok != len(ids):
        sys.exit(3)
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
