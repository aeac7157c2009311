"""bench.py -- instances/sec of the GWTF routing hot path (BASELINE.json metric) on N B200s.

One step = one pass of the whole hot path over this GPU's batch of the churn protocol
(SURVEY.md 8(d)): apply_churn (crash/rejoin masks) -> cold exact SSP solve on the masked
graph -> decentralized repair rounds to steady state -> (N>1) NCCL all_gather of the
per-instance results.  The pre-churn converged state is built once (untimed) and restored
before every step (untimed, like the L2 flush).  Workload: configs[1] of BASELINE.json
(GPT-like 300M: 6 stages x 16 clients, 64 microbatches, 10% churn), B instances per GPU
(weak scaling).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config gpt]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gwtf", choices=["gwtf", "reference"])
    ap.add_argument("--config", default="gpt")
    ap.add_argument("--batch", type=int, default=0, help="instances per GPU (default: the config's B)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle instances for cpu_baseline (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip e2e, cpu baseline and stress tier (profiling runs)")
    ap.add_argument("--no-stress-tier", action="store_true", help="skip the stress-config exact-solve measurement")
    ap.add_argument("--no-addition", action="store_true", help="skip the node-addition optimizer measurement")
    return ap.parse_args()


def workload_name(cfg):
    return (f"{cfg.name}: {cfg.S} stages x {cfg.n} clients/stage, M={cfg.M} microbatches, caps U{{{cfg.cap[0]}..{cfg.cap[1]}}}, "
            + ("Eq.1 costs over 10 locations" if cfg.cost_kind == gen.COST_EQ1 else f"costs U{{{cfg.cost[0]}..{cfg.cost[1]}}}")
            + f", churn={cfg.churn}")


def algorithmic_bytes_ssp(cfg, A_total):
    """an SSP shortest-path step examines every forward arc once:
    bytes/augmentation = E x sizeof(cost), E = (S-1) n^2 + 2n, int32 costs."""
    E = (cfg.S - 1) * cfg.n * cfg.n + 2 * cfg.n
    return float(A_total) * E * 4


def load_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture of this bench
    command (profiles/<round>/traffic.json, written by scripts/ncu_traffic.py), else None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")), reverse=True):
        try:
            with open(path) as f:
                t = json.load(f)
            if kernel in t.get("kernels", {}):
                return t["kernels"][kernel], os.path.relpath(path, ROOT)
        except Exception:
            pass
    return None, None


def stress_tier(dev):
    """The HBM-streaming tier on the stress config (SURVEY.md 8(d) tier G): 8 instances of 64
    stages x 1,024 clients, M = 4,096, one cold exact solve through the cluster-tier kernel.
    Algorithmic bytes = sum_b A_b x E x 4 (E = (S-1) n^2 + 2n int32 arc costs per augmentation)."""
    import torch

    from paper_2509_21221_b200 import Flow
    from tests import harness
    cfg = gen.CONFIGS["stress"]
    bt, src, snk, link = harness.device_inputs(cfg, 0, cfg.B, device=dev)
    fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
    del link
    torch.cuda.synchronize()
    fl.set_profiling(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(fl.stream)
    sol = fl.solve_batch()
    ev1.record(fl.stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    kt = fl.kernel_times()
    ev0.record(fl.stream)
    rr = fl.decentralized_rounds(cfg.max_rounds)  # cold, to steady state (W = 5) or max_rounds
    ev1.record(fl.stream)
    torch.cuda.synchronize()
    rms = ev0.elapsed_time(ev1)
    fl.set_profiling(False)
    A = int(sol.augmentations.sum().item())
    alg = algorithmic_bytes_ssp(cfg, A)
    kname = "ssp_cluster_kernel" if "ssp_cluster_kernel" in kt else max(kt, key=lambda k: kt[k][0])
    kms = kt[kname][0]
    peak, peak_src = load_peaks()
    tr, tsrc = load_traffic("stress:" + kname)
    # the capture ran a supply-capped solve: its DRAM bytes per augmentation x this launch's A
    traffic = tr["dram_bytes_per_aug"] * A if tr and "dram_bytes_per_aug" in tr else None
    out = {"workload": workload_name(cfg), "instances": cfg.B, "solve_ms": ms, "rounds_ms": rms,
           "instances_per_s": cfg.B / ((ms + rms) / 1e3), "ssp_instances_per_s": cfg.B / (ms / 1e3),
           "rounds_instances_per_s": cfg.B / (rms / 1e3), "augmentations": A,
           "rounds_run": [int(x) for x in rr.rounds_run.tolist()], "max_rounds": cfg.max_rounds,
           "F": int(sol.flow_value.sum().item()), "cost": int(sol.total_cost.sum().item()),
           "F_dec": int(rr.dec_flow.sum().item()), "cost_dec": int(rr.dec_cost.sum().item()),
           "status_ok": bool((sol.status == 0).all().item()),
           "roofline": {"kernel": kname, "bound": "hbm", "achieved": alg / (kms / 1e3) / 1e9, "peak": peak,
                        "unit": "GB/s", "frac": alg / (kms / 1e3) / 1e9 / peak, "peak_source": peak_src,
                        "algorithmic_bytes_per_launch": alg, "traffic": traffic, "traffic_source": tsrc}}
    fl.close()
    return out


def node_addition(dev, steps=5):
    """SURVEY.md 8(f) f1 on node-addition setting 1 (PAPER.md Table "Node addition", 8 stages x 12
    clients + 8 candidates): all 8! = 40,320 placements built, solved and reduced on the device per
    step; improvement (cost_now - cost_after)/cost_now of the optimal placement and the two
    baselines (capacity-first, random) over the base instance."""
    import torch

    from paper_2509_21221_b200 import Flow, addition
    cfg = gen.CONFIGS["addition"]
    bt = gen.generate(cfg, 0, 1)
    cand = gen.generate_candidates(cfg, 0)
    cap = (bt.cap[0] * (bt.alive[0] != 0)).astype(np.int32)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    args = (d(cap), d(bt.src[0]), d(bt.snk[0]), d(bt.link[0]), d(cand["cap"]), d(cand["cin"]), d(cand["cout"]),
            d(cand["cc"]), int(cfg.M))
    r = addition.optimal_addition(*args, max_cap=cfg.max_cap)  # warm-up
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(steps):
        r = addition.optimal_addition(*args, max_cap=cfg.max_cap)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    base = Flow(d(cap[None]), d(bt.src[:1]), d(bt.snk[:1]), d(bt.link[:1]),
                torch.full((1,), cfg.M, dtype=torch.int64, device=dev), max_cap=cfg.max_cap)
    bs = base.solve_batch()
    F0, C0 = int(bs.flow_value[0]), int(bs.total_cost[0])
    base.close()
    cost = r["all_cost"].cpu().numpy()
    cf = addition.placement_index(addition.capacity_first(cand["cap"], cap.sum(axis=1), F0))
    rnd = addition.placement_index(addition.random_placement(cfg.S, 0))
    return {"workload": f"node addition setting 1: {cfg.S} stages x {cfg.n} clients + {cfg.S} candidates, "
                        f"M={cfg.M}, caps U{{1..20}}, costs U{{1..100}}",
            "placements": addition.num_placements(cfg.S), "ms_per_optimization": ms,
            "placements_per_s": addition.num_placements(cfg.S) / (ms / 1e3),
            "base": {"F": F0, "cost": C0}, "optimal": {"perm": r["perm"], "F": r["F"], "cost": r["cost"],
                                                       "improvement": addition.improvement(C0, r["cost"])},
            "capacity_first": {"cost": int(cost[cf]), "improvement": addition.improvement(C0, int(cost[cf]))},
            "random": {"cost": int(cost[rnd]), "improvement": addition.improvement(C0, int(cost[rnd]))}}


def flow_quality(dev, B=256):
    """PAPER.md:612-620 ablation, flow-test settings 1-4: the decentralized rounds
    (120 iterations), the SWARM greedy baseline and the optimum (exact solve) on B seeded
    instances each; mean costs, mean flows and GWTF's improvement over SWARM
    (cost_swarm - cost_gwtf) / cost_swarm over the instances where both route the same flow."""
    import torch

    from paper_2509_21221_b200 import Flow
    from tests import harness
    out = {}
    for name in ("flow1", "flow2", "flow3", "flow4"):
        cfg = gen.CONFIGS[name]
        bt, src, snk, link = harness.device_inputs(cfg, 0, B, device=dev)
        fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
        sol = fl.solve_batch()
        rr = fl.decentralized_rounds(120)
        gF, gC = fl.greedy_baseline()
        torch.cuda.synchronize()
        F, C = sol.flow_value.double(), sol.total_cost.double()
        dF, dC = rr.dec_flow.double(), rr.dec_cost.double()
        same = (dF == gF.double()) & (gF > 0)
        imp = ((gC.double() - dC) / gC.double())[same]
        out[name] = {"instances": B, "F_opt": float(F.mean()), "F_gwtf": float(dF.mean()), "F_swarm": float(gF.double().mean()),
                     "cost_opt": float(C.mean()), "cost_gwtf": float(dC.mean()), "cost_swarm": float(gC.double().mean()),
                     "gwtf_vs_swarm_improvement_mean": float(imp.mean()) if imp.numel() else None,
                     "gwtf_vs_swarm_improvement_max": float(imp.max()) if imp.numel() else None,
                     "same_flow_instances": int(same.sum())}
        fl.close()
    return out


def other_configs(dev, steps=5, warmup=3):
    """The other churn-protocol configs of SURVEY.md 8(d) on this GPU, same step and timing as the
    main line (device events, L2 flushed, restore untimed): tiny (cold, no churn), llama (victim
    crash), churn (random crash/rejoin + link drops)."""
    import torch

    from paper_2509_21221_b200 import Flow
    from tests import harness
    out = {}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for name in ("tiny", "llama", "churn"):
        cfg = gen.CONFIGS[name]
        B, mr = cfg.B, cfg.max_rounds
        bt, src, snk, link = harness.device_inputs(cfg, 0, B, device=dev)
        fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
        an = upd = None
        if cfg.churn != "none":
            fl.decentralized_rounds(mr)
            if cfg.churn == "random":
                an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
            else:
                st = fl.export_round_state()
                an = torch.from_numpy(gen.llama_victims(st["up"].cpu().numpy(), st["down"].cpu().numpy(),
                                                        bt.alive.cpu().numpy(), gen.victim_draws(cfg, 0, B))).to(dev)
        fl.snapshot()
        sol = fl.solve_batch()
        rr = fl.decentralized_rounds(mr)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        total = 0.0
        for it in range(warmup + steps):
            fl.restore()
            flush.random_(0, 255)
            torch.cuda.synchronize()
            ev0.record(fl.stream)
            if an is not None or upd is not None:
                fl.apply_churn(an, upd)
            fl.solve_batch(out=sol)
            fl.decentralized_rounds(mr, out=rr)
            ev1.record(fl.stream)
            torch.cuda.synchronize()
            if it >= warmup:
                total += ev0.elapsed_time(ev1)
        out[name] = {"workload": workload_name(cfg), "instances": B, "ms_per_step": total / steps,
                     "instances_per_s": B * steps / (total / 1e3),
                     "augmentations_mean": float(sol.augmentations.double().mean()),
                     "rounds_mean": float(rr.rounds_run.double().mean())}
        fl.close()
    return out


def warm_reroute(dev, names=("gpt", "llama"), steps=5, warmup=3):
    """warm-start rerouting (gwtf_flow_warm_reroute) after the config's churn event,
    from the pre-churn optimum, against the cold exact solve of the same churned graph (device events,
    L2 flushed, restore and the assignment copy untimed).  (F, cost) must agree on every instance."""
    import torch

    from paper_2509_21221_b200 import Flow
    from tests import harness
    out = {}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for name in names:
        cfg = gen.CONFIGS[name]
        B = cfg.B
        bt, src, snk, link = harness.device_inputs(cfg, 0, B, device=dev)
        fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0)
        fl.solve_batch()
        base = [t.clone() for t in fl.get_assignment()]
        if cfg.churn == "random":
            an, upd = harness.churn_inputs(cfg, 0, bt.alive, device=dev)
        else:  # victim churn needs the round state: run the base rounds first
            fl.decentralized_rounds(cfg.max_rounds)
            st = fl.export_round_state()
            an = torch.from_numpy(gen.llama_victims(st["up"].cpu().numpy(), st["down"].cpu().numpy(),
                                                    bt.alive.cpu().numpy(), gen.victim_draws(cfg, 0, B))).to(dev)
            upd = None
        fl.snapshot()
        work = [t.clone() for t in base]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        tw = tc = 0.0
        for it in range(warmup + steps):
            fl.restore()
            fl.apply_churn(an, upd)
            for w, b0 in zip(work, base):
                w.copy_(b0)
            flush.random_(0, 255)
            torch.cuda.synchronize()
            ev[0].record(fl.stream)
            F, C, S, Q = fl.warm_reroute(*work)
            ev[1].record(fl.stream)
            flush.random_(0, 255)
            ev[2].record(fl.stream)
            cold = fl.solve_batch()
            ev[3].record(fl.stream)
            torch.cuda.synchronize()
            if it >= warmup:
                tw += ev[0].elapsed_time(ev[1])
                tc += ev[2].elapsed_time(ev[3])
        out[name] = {"workload": workload_name(cfg), "instances": B, "warm_ms": tw / steps, "cold_ms": tc / steps,
                     "warm_instances_per_s": B * steps / (tw / 1e3), "cold_instances_per_s": B * steps / (tc / 1e3),
                     "F_cost_mismatches": int(((F != cold.flow_value) | (C != cold.total_cost)).sum()),
                     "status_nonzero": int((Q != 0).sum()), "stripped": int(S[:, 0].sum()),
                     "cycles": int(S[:, 1].sum()), "augmentations": int(S[:, 2].sum()),
                     "cold_augmentations": int(cold.augmentations.sum())}
        fl.close()
    return out


def multi_source(dev, B=8192, reps=1):
    """SURVEY.md 8(f) f2, exact-solve part: flow-test settings 5 and 6 (2 / 4 data nodes),
    single-commodity solves over the residual capacities in round-robin order, one
    microbatch per data node per turn, B instances."""
    import torch

    from paper_2509_21221_b200.multisource import multi_source_ssp_unit as multi_source_ssp
    out = {}
    for name in ("flow5", "flow6"):
        cfg = gen.CONFIGS[name]
        K = cfg.extra["data_nodes"]
        bt = gen.generate(cfg, 0, B)
        xs, xk = gen.generate_data_nodes(cfg, 0, B, K)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        srcs = [d(bt.src)] + [d(xs[k]) for k in range(K - 1)]
        snks = [d(bt.snk)] + [d(xk[k]) for k in range(K - 1)]
        sup = [d(np.full(B, cfg.M, np.int64)) for _ in range(K)]
        args = (d(bt.cap), d(bt.alive), d(bt.link), srcs, snks, sup)
        multi_source_ssp(*args, max_cap=cfg.max_cap)  # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            res = multi_source_ssp(*args, max_cap=cfg.max_cap)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
        out[name] = {"data_nodes": K, "instances": B, "ms": dt * 1e3, "instances_per_s": B / dt,
                     "F_per_data_node": [float(r[0].double().mean()) for r in res],
                     "cost_per_data_node": [float(r[1].double().mean()) for r in res],
                     "what": "wall clock per batch, one microbatch per data node per turn (a supply-1 solve "
                             "and a handle create per turn)"}
    return out


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 100 ms during the timed loop
    (one `nvidia-smi -lms` stream, started before and stopped after the timed steps)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.strip().splitlines():
            self.rows.append([x.strip() for x in line.split(",")])

    def summary(self):
        num = lambda x: x.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(r[0]) for r in self.rows if r and num(r[0])]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and num(r[1])]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm)}


def cpu_baseline(cfg, target_s=15.0, inst0=0):
    """The oracle (as it stands) on the host cores, on a bounded sample of the same workload,
    sized for about target_s seconds of CPU work (calibrated on a small first sample)."""
    from tests import harness
    threads = os.cpu_count() or 1
    cal = max(threads * 4, 32)
    t = time.perf_counter()
    harness.oracle_pipeline(cfg, inst0, cal, seed=0, threads=threads)
    rate = cal / max(time.perf_counter() - t, 1e-6)
    sample = int(min(max(rate * target_s, cal), 200000))
    t = time.perf_counter()
    harness.oracle_pipeline(cfg, inst0 + cal, sample, seed=0, threads=threads)
    dt = time.perf_counter() - t
    return {"value": sample / dt, "unit": "instances/s", "cores": threads, "kind": "oracle",
            "sample": f"{sample} instances of the same workload (full step: pre-churn rounds + churn + SSP + "
                      f"repair rounds), {dt:.1f} s on {threads} threads, one instance per thread"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle as it stands on the host cores, same metric/config."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = args.cpu_sample or max(64, threads * 48)
    from tests import harness
    for w in range(max(args.warmup, 0)):
        harness.oracle_pipeline(cfg, w * sample, min(sample, 64), seed=0, threads=threads)
    t = time.perf_counter()
    for k in range(args.steps):
        harness.oracle_pipeline(cfg, k * sample, sample, seed=0, threads=threads)
    dt = time.perf_counter() - t
    value = args.steps * sample / dt
    line = {"impl": "reference", "metric": "min-cost-flow instances solved/sec", "value": value,
            "unit": "instances/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "instances_per_step": sample, "parallelism": "host threads"},
            "cpu_baseline": {"value": value, "unit": "instances/s", "cores": threads, "kind": "oracle",
                             "sample": f"{sample} instances per step (bounded sample of the workload)"},
            "e2e": {"value": value, "unit": "instances/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = gen.CONFIGS[args.config]
    if args.batch:
        cfg = cfg.with_(B=args.batch)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2509_21221_b200 import Flow
    from paper_2509_21221_b200.dist import gather_results
    from tests import harness

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B = cfg.B
    inst0 = rank * B  # weak scaling: every rank owns B instances
    mr = cfg.max_rounds

    # ---------------- untimed setup: inputs resident in HBM, pre-churn converged state ----------
    bt, src, snk, link = harness.device_inputs(cfg, inst0, B, device=dev)
    fl = Flow(bt.cap, src, snk, link, bt.supply, max_cap=cfg.max_cap, alive=bt.alive, seed=0, inst_base=inst0)
    fl.decentralized_rounds(mr)
    an, upd = None, None
    if cfg.churn == "random":
        an, upd = harness.churn_inputs(cfg, inst0, bt.alive, device=dev)
    elif cfg.churn == "victim":
        st = fl.export_round_state()
        an = torch.from_numpy(gen.llama_victims(st["up"].cpu().numpy(), st["down"].cpu().numpy(),
                                                bt.alive.cpu().numpy(), gen.victim_draws(cfg, inst0, B))).to(dev)
    fl.snapshot()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    sol = fl.solve_batch()
    rr = fl.decentralized_rounds(mr)
    stream = fl.stream

    # GWTF_BENCH_CONCURRENT=1: the step's solve and rounds through gwtf_flow_solve_and_rounds (two
    # streams; measured ~3% shorter steps, but the per-kernel times then overlap)
    concurrent = os.environ.get("GWTF_BENCH_CONCURRENT", "0") == "1"

    def step():
        fl.apply_churn(an, upd)
        if concurrent:  # exact solve and repair rounds of the step on two streams (independent work)
            fl.solve_and_rounds(mr, out_sol=sol, out_rounds=rr)
        else:
            fl.solve_batch(out=sol)
            fl.decentralized_rounds(mr, out=rr)
        return gather_results(sol, rr, world)

    def prep():
        fl.restore()
        flush.random_(0, 255)  # evict L2 between timed steps

    for _ in range(args.warmup):
        prep()
        step()
    torch.cuda.synchronize()

    fl.set_profiling(True)
    total_ms = 0.0
    A_total = 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = int(fl.stats(raw=True)[15])
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            prep()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            ev0.record(stream)
            g = step()
            ev1.record(stream)
            torch.cuda.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            A_total += int(sol.augmentations.sum().item())
    ktimes = fl.kernel_times()
    fl.set_profiling(False)
    # restore() between steps launches no kernels (device memcpys), so the difference is the steps'
    launches_timed = int(fl.stats(raw=True)[15]) - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = world * B * args.steps / (total_ms / 1e3)

    # ---------------- roofline of the dominant kernel ----------------
    peak, peak_src = load_peaks()
    dom = max(ktimes, key=lambda k: ktimes[k][0])
    dom_ms, dom_launches = ktimes[dom]
    tr, tsrc = load_traffic(dom)
    roof = {"kernel": dom, "bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": peak_src,
            "traffic": tr["dram_bytes_per_launch"] if tr else None, "traffic_source": tsrc}
    if dom == "ssp_kernel":
        alg = algorithmic_bytes_ssp(cfg, A_total)
        roof["achieved"] = alg / (dom_ms / 1e3) / 1e9
        roof["algorithmic_bytes_per_launch"] = alg / max(dom_launches, 1)
    else:
        # rounds: per round every slot's (up, down) state and every relay's advertiser row of the
        # next stage is read once; units from the rounds actually run
        rounds_total = int(rr.rounds_run.sum().item()) * args.steps
        per_round = cfg.S * cfg.n * cfg.max_cap * 8 + cfg.S * cfg.n * cfg.n * 4 + 2 * cfg.M * 4
        alg = float(rounds_total) * per_round
        roof["achieved"] = alg / (dom_ms / 1e3) / 1e9
        roof["algorithmic_bytes_per_launch"] = alg / max(dom_launches, 1)
    roof["frac"] = roof["achieved"] / peak
    kshare = {k: {"ms_total": v[0], "launches": v[1], "share": v[0] / total_ms if total_ms else None}
              for k, v in ktimes.items()}

    line = {"metric": "min-cost-flow instances solved/sec", "value": value, "unit": "instances/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded generator, SURVEY.md 8(d))",
            "config": {"workload": workload_name(cfg), "instances_per_gpu": B, "global_instances": world * B,
                       "max_rounds": mr, "l2": "flushed (256 MiB write) between timed steps; state restore untimed",
                       "parallelism": f"instance-sharded x{world}"},
            "roofline": roof, "kernels": kshare, "clocks": clk.summary(),
            "gpu_launches": None}
    # our kernels launched inside the timed steps, counted by the library (gwtf_flow_stats[15])
    line["gpu_launches"] = launches_timed

    if rank == 0 and not (args.quick or args.no_e2e):
        line["e2e"] = e2e(cfg, B, inst0, dev, args)
    if rank == 0 and not (args.quick or args.no_cpu_baseline):
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0 and world == 1 and not (args.quick or args.no_stress_tier):
        line["stress_tier"] = stress_tier(dev)
    if rank == 0 and world == 1 and not (args.quick or args.no_addition):
        line["node_addition"] = node_addition(dev)
        line["flow_quality"] = flow_quality(dev)
        line["other_configs"] = other_configs(dev)
        line["multi_source"] = multi_source(dev)
        line["warm_reroute"] = warm_reroute(dev)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e(cfg, B, inst0, dev, args):
    """The same metric end to end through the public API in host-pointer mode (GWTF_HOST_PTRS):
    the graph and its pre-churn converged state are resident (created once from pinned host buffers,
    untimed, like the device-timed value's setup); every timed step passes that step's inputs -- the
    churn events (alive mask, link updates) -- from pinned host memory (apply_churn), runs the cold
    exact solve and the repair rounds, and reads every per-instance result back to pinned host
    memory.  Wall clock per step, median; the state restore between steps is untimed.  The
    from-scratch pipeline (create + base rounds + churn + solve + repair) is reported as e2e_cold."""
    import torch

    from paper_2509_21221_b200 import Flow
    from tests import harness
    bt, src, snk, link = harness.device_inputs(cfg, inst0, B, device=dev)
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    h = {k: pin(v) for k, v in dict(cap=bt.cap, alive=bt.alive, src=src, snk=snk, link=link, supply=bt.supply).items()}
    mr = cfg.max_rounds
    fl = Flow(h["cap"], h["src"], h["snk"], h["link"], h["supply"], max_cap=cfg.max_cap, alive=h["alive"],
              seed=0, inst_base=inst0, host=True)
    fl.decentralized_rounds(mr)
    an = upd = None
    if cfg.churn == "random":
        a, u = harness.churn_inputs(cfg, inst0, bt.alive, device=dev)
        an, upd = pin(a), (pin(u) if u is not None else None)
    elif cfg.churn == "victim":
        st = fl.export_round_state()
        an = torch.from_numpy(gen.llama_victims(st["up"].numpy(), st["down"].numpy(), h["alive"].numpy(),
                                                gen.victim_draws(cfg, inst0, B))).pin_memory()
    fl.snapshot()
    h2d = (an.numel() if an is not None else 0) + (upd.numel() * 4 if upd is not None else 0)
    d2h = B * (8 + 8 + 4 + 4) + B * (4 + 8 + 8 + 4)
    times = []
    for it in range(3 + max(3, min(args.steps, 20))):
        fl.restore()
        torch.cuda.synchronize()
        t = time.perf_counter()
        if an is not None or upd is not None:
            fl.apply_churn(an, upd)
        fl.solve_batch()
        fl.decentralized_rounds(mr)
        torch.cuda.synchronize()
        if it >= 3:
            times.append(time.perf_counter() - t)
    fl.close()
    tm = float(np.median(times))
    cold = []
    for it in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f2 = Flow(h["cap"], h["src"], h["snk"], h["link"], h["supply"], max_cap=cfg.max_cap, alive=h["alive"],
                  seed=0, inst_base=inst0, host=True)
        f2.decentralized_rounds(mr)
        if an is not None or upd is not None:
            f2.apply_churn(an, upd)
        f2.solve_batch()
        f2.decentralized_rounds(mr)
        f2.close()
        torch.cuda.synchronize()
        if it >= 1:
            cold.append(time.perf_counter() - t)
    cold_h2d = sum(v.numel() * v.element_size() for v in h.values()) + h2d
    return {"value": B / tm, "unit": "instances/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "what": "per step from pinned host memory: churn events H2D (apply_churn) + cold exact solve + repair "
                    "rounds + every per-instance result D2H; resident graph and pre-churn state (restored, untimed)",
            "e2e_cold": {"value": B / float(np.median(cold)), "unit": "instances/s", "h2d_bytes_per_step": int(cold_h2d),
                         "d2h_bytes_per_step": int(d2h) * 2,
                         "what": "create from pinned host buffers + base rounds + churn + solve + repair rounds + D2H"}}


if __name__ == "__main__":
    main()
