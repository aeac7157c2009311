"""SWARM-style greedy routing baseline:
the oracle pinned by the SPEC examples and the optimality invariant, and (-m gpu) the CUDA
kernel against it."""
import numpy as np
import pytest
import torch

import gen
import oracle
from oracle import ABSENT, Instance
from tests import harness


def _one_stage(src, cap, snk=None, M=1):
    n = len(src)
    return Instance(1, n, 3, M, np.array([cap]), np.array(src), np.array(snk or [0] * n), np.zeros((0, n, n)))


def test_greedy_spec_examples():
    """successors 7, 3, 5 -> the 3; all full -> nothing routed; tie -> lowest id."""
    F, C, paths = oracle.greedy_route(_one_stage([7, 3, 5], [1, 1, 1], snk=[0, 10, 0]))
    assert (F, C, paths) == (1, 13, [[1]])
    assert oracle.greedy_route(_one_stage([7, 3, 5], [0, 0, 0]))[0] == 0
    assert oracle.greedy_route(_one_stage([9, 3, 3], [1, 1, 1]))[2] == [[1]]
    # capacity runs out one hop at a time: M = 3 over caps 1, 1, 1 takes ids 1, 2, 0 (costs 3, 5, 7)
    F, C, paths = oracle.greedy_route(_one_stage([7, 3, 5], [1, 1, 1], M=3))
    assert (F, C, paths) == (3, 15, [[1], [2], [0]])
    # a dead end stops the routing and releases the partial path: stage 1 reachable only from id 0
    link = np.full((1, 2, 2), ABSENT)
    link[0, :, 0] = 1
    I = Instance(2, 2, 3, 2, np.array([[1, 1], [1, 1]]), np.array([5, 1]), np.array([0, 0]), link)
    assert oracle.greedy_route(I)[:2] == (0, 0)  # greedy picks id 1 first: no successor


@pytest.mark.parametrize("name", ["tiny", "flow1", "flow2", "flow3", "flow4", "gpt", "churn"])
def test_greedy_invariants(name):
    """the oracle's optimum costs no more than the greedy assignment at the same flow
    value; greedy paths respect capacities and their costs add up."""
    cfg = gen.CONFIGS[name]
    bt, src, snk, link = harness.host_inputs(cfg, 0, 6)
    for b in range(6):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        F, C, paths = oracle.greedy_route(I)
        r = oracle.ssp(I)
        I.M = F  # the oracle's minimum cost of exactly F microbatches
        rF = oracle.ssp(I)
        assert F <= r.F and rF.F == F and C >= rF.cost, (name, b)
        use = np.zeros((I.S, I.n), np.int64)
        total = 0
        for p in paths:
            total += int(I.src[p[0]]) + sum(int(I.link[s, p[s + 1], p[s]]) for s in range(I.S - 1)) + int(I.snk[p[-1]])
            for s, v in enumerate(p):
                use[s, v] += 1
        assert total == C and (use <= I.cap_eff()).all(), (name, b)


@pytest.mark.gpu
@pytest.mark.parametrize("name,B", [("tiny", 64), ("flow1", 32), ("flow3", 32), ("flow4", 32), ("gpt", 48),
                                    ("churn", 8), ("llama", 4), ("stress_s", 2)])
def test_greedy_gpu_parity(name, B):
    from paper_2509_21221_b200 import Flow
    cfg = gen.CONFIGS[name]
    dbt, dsrc, dsnk, dlink = harness.device_inputs(cfg, 0, B)
    fl = Flow(dbt.cap, dsrc, dsnk, dlink, dbt.supply, max_cap=cfg.max_cap, alive=dbt.alive)
    F, C = fl.greedy_baseline()
    torch.cuda.synchronize()
    bt, src, snk, link = harness.host_inputs(cfg, 0, B)
    for b in range(B):
        I = oracle.instance_from_batch(bt, b, link[b], src[b], snk[b])
        f, c, _ = oracle.greedy_route(I)
        assert (int(F[b]), int(C[b])) == (f, c), (name, b)
    fl.close()
