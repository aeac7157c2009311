"""Multi-data-node flows, exact-solve part: the oracle's
decomposition pinned (one data node = the plain SSP; capacities never exceeded; data node k only
uses what the earlier ones left, so it matches a plain SSP on those residual capacities), and
(-m gpu) the CUDA path against it on flow-test settings 5 and 6."""
import numpy as np
import pytest
import torch

import gen
import oracle
from oracle import Instance


def _inputs(name, B):
    cfg = gen.CONFIGS[name]
    K = cfg.extra["data_nodes"]
    bt = gen.generate(cfg, 0, B)
    xs, xk = gen.generate_data_nodes(cfg, 0, B, K)
    srcs = [bt.src] + [xs[k] for k in range(K - 1)]
    snks = [bt.snk] + [xk[k] for k in range(K - 1)]
    return cfg, K, bt, srcs, snks


@pytest.mark.parametrize("name", ["flow5", "flow6"])
def test_multisource_oracle_pins(name):
    cfg, K, bt, srcs, snks = _inputs(name, 8)
    for b in range(8):
        I = oracle.instance_from_batch(bt, b)
        res = oracle.multi_source_ssp(I, [s[b] for s in srcs], [k[b] for k in snks], [cfg.M] * K)
        r0 = oracle.ssp(I)
        assert (res[0][0], res[0][1]) == (r0.F, r0.cost)  # data node 0 alone = the plain SSP
        used = sum(r[2] for r in res)
        assert (used <= I.cap_eff()).all()
        cap = I.cap_eff().copy()
        for k, (F, C, nf) in enumerate(res):  # each data node: a plain SSP on what was left
            Ik = Instance(I.S, I.n, I.max_cap, cfg.M, cap, srcs[k][b], snks[k][b], I.link)
            rk = oracle.ssp(Ik)
            assert (F, C) == (rk.F, rk.cost) and np.array_equal(nf, rk.node_flow)
            assert oracle.network_simplex(Ik) == (F, C)  # and it is that problem's optimum
            cap = cap - nf


def test_multisource_unit_oracle_pins():
    """Round-robin by microbatch.  With one data node on these complete layered graphs (every link
    present, every relay alive) routing unit by unit still reaches the max flow (a stage with spare
    capacity always connects to the next), and its first unit costs what the plain SSP's first
    augmentation costs (the cost curve at 1); later units cannot reroute earlier ones, so the total
    is at least the optimum.  With several data nodes: capacities respected, and the data nodes'
    flows add up to at most the single-commodity max flow."""
    cfg, K, bt, srcs, snks = _inputs("flow5", 6)
    for b in range(6):
        I = oracle.instance_from_batch(bt, b)
        one = oracle.multi_source_ssp_unit(I, [srcs[0][b]], [snks[0][b]], [cfg.M])
        r0 = oracle.ssp(I, curve=True)
        assert one[0][0] == r0.F and one[0][1] >= r0.cost
        first = oracle.multi_source_ssp_unit(I, [srcs[0][b]], [snks[0][b]], [1])
        assert first[0][1] == r0.curve[1]
        res = oracle.multi_source_ssp_unit(I, [s[b] for s in srcs], [k[b] for k in snks], [cfg.M] * K)
        assert (sum(r[2] for r in res) <= I.cap_eff()).all()
        assert sum(r[0] for r in res) <= r0.F


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["flow5", "flow6"])
def test_multisource_unit_gpu_parity(name):
    from paper_2509_21221_b200.multisource import multi_source_ssp_unit
    B = 32
    cfg, K, bt, srcs, snks = _inputs(name, B)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sup = [d(np.full(B, cfg.M, np.int64)) for _ in range(K)]
    res = multi_source_ssp_unit(d(bt.cap), d(bt.alive), d(bt.link), [d(s) for s in srcs], [d(k) for k in snks], sup,
                                max_cap=cfg.max_cap)
    torch.cuda.synchronize()
    for b in range(B):
        I = oracle.instance_from_batch(bt, b)
        o = oracle.multi_source_ssp_unit(I, [s[b] for s in srcs], [k[b] for k in snks], [cfg.M] * K)
        for k in range(K):
            assert (int(res[k][0][b]), int(res[k][1][b])) == (o[k][0], o[k][1]), (b, k)
            assert np.array_equal(res[k][2][b].cpu().numpy(), o[k][2]), (b, k)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["flow5", "flow6"])
def test_multisource_gpu_parity(name):
    from paper_2509_21221_b200.multisource import multi_source_ssp
    B = 64
    cfg, K, bt, srcs, snks = _inputs(name, B)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sup = [d(np.full(B, cfg.M, np.int64)) for _ in range(K)]
    res = multi_source_ssp(d(bt.cap), d(bt.alive), d(bt.link), [d(s) for s in srcs], [d(k) for k in snks], sup,
                           max_cap=cfg.max_cap)
    torch.cuda.synchronize()
    for b in range(B):
        I = oracle.instance_from_batch(bt, b)
        o = oracle.multi_source_ssp(I, [s[b] for s in srcs], [k[b] for k in snks], [cfg.M] * K)
        for k in range(K):
            assert (int(res[k][0][b]), int(res[k][1][b])) == (o[k][0], o[k][1]), (b, k)
            assert np.array_equal(res[k][2][b].cpu().numpy(), o[k][2]), (b, k)
