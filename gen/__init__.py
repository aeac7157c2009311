"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

Input plumbing only (see gen/gwtf_gen.h): raw random fields, no method arithmetic.
The config registry below is the recipe DESIGN.md section 4 documents; the shapes
follow BASELINE.json "configs" and SURVEY.md 8(d).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field, replace

import numpy as np

BASE_SEED = 250921221
ABSENT = np.iinfo(np.int32).max
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _thr(p: float) -> int:
    """Probability -> 32-bit threshold used by gen_bernoulli ((draw>>32) < thr)."""
    return min(1 << 32, int(round(p * (1 << 32))))


class GenConfig(ctypes.Structure):
    _fields_ = [
        ("cfg_id", ctypes.c_uint32), ("S", ctypes.c_int32), ("n", ctypes.c_int32),
        ("max_cap", ctypes.c_int32), ("M", ctypes.c_int64),
        ("cap_lo", ctypes.c_int32), ("cap_hi", ctypes.c_int32),
        ("alive_thr", ctypes.c_uint64), ("absent_thr", ctypes.c_uint64),
        ("cost_kind", ctypes.c_int32), ("cost_lo", ctypes.c_int32), ("cost_hi", ctypes.c_int32),
        ("L", ctypes.c_int32), ("comp_lo", ctypes.c_int32), ("comp_hi", ctypes.c_int32),
        ("lat_inter_lo", ctypes.c_int32), ("lat_inter_hi", ctypes.c_int32),
        ("lat_intra_lo", ctypes.c_int32), ("lat_intra_hi", ctypes.c_int32),
        ("bw_inter_lo", ctypes.c_int32), ("bw_inter_hi", ctypes.c_int32), ("bw_intra", ctypes.c_int32),
        ("size_kbit", ctypes.c_int64),
        ("crash_thr", ctypes.c_uint64), ("rejoin_thr", ctypes.c_uint64), ("linkdrop_thr", ctypes.c_uint64),
    ]


COST_DIRECT, COST_EQ1 = 0, 1


@dataclass(frozen=True)
class Config:
    """One workload: instance shape, value distributions, churn protocol and bench batch."""
    name: str
    cfg_id: int
    S: int
    n: int
    M: int
    max_cap: int
    cap: tuple
    B: int                       # instances per GPU in bench / full-size parity
    cost_kind: int = COST_DIRECT
    cost: tuple = (1, 20)
    alive_p: float = 1.0
    absent_p: float = 0.0
    # Eq. 1 raw parameters (C6 #22-23 of SURVEY.md)
    L: int = 10
    comp: tuple = (50, 200)
    lat_inter: tuple = (10, 150)
    lat_intra: tuple = (1, 5)
    bw_inter: tuple = (50, 500)
    bw_intra: int = 1000
    size_kbit: int = 0
    # churn (SURVEY.md 8(d) churn protocol)
    churn: str = "none"          # none | random | victim
    crash_p: float = 0.0
    rejoin_p: float = 0.0
    linkdrop_p: float = 0.0
    max_rounds: int = 0          # 120 + 2M (PAPER.md:618 budget + fill time)
    extra: dict = field(default_factory=dict)

    def ctype(self) -> GenConfig:
        c = GenConfig()
        c.cfg_id, c.S, c.n, c.max_cap, c.M = self.cfg_id, self.S, self.n, self.max_cap, self.M
        c.cap_lo, c.cap_hi = self.cap
        c.alive_thr, c.absent_thr = _thr(self.alive_p), _thr(self.absent_p)
        c.cost_kind = self.cost_kind
        c.cost_lo, c.cost_hi = self.cost
        c.L = self.L
        c.comp_lo, c.comp_hi = self.comp
        c.lat_inter_lo, c.lat_inter_hi = self.lat_inter
        c.lat_intra_lo, c.lat_intra_hi = self.lat_intra
        c.bw_inter_lo, c.bw_inter_hi = self.bw_inter
        c.bw_intra, c.size_kbit = self.bw_intra, self.size_kbit
        c.crash_thr, c.rejoin_thr, c.linkdrop_thr = _thr(self.crash_p), _thr(self.rejoin_p), _thr(self.linkdrop_p)
        return c

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


# GPT activation: microbatch 4 x seq 512 x d_model 1024 x 2 B x 32 = 1,073,741,824 bit
# LLaMA-7B activation: seq 4096 x d 4096 x 2 B = 268,435,456 bit
CONFIGS = {
    "tiny": Config("tiny", 0, S=3, n=3, M=8, max_cap=3, cap=(1, 3), B=65536, cost=(1, 20),
                   max_rounds=120 + 2 * 8),
    "gpt": Config("gpt", 1, S=6, n=16, M=64, max_cap=3, cap=(1, 3), B=16384, cost_kind=COST_EQ1,
                  alive_p=0.9, size_kbit=1073742, churn="random", crash_p=0.1, rejoin_p=0.1,
                  max_rounds=120 + 2 * 64),
    "llama": Config("llama", 2, S=16, n=32, M=256, max_cap=3, cap=(1, 3), B=4096, cost_kind=COST_EQ1,
                    size_kbit=268435, churn="victim", max_rounds=120 + 2 * 256),
    "churn": Config("churn", 3, S=8, n=64, M=256, max_cap=20, cap=(1, 20), B=8192, cost=(1, 100),
                    alive_p=0.9, churn="random", crash_p=0.1, rejoin_p=0.1, linkdrop_p=0.01,
                    max_rounds=120 + 2 * 256),
    "stress": Config("stress", 4, S=64, n=1024, M=4096, max_cap=20, cap=(1, 20), B=8, cost=(1, 100),
                     max_rounds=120 + 2 * 4096),
    # stress shape scaled down (same distributions) for oracle parity of the cluster tier
    "stress_s": Config("stress_s", 5, S=8, n=256, M=512, max_cap=20, cap=(1, 20), B=8, cost=(1, 100),
                       max_rounds=120 + 2 * 512),
    # stress distributions at 64 x 512: 2Sn+2 >= 2^16 hop values, so the cluster tier's 32-bit keys
    # carry >= 17 hop bits (its shift-and-mask weight path), with a small supply for the oracle
    "stress_h": Config("stress_h", 6, S=64, n=512, M=16, max_cap=20, cap=(1, 20), B=2, cost=(1, 100),
                       max_rounds=120 + 2 * 16),
    # stress distributions at 3 x 1,024: the cluster tier's 1,024-column 8-bit fast path (register keys)
    # with a supply small enough for the oracle in seconds
    "stress_w": Config("stress_w", 8, S=3, n=1024, M=1500, max_cap=20, cap=(1, 20), B=2, cost=(1, 100),
                       max_rounds=120 + 2 * 1500),
    # node-addition setting 1 (PAPER.md:446-471 and its Table, "Node addition (top)"): 97 nodes = 1 data
    # holder + 8 stages x 12 clients, capacities U{1..20}, interlayer costs U{1..100}; S candidates join
    "addition": Config("addition", 7, S=8, n=12, M=64, max_cap=20, cap=(1, 20), B=1, cost=(1, 100),
                       max_rounds=120 + 2 * 64),
    # flow-test settings 1-4: 1 source, 40 relays, 8 or 10 stages
    "flow1": Config("flow1", 11, S=8, n=5, M=128, max_cap=3, cap=(1, 3), B=64, cost=(1, 20), max_rounds=120 + 256),
    "flow2": Config("flow2", 12, S=10, n=4, M=128, max_cap=3, cap=(1, 3), B=64, cost=(1, 20), max_rounds=120 + 256),
    "flow3": Config("flow3", 13, S=8, n=5, M=128, max_cap=15, cap=(5, 15), B=64, cost=(1, 20), max_rounds=120 + 256),
    "flow4": Config("flow4", 14, S=8, n=5, M=128, max_cap=3, cap=(1, 3), B=64, cost=(5, 100), max_rounds=120 + 256),
    # flow-test settings 5-6: 2 / 4 data nodes, 40 / 80 relays over 8 stages; the extra
    # data nodes' source and sink costs come from generate_data_nodes()
    "flow5": Config("flow5", 15, S=8, n=5, M=128, max_cap=3, cap=(1, 3), B=64, cost=(1, 20), max_rounds=120 + 256,
                    extra={"data_nodes": 2}),
    "flow6": Config("flow6", 16, S=8, n=10, M=128, max_cap=3, cap=(1, 3), B=64, cost=(1, 20), max_rounds=120 + 256,
                    extra={"data_nodes": 4}),
}


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgwtfgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        L.gen_instances_host.argtypes = [ctypes.POINTER(GenConfig), ctypes.c_uint64, ctypes.c_int64,
                                         ctypes.c_int64] + [P] * 11
        L.gen_churn_host.argtypes = [ctypes.POINTER(GenConfig), ctypes.c_uint64, ctypes.c_int64,
                                     ctypes.c_int64, P, P, P]
        L.gen_instances_device.argtypes = L.gen_instances_host.argtypes + [P]
        L.gen_churn_device.argtypes = L.gen_churn_host.argtypes + [P]
        _LIB = L
    return _LIB


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


@dataclass
class Batch:
    """Raw generated fields of instances [inst0, inst0+B) (numpy on host or torch on device)."""
    cfg: Config
    inst0: int
    B: int
    cap: object
    alive: object
    supply: object
    src: object = None
    snk: object = None
    link: object = None
    comp: object = None
    loc: object = None
    dloc: object = None
    lat: object = None
    bw: object = None


def _alloc(cfg, B, device):
    S, n, L = cfg.S, cfg.n, cfg.L
    if device is None:
        z = lambda shape, dt: np.zeros(shape, dtype=dt)  # noqa: E731
    else:
        import torch
        tmap = {np.int32: torch.int32, np.uint8: torch.uint8, np.int64: torch.int64}
        z = lambda shape, dt: torch.zeros(shape, dtype=tmap[dt], device=device)  # noqa: E731
    bt = Batch(cfg, 0, B, z((B, S, n), np.int32), z((B, S, n), np.uint8), z((B,), np.int64))
    if cfg.cost_kind == COST_DIRECT:
        bt.src, bt.snk = z((B, n), np.int32), z((B, n), np.int32)
        bt.link = z((B, max(S - 1, 0), n, n), np.int32)
    else:
        bt.comp, bt.loc = z((B, S, n), np.int32), z((B, S, n), np.int32)
        bt.dloc, bt.lat, bt.bw = z((B,), np.int32), z((B, L, L), np.int32), z((B, L, L), np.int32)
    return bt


def generate(cfg: Config, inst0: int, B: int, device=None, stream=None, base_seed: int = BASE_SEED) -> Batch:
    """Generate instances [inst0, inst0+B).  device=None -> numpy (host C loop);
    otherwise torch tensors filled by the device twin of the same generator."""
    bt = _alloc(cfg, B, device)
    bt.inst0 = inst0
    c = cfg.ctype()
    args = [bt.cap, bt.alive, bt.supply, bt.src, bt.snk, bt.link, bt.comp, bt.loc, bt.dloc, bt.lat, bt.bw]
    if device is None:
        rc = lib().gen_instances_host(ctypes.byref(c), base_seed, inst0, B, *[_p(a) for a in args])
    else:
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
        rc = lib().gen_instances_device(ctypes.byref(c), base_seed, inst0, B, *[_p(a) for a in args], st)
    if rc != 0:
        raise RuntimeError(f"generator failed rc={rc}")
    return bt


def generate_churn(cfg: Config, inst0: int, alive_base, device=None, stream=None, base_seed: int = BASE_SEED,
                   with_links: bool = True):
    """Churn draws for the 'random' protocol: per relay crash (alive) / rejoin (dead) with
    p and per inter-stage link drop.  Returns (alive_new, linkdrop)."""
    B = alive_base.shape[0]
    S, n = cfg.S, cfg.n
    c = cfg.ctype()
    want_links = with_links and cfg.linkdrop_p > 0 and S > 1
    if device is None:
        alive_new = np.zeros_like(alive_base)
        ld = np.zeros((B, S - 1, n, n), np.uint8) if want_links else None
        rc = lib().gen_churn_host(ctypes.byref(c), base_seed, inst0, B, _p(alive_base), _p(alive_new), _p(ld))
    else:
        import torch
        alive_new = torch.zeros_like(alive_base)
        ld = torch.zeros((B, S - 1, n, n), dtype=torch.uint8, device=device) if want_links else None
        st = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
        rc = lib().gen_churn_device(ctypes.byref(c), base_seed, inst0, B, _p(alive_base), _p(alive_new), _p(ld), st)
    if rc != 0:
        raise RuntimeError(f"churn generator failed rc={rc}")
    return alive_new, ld


def linkdrop_to_updates(linkdrop, inst_offset: int = 0):
    """Dense drop mask [B][S-1][n][n] -> edge update list [k][5] = {b, s, v, u, ABSENT} (int32).
    Pure index bookkeeping (numpy or torch)."""
    if linkdrop is None:
        return None
    if isinstance(linkdrop, np.ndarray):
        idx = np.argwhere(linkdrop != 0).astype(np.int32)
        out = np.empty((idx.shape[0], 5), np.int32)
        out[:, :4] = idx
        out[:, 0] += inst_offset
        out[:, 4] = ABSENT
        return out
    import torch
    idx = torch.nonzero(linkdrop).to(torch.int32)
    out = torch.empty((idx.shape[0], 5), dtype=torch.int32, device=linkdrop.device)
    out[:, :4] = idx
    out[:, 0] += inst_offset
    out[:, 4] = ABSENT
    return out


# ----------------------------------------------------------------------------------------
# Python twins of the counter hash (for the LLaMA victim draws) and the victim rule.  The
# victim rule is harness logic (which relay crashes "during backward"): it
# reads only slot occupancy of an exported round state, never the method's arithmetic.
# ----------------------------------------------------------------------------------------
_M64 = (1 << 64) - 1
GEN_F_VICTIM_STAGE, GEN_F_VICTIM_PICK = 15, 16
GEN_F_CAND_CAP, GEN_F_CAND_IN, GEN_F_CAND_OUT, GEN_F_CAND_CC = 17, 18, 19, 20
GEN_F_DN_SRC, GEN_F_DN_SNK = 21, 22


def mix64(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def instance_seed(cfg: Config, inst: int, base_seed: int = BASE_SEED) -> int:
    return mix64(base_seed ^ (cfg.cfg_id << 48) ^ inst)


def draw(iseed: int, field_id: int, idx: int) -> int:
    return mix64(mix64((iseed + field_id * 0x9E3779B97F4A7C15) & _M64) ^ idx)


def pick(x: int, m: int) -> int:
    return ((x >> 32) * m) >> 32


def victim_draws(cfg: Config, inst0: int, B: int, base_seed: int = BASE_SEED) -> np.ndarray:
    out = np.zeros((B, 2), np.uint64)
    for b in range(B):
        s = instance_seed(cfg, inst0 + b, base_seed)
        out[b] = (draw(s, GEN_F_VICTIM_STAGE, 0), draw(s, GEN_F_VICTIM_PICK, 0))
    return out


def llama_victims(up, down, alive, draws) -> np.ndarray:
    """'Crash during backward': draw a stage; among its alive relays holding a PAIRED slot
    (ascending index) crash the drawn one; if none, try the next stage.  up/down [B][S][n][MC]
    (numpy, exported round state), alive [B][S][n].  Returns the new alive mask."""
    up, down, alive = np.asarray(up), np.asarray(down), np.asarray(alive)
    B, S, n, _ = up.shape
    paired = ((up != -1) & (down != -1)).any(axis=3) & (alive != 0)
    out = alive.copy()
    for b in range(B):
        s0 = pick(int(draws[b, 0]), S)
        for t in range(S):
            s = (s0 + t) % S
            cand = np.nonzero(paired[b, s])[0]
            if cand.size:
                out[b, s, cand[pick(int(draws[b, 1]), cand.size)]] = 0
                break
    return out


_C1, _C2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)


def _mix_np(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def _uniform_np(iseed: int, field_id: int, idx, lo: int, hi: int):
    """draw(iseed, field, idx) -> U{lo..hi} for an index array (the same counter hash as draw())."""
    with np.errstate(over="ignore"):
        base = np.uint64((iseed + field_id * 0x9E3779B97F4A7C15) & _M64)
    d = _mix_np(_mix_np(base) ^ np.asarray(idx, dtype=np.uint64))
    return (np.uint64(lo) + (((d >> np.uint64(32)) * np.uint64(hi - lo + 1)) >> np.uint64(32))).astype(np.int32)


def generate_candidates(cfg: Config, inst: int, base_seed: int = BASE_SEED):
    """S joining candidates of node-addition instance `inst` ("every node is a
    candidate for each stage ... each node knows its costs for each stage"): capacity U{cap},
    cost to / from every client of every stage and between candidates U{cost} (inputs of
    gwtf_addition_build; include/gwtf.h documents the layout)."""
    S, n = cfg.S, cfg.n
    s = instance_seed(cfg, inst, base_seed)
    cap = _uniform_np(s, GEN_F_CAND_CAP, np.arange(S), cfg.cap[0], cfg.cap[1])
    cin = _uniform_np(s, GEN_F_CAND_IN, np.arange(S * S * n), cfg.cost[0], cfg.cost[1]).reshape(S, S, n)
    cout = _uniform_np(s, GEN_F_CAND_OUT, np.arange(S * S * n), cfg.cost[0], cfg.cost[1]).reshape(S, S, n)
    cc = _uniform_np(s, GEN_F_CAND_CC, np.arange(S * S), cfg.cost[0], cfg.cost[1]).reshape(S, S)
    return {"cap": cap, "cin": cin, "cout": cout, "cc": cc}


def generate_data_nodes(cfg: Config, inst0: int, B: int, K: int, base_seed: int = BASE_SEED):
    """Source and sink costs of data nodes 1..K-1 of instances inst0.. (data node 0 keeps the batch's
    src/snk): src [K-1][B][n], snk [K-1][B][n], costs U{cost} like the flow-test links."""
    n = cfg.n
    src = np.zeros((max(K - 1, 0), B, n), np.int32)
    snk = np.zeros_like(src)
    for b in range(B):
        s = instance_seed(cfg, inst0 + b, base_seed)
        for k in range(1, K):
            idx = np.arange((k - 1) * n, k * n)
            src[k - 1, b] = _uniform_np(s, GEN_F_DN_SRC, idx, cfg.cost[0], cfg.cost[1])
            snk[k - 1, b] = _uniform_np(s, GEN_F_DN_SNK, idx, cfg.cost[0], cfg.cost[1])
    return src, snk
