"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product path (paper_2509_21221_b200/) never does.

ctypes wrapper over oracle/liboracle.so (plain C++, see oracle.h) plus small pure-Python
helpers (brute force over path multisets, digests) that pin the oracle in tests.
"""
from __future__ import annotations

import ctypes
import itertools
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
ABSENT = np.iinfo(np.int32).max
OBJ_SUM, OBJ_MINIMAX = 0, 1
P = ctypes.c_void_p


class OrcInstance(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int32), ("n", ctypes.c_int32), ("max_cap", ctypes.c_int32),
                ("M", ctypes.c_int64), ("cap", P), ("alive", P), ("src", P), ("snk", P), ("link", P)]


class OrcResult(ctypes.Structure):
    _fields_ = [("F", ctypes.c_int64), ("cost", ctypes.c_int64), ("A", ctypes.c_int32),
                ("rounds", ctypes.c_int32), ("F_dec", ctypes.c_int64), ("cost_dec", ctypes.c_int64),
                ("dangling", ctypes.c_int32), ("pre_rounds", ctypes.c_int32), ("digest", ctypes.c_uint64),
                ("step_ns", ctypes.c_int64)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        IP = ctypes.POINTER(OrcInstance)
        L.orc_eq1.argtypes = [ctypes.c_int32] * 3 + [P, P, ctypes.c_int32, P, P, ctypes.c_int64, P, P, P]
        L.orc_ssp.argtypes = [IP, P, P, P, P, P, P, P, P]
        L.orc_ssp_batch.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32] + [P] * 6 + [P, P, P, ctypes.c_int32]
        L.orc_network_simplex.argtypes = [IP, P, P]
        L.orc_warm_reroute.argtypes = [IP, P, P, P, P, IP] + [P] * 7
        L.orc_certify.argtypes = [IP, ctypes.c_int64, ctypes.c_int64, P, P, P, P]
        L.orc_anneal_table.argtypes = [ctypes.c_double, ctypes.c_double, P, P, P, ctypes.c_int64]
        L.orc_rounds_create.restype = P
        L.orc_rounds_create.argtypes = [IP, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.orc_rounds_destroy.argtypes = [P]
        L.orc_rounds_run.argtypes = [P, ctypes.c_int32, P, P, P, P, P]
        L.orc_rounds_apply_churn.argtypes = [P, P, P, ctypes.c_int64]
        L.orc_rounds_export.argtypes = [P] + [P] * 8
        L.orc_rounds_digest.restype = ctypes.c_uint64
        L.orc_rounds_import.argtypes = [P] + [P] * 6 + [ctypes.c_int32, ctypes.c_int64]
        L.orc_mix64.restype = ctypes.c_uint64
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_rng_h.restype = ctypes.c_uint64
        L.orc_rng_h.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
        L.orc_pick.restype = ctypes.c_uint32
        L.orc_pick.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
        L.orc_rounds_digest.argtypes = [P]
        L.orc_rounds_instance.argtypes = [P] + [P] * 5
        L.orc_llama_victim.restype = ctypes.c_int32
        L.orc_llama_victim.argtypes = [P, ctypes.c_uint64, ctypes.c_uint64]
        L.orc_mc_rounds_create.restype = P
        L.orc_mc_rounds_create.argtypes = [IP, ctypes.c_int32, P, P, P, ctypes.c_uint64, ctypes.c_int64,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32]
        L.orc_mc_rounds_destroy.argtypes = [P]
        L.orc_mc_rounds_run.argtypes = [P, ctypes.c_int32, P, P, P, P, P]
        L.orc_mc_rounds_export.argtypes = [P] + [P] * 9
        L.orc_mc_rounds_import.argtypes = [P] + [P] * 7 + [ctypes.c_int32, ctypes.c_int64]
        L.orc_mc_rounds_digest.restype = ctypes.c_uint64
        L.orc_mc_rounds_digest.argtypes = [P]
        L.orc_pipeline_batch.argtypes = ([ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32] + [P] * 6
                                         + [ctypes.c_int32, P, P, ctypes.c_int64, P, ctypes.c_uint64, ctypes.c_int64,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P])
        _LIB = L
    return _LIB


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class Instance:
    """One instance, host numpy arrays (layouts of oracle.h / include/gwtf.h)."""
    S: int
    n: int
    max_cap: int
    M: int
    cap: np.ndarray            # [S][n] i32
    src: np.ndarray            # [n] i32
    snk: np.ndarray            # [n] i32
    link: np.ndarray           # [S-1][n][n] i32, dest-major
    alive: np.ndarray = None   # [S][n] u8

    def __post_init__(self):
        self.cap = np.ascontiguousarray(self.cap, np.int32)
        self.src = np.ascontiguousarray(self.src, np.int32)
        self.snk = np.ascontiguousarray(self.snk, np.int32)
        self.link = np.ascontiguousarray(np.asarray(self.link, np.int32).reshape(max(self.S - 1, 0), self.n, self.n))
        if self.alive is None:
            self.alive = np.ones((self.S, self.n), np.uint8)
        self.alive = np.ascontiguousarray(self.alive, np.uint8)

    def c(self) -> OrcInstance:
        o = OrcInstance()
        o.S, o.n, o.max_cap, o.M = self.S, self.n, self.max_cap, self.M
        o.cap, o.alive, o.src, o.snk = _ptr(self.cap), _ptr(self.alive), _ptr(self.src), _ptr(self.snk)
        o.link = _ptr(self.link) if self.link.size else None
        return o

    def cap_eff(self):
        return np.where(self.alive != 0, self.cap, 0)


def instance_from_batch(bt, b: int, link=None, src=None, snk=None) -> Instance:
    """Instance b of a generated host batch (gen.Batch); Eq. 1 batches pass link/src/snk from eq1()."""
    cfg = bt.cfg
    return Instance(cfg.S, cfg.n, cfg.max_cap, int(bt.supply[b]), bt.cap[b],
                    bt.src[b] if src is None else src, bt.snk[b] if snk is None else snk,
                    bt.link[b] if link is None else link, bt.alive[b])


def eq1(S, n, L, comp, loc, dloc, lat, bw, size_kbit):
    """Oracle Eq. 1 in integer half-units -> (src[n], snk[n], link[S-1][n][n])."""
    src = np.zeros(n, np.int32)
    snk = np.zeros(n, np.int32)
    link = np.zeros((max(S - 1, 0), n, n), np.int32)
    comp = np.ascontiguousarray(comp, np.int32)
    loc = np.ascontiguousarray(loc, np.int32)
    lat = np.ascontiguousarray(lat, np.int32)
    bw = np.ascontiguousarray(bw, np.int32)
    lib().orc_eq1(S, n, L, _ptr(comp), _ptr(loc), int(dloc), _ptr(lat), _ptr(bw), int(size_kbit),
                  _ptr(src), _ptr(snk), _ptr(link) if link.size else None)
    return src, snk, link


def eq1_batch(bt):
    """Oracle Eq. 1 for every instance of a host gen.Batch -> (src[B][n], snk[B][n], link[B][S-1][n][n])."""
    cfg = bt.cfg
    B = bt.B
    src = np.zeros((B, cfg.n), np.int32)
    snk = np.zeros((B, cfg.n), np.int32)
    link = np.zeros((B, max(cfg.S - 1, 0), cfg.n, cfg.n), np.int32)
    for b in range(B):
        src[b], snk[b], link[b] = eq1(cfg.S, cfg.n, cfg.L, bt.comp[b], bt.loc[b], bt.dloc[b], bt.lat[b], bt.bw[b],
                                      cfg.size_kbit)
    return src, snk, link


@dataclass
class SSPResult:
    F: int
    cost: int
    A: int
    node_flow: np.ndarray
    src_flow: np.ndarray
    snk_flow: np.ndarray
    arc_flow: np.ndarray
    curve: np.ndarray = None


def ssp(I: Instance, curve: bool = False) -> SSPResult:
    """Canonical SSP."""
    F = ctypes.c_int64()
    cost = ctypes.c_int64()
    A = ctypes.c_int32()
    nf = np.zeros((I.S, I.n), np.int32)
    sf = np.zeros(I.n, np.int32)
    kf = np.zeros(I.n, np.int32)
    af = np.zeros((max(I.S - 1, 0), I.n, I.n), np.int32)
    cv = np.zeros(I.M + 1, np.int64) if curve else None
    c = I.c()
    rc = lib().orc_ssp(ctypes.byref(c), ctypes.byref(F), ctypes.byref(cost), ctypes.byref(A), _ptr(nf), _ptr(sf),
                       _ptr(kf), _ptr(af) if af.size else None, _ptr(cv))
    if rc != 0:
        raise RuntimeError(f"oracle SSP internal check failed rc={rc}")
    r = SSPResult(F.value, cost.value, A.value, nf, sf, kf, af)
    if curve:
        r.curve = cv[: F.value + 1]
    return r


def network_simplex(I: Instance):
    F = ctypes.c_int64()
    cost = ctypes.c_int64()
    c = I.c()
    rc = lib().orc_network_simplex(ctypes.byref(c), ctypes.byref(F), ctypes.byref(cost))
    if rc != 0:
        raise RuntimeError(f"network simplex failed rc={rc}")
    return F.value, cost.value


def warm_reroute(I_old: Instance, base: SSPResult, I_new: Instance):
    """Warm-start rerouting after churn: keep the
    pre-churn assignment `base` of I_old, strip what I_new cannot carry, cancel negative
    residual cycles, resume SSP.  -> (SSPResult with the new assignment, stats dict)."""
    F = ctypes.c_int64()
    cost = ctypes.c_int64()
    st = np.zeros(3, np.int64)
    nf = np.zeros((I_new.S, I_new.n), np.int32)
    sf = np.zeros(I_new.n, np.int32)
    kf = np.zeros(I_new.n, np.int32)
    af = np.zeros((max(I_new.S - 1, 0), I_new.n, I_new.n), np.int32)
    arrs = [np.ascontiguousarray(a, np.int32) for a in (base.node_flow, base.src_flow, base.snk_flow, base.arc_flow)]
    co, cn = I_old.c(), I_new.c()
    rc = lib().orc_warm_reroute(ctypes.byref(co), *[_ptr(a) if a.size else None for a in arrs], ctypes.byref(cn),
                                ctypes.byref(F), ctypes.byref(cost), _ptr(st), _ptr(nf), _ptr(sf), _ptr(kf),
                                _ptr(af) if af.size else None)
    if rc != 0:
        raise RuntimeError(f"oracle warm reroute failed rc={rc}")
    r = SSPResult(F.value, cost.value, int(st[2]), nf, sf, kf, af)
    return r, {"stripped": int(st[0]), "cycles": int(st[1]), "augment": int(st[2])}


def certify(I: Instance, F, cost, node_flow, src_flow, snk_flow, arc_flow) -> int:
    c = I.c()
    arrs = [np.ascontiguousarray(a, np.int32) for a in (node_flow, src_flow, snk_flow, arc_flow)]
    return lib().orc_certify(ctypes.byref(c), int(F), int(cost), *[_ptr(a) if a.size else None for a in arrs])


def anneal_table(T0: float, alpha: float):
    w = ctypes.c_int32()
    K = ctypes.c_int32()
    rc = lib().orc_anneal_table(T0, alpha, ctypes.byref(w), ctypes.byref(K), None, 0)
    if rc:
        raise ValueError(f"anneal table rc={rc}")
    t = np.zeros((K.value + 1) * w.value, np.uint32)
    lib().orc_anneal_table(T0, alpha, ctypes.byref(w), ctypes.byref(K), _ptr(t), t.size)
    return t.reshape(K.value + 1, w.value), w.value, K.value


class Rounds:
    """Synchronous decentralized rounds of one instance."""

    def __init__(self, I: Instance, seed=0, inst_id=0, T0=1.7, alpha=0.95, objective=OBJ_SUM, W=5, deny_after=3):
        self.I = I
        c = I.c()
        self.h = lib().orc_rounds_create(ctypes.byref(c), seed, inst_id, T0, alpha, objective, W, deny_after)
        if not self.h:
            raise ValueError("orc_rounds_create rejected the parameters")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_rounds_destroy(self.h)
            self.h = None

    def run(self, max_rounds, digests=False):
        rr = ctypes.c_int32()
        F = ctypes.c_int64()
        C = ctypes.c_int64()
        dg = ctypes.c_int32()
        d = np.zeros(max(max_rounds, 1), np.uint64) if digests else None
        lib().orc_rounds_run(self.h, max_rounds, ctypes.byref(rr), ctypes.byref(F), ctypes.byref(C),
                             ctypes.byref(dg), _ptr(d))
        out = dict(rounds=rr.value, F_dec=F.value, cost_dec=C.value, dangling=dg.value)
        if digests:
            out["digests"] = d[: rr.value]
        return out

    def apply_churn(self, alive_new=None, updates=None):
        a = None if alive_new is None else np.ascontiguousarray(alive_new, np.uint8)
        u = None if updates is None else np.ascontiguousarray(updates, np.int32).reshape(-1, 5)
        lib().orc_rounds_apply_churn(self.h, _ptr(a), _ptr(u) if u is not None and u.size else None,
                                     0 if u is None else u.shape[0])

    def export(self):
        I = self.I
        up = np.zeros((I.S, I.n, I.max_cap), np.int32)
        dn = np.zeros_like(up)
        sd = np.zeros(I.M, np.int32)
        su = np.zeros(I.M, np.int32)
        k = np.zeros((I.S, I.n), np.int32)
        dw = np.zeros_like(k)
        q = ctypes.c_int32()
        r = ctypes.c_int64()
        lib().orc_rounds_export(self.h, _ptr(up), _ptr(dn), _ptr(sd), _ptr(su), _ptr(k), _ptr(dw), ctypes.byref(q),
                                ctypes.byref(r))
        return dict(up=up, down=dn, src_down=sd, snk_up=su, kacc=k, deny=dw, quiet=q.value, round=r.value)

    def import_state(self, st: dict):
        """Install a round state in export()'s layouts (checkpoint / resume); raises if it is not a
        valid pairing."""
        c = lambda k: np.ascontiguousarray(np.asarray(st[k], np.int32).reshape(-1))  # noqa: E731
        arrs = [c("up"), c("down"), c("src_down"), c("snk_up"), c("kacc"), c("deny")]
        rc = lib().orc_rounds_import(self.h, *[_ptr(a) for a in arrs], int(st.get("quiet", 0)), int(st.get("round", 0)))
        if rc != 0:
            raise ValueError("orc_rounds_import: not a valid pairing state")

    def digest(self) -> int:
        return int(lib().orc_rounds_digest(self.h))

    def instance(self) -> Instance:
        I = self.I
        ce = np.zeros((I.S, I.n), np.int32)
        al = np.zeros((I.S, I.n), np.uint8)
        src = np.zeros(I.n, np.int32)
        snk = np.zeros(I.n, np.int32)
        link = np.zeros((max(I.S - 1, 0), I.n, I.n), np.int32)
        lib().orc_rounds_instance(self.h, _ptr(ce), _ptr(al), _ptr(src), _ptr(snk), _ptr(link) if link.size else None)
        return Instance(I.S, I.n, I.max_cap, I.M, I.cap.copy(), src, snk, link, al)

    def llama_victim(self, draw_stage: int, draw_pick: int) -> int:
        return int(lib().orc_llama_victim(self.h, draw_stage, draw_pick))


def pipeline_batch(cfg, cap, alive, src, snk, link, supply, churn_kind=0, alive_new=None, updates=None,
                   victim_draws=None, seed=0, inst_base=0, T0=1.7, alpha=0.95, objective=OBJ_SUM, W=5, deny_after=3,
                   max_rounds=None, threads=None):
    """Whole bench-step workload per instance (oracle.h orc_pipeline_batch)."""
    B = cap.shape[0]
    out = (OrcResult * B)()
    max_rounds = cfg.max_rounds if max_rounds is None else max_rounds
    threads = threads or os.cpu_count() or 1
    arrs = [np.ascontiguousarray(a) for a in (cap, alive, src, snk, link, supply)]
    un = None if updates is None else np.ascontiguousarray(updates, np.int32)
    an = None if alive_new is None else np.ascontiguousarray(alive_new, np.uint8)
    vd = None if victim_draws is None else np.ascontiguousarray(victim_draws, np.uint64)
    rc = lib().orc_pipeline_batch(B, cfg.S, cfg.n, cfg.max_cap, *[_ptr(a) for a in arrs], churn_kind, _ptr(an),
                                  _ptr(un) if un is not None and un.size else None, 0 if un is None else un.shape[0],
                                  _ptr(vd), seed, inst_base, T0, alpha, objective, W, deny_after, max_rounds, threads,
                                  out)
    if rc != 0:
        raise RuntimeError(f"oracle pipeline failed rc={rc}")
    dt = {"digest": np.uint64, "F": np.int64, "cost": np.int64, "F_dec": np.int64, "cost_dec": np.int64,
          "step_ns": np.int64}
    return {k: np.array([getattr(out[b], k) for b in range(B)], dtype=dt.get(k, np.int32))
            for k, _ in OrcResult._fields_}


# ----------------------------------------------------------------------------------------
# Pure-Python pins (independent of liboracle)
# ----------------------------------------------------------------------------------------
def brute_force(I: Instance):
    """Max flow value and min cost by exhaustive enumeration of path multisets (SPEC S:212,
    SURVEY C7).  Every unit of flow follows a path D -> (0,i0) -> ... -> (S-1,i_{S-1}) -> D;
    a flow is a multiset of such paths within node capacities.  Tiny instances only."""
    S, n = I.S, I.n
    ce = I.cap_eff()
    paths = []
    for combo in itertools.product(range(n), repeat=S):
        c = int(I.src[combo[0]]) if I.src[combo[0]] != ABSENT else None
        if c is None or ce[0, combo[0]] == 0:
            continue
        ok = True
        for s in range(S - 1):
            w = I.link[s, combo[s + 1], combo[s]]
            if w == ABSENT or ce[s + 1, combo[s + 1]] == 0:
                ok = False
                break
            c += int(w)
        if not ok or I.snk[combo[-1]] == ABSENT:
            continue
        paths.append((combo, c + int(I.snk[combo[-1]])))
    best = [0, 0]
    rem = ce.astype(np.int64).copy()

    def rec(k, F, cost):
        if F > best[0] or (F == best[0] and cost < best[1]):
            best[0], best[1] = F, cost
        if k == len(paths) or F == I.M:
            return
        combo, c = paths[k]
        m = min([int(rem[s, combo[s]]) for s in range(S)] + [I.M - F])
        for t in range(m, -1, -1):
            for s in range(S):
                rem[s, combo[s]] -= t
            rec(k + 1, F + t, cost + t * c)
            for s in range(S):
                rem[s, combo[s]] += t

    rec(0, 0, 0)
    return best[0], best[1]


def mix64(z: int) -> int:
    m = (1 << 64) - 1
    z &= m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def digest_state(st: dict, S: int, n: int, MC: int, M: int) -> int:
    """Python re-statement of the round-state digest of DESIGN.md 2.3 (order-independent sum)."""
    m = (1 << 64) - 1
    up = st["up"].reshape(-1)
    dn = st["down"].reshape(-1)
    vals = []
    for p in range(up.size):
        u, d = int(up[p]), int(dn[p])
        state = (2 if u != -1 else 0) | (1 if d != -1 else 0)
        eu = 0 if u == -1 else (1 + u if u >= 0 else (1 << 40) + (-2 - u))
        ed = 0 if d == -1 else (1 + d if d >= 0 else (1 << 41) + (-2 - d))
        vals += [state, eu, ed]
    vals += [0 if int(x) == -1 else 1 + int(x) for x in st["src_down"]]
    vals += [0 if int(x) == -1 else 1 + int(x) for x in st["snk_up"]]
    for g in range(S * n):
        vals += [int(st["kacc"].reshape(-1)[g]) & 0xFFFFFFFF, int(st["deny"].reshape(-1)[g]) & 0xFFFFFFFF]
    vals.append(int(st["quiet"]) & 0xFFFFFFFF)
    return sum(mix64(mix64(pos) ^ v) for pos, v in enumerate(vals)) & m


# ---- node addition ----

def placed_instance(I: Instance, cand: dict, assign) -> Instance:
    """The base instance with candidate assign[s] joined to stage s as client n (assign[s] < 0:
    no candidate, a zero-capacity client).  Costs as generated (gen.generate_candidates):
    cin[c][s][u] = d((s-1,u) -> c@s), cin[c][0][0] = d(D -> c@0); cout[c][s][v] = d(c@s -> (s+1,v)),
    cout[c][S-1][0] = d(c@S-1 -> D); cc[c1][c2] = d(c1@s -> c2@s+1)."""
    S, n = I.S, I.n
    n1 = n + 1
    cap = np.zeros((S, n1), np.int32)
    cap[:, :n] = I.cap_eff()
    src = np.full(n1, ABSENT, np.int32)
    snk = np.full(n1, ABSENT, np.int32)
    src[:n], snk[:n] = I.src, I.snk
    link = np.full((max(S - 1, 0), n1, n1), ABSENT, np.int32)
    if S > 1:
        link[:, :n, :n] = I.link
    for s in range(S):
        c = assign[s]
        if c < 0:
            continue
        cap[s, n] = cand["cap"][c]
        if s == 0:
            src[n] = cand["cin"][c][0][0]
        else:
            link[s - 1, n, :n] = cand["cin"][c][s]          # (s-1,u) -> c@s
        if s == S - 1:
            snk[n] = cand["cout"][c][S - 1][0]
        else:
            link[s, :n, n] = cand["cout"][c][s]             # c@s -> (s+1,v)
            if assign[s + 1] >= 0:
                link[s, n, n] = cand["cc"][c][assign[s + 1]]
    return Instance(S, n1, max(I.max_cap, int(cand["cap"].max(initial=0))), I.M, cap, src, snk, link)


def optimal_addition(I: Instance, cand: dict):
    """The optimal placement of S candidates, one per stage, by exhaustive enumeration
    ("for each combination of S candidate nodes added to each of the S stages"):
    every permutation in lexicographic order (itertools.permutations of range(S)), each solved
    by the oracle SSP.  Best = max F, then min cost, then the first (lexicographic) placement
    (SPEC.md:193).  Returns (best index, its permutation, F[], cost[])."""
    perms = list(itertools.permutations(range(I.S)))
    F = np.zeros(len(perms), np.int64)
    C = np.zeros(len(perms), np.int64)
    for k, p in enumerate(perms):
        r = ssp(placed_instance(I, cand, p))
        F[k], C[k] = r.F, r.cost
    best = 0
    for k in range(1, len(perms)):
        if F[k] > F[best] or (F[k] == F[best] and C[k] < C[best]):
            best = k
    return best, perms[best], F, C


def improvement(cost_now: float, cost_after: float) -> float:
    """(cost_now - cost_after) / cost_now."""
    return (cost_now - cost_after) / cost_now


# ---- SWARM-style greedy baseline ----

def greedy_route(I: Instance):
    """Microbatches routed one at a time from the data node D: each hop goes to the alive
    next-stage client with spare capacity and a link, minimum cost first, lowest index on ties
    (SPEC.md:202); a microbatch without a successor or sink arc is not routed, its reservations
    are released and routing stops (every later microbatch would retrace it).  Returns
    (routed microbatches, total cost, per-microbatch paths)."""
    rem = I.cap_eff().astype(np.int64).copy()
    F, cost, paths = 0, 0, []
    for _ in range(I.M):
        path, c, u = [], 0, None
        for s in range(I.S):
            best = None
            for v in range(I.n):
                d = int(I.src[v]) if s == 0 else int(I.link[s - 1, v, u])
                if d == ABSENT or rem[s, v] <= 0:
                    continue
                if best is None or d < best[0]:
                    best = (d, v)
            if best is None:
                break
            rem[s, best[1]] -= 1
            path.append(best[1])
            c += best[0]
            u = best[1]
        if len(path) < I.S or int(I.snk[u]) == ABSENT:
            for s, v in enumerate(path):
                rem[s, v] += 1
            break
        F += 1
        cost += c + int(I.snk[u])
        paths.append(path)
    return F, cost, paths


# ---- multi-data-node flows ----

def multi_source_ssp_unit(I: Instance, srcs, snks, supplies):
    """Round-robin by microbatch (the other reading of SPEC.md:215's "round-robin order"): the data
    nodes take turns, each turn routing one microbatch of one data node by a single-commodity
    canonical SSP with supply 1 on the node capacities left so far; a data node that cannot route
    drops out.  Returns per data node (F, cost, node_flow)."""
    K = len(srcs)
    cap = I.cap_eff().astype(np.int32).copy()
    F = [0] * K
    C = [0] * K
    nf = [np.zeros((I.S, I.n), np.int32) for _ in range(K)]
    active = [int(M) > 0 for M in supplies]
    while any(active):
        for k in range(K):
            if not active[k]:
                continue
            r = ssp(Instance(I.S, I.n, I.max_cap, 1, cap, srcs[k], snks[k], I.link))
            if r.F == 0:
                active[k] = False
                continue
            F[k] += 1
            C[k] += r.cost
            nf[k] += r.node_flow
            cap = cap - r.node_flow
            if F[k] >= int(supplies[k]):
                active[k] = False
    return [(F[k], C[k], nf[k]) for k in range(K)]


def multi_source_ssp(I: Instance, srcs, snks, supplies):
    """One single-commodity canonical SSP per data node, in data-node order, each on the node
    capacities the earlier data nodes left ("one single-commodity problem per data node
    over residual capacities in round-robin order" -- a heuristic decomposition; the paper does not
    compare settings 5-6 with an optimum).  Returns per data node (F, cost, node_flow)."""
    cap = I.cap_eff().astype(np.int32).copy()
    out = []
    for src, snk, M in zip(srcs, snks, supplies):
        Ik = Instance(I.S, I.n, I.max_cap, int(M), cap, src, snk, I.link)
        r = ssp(Ik)
        out.append((r.F, r.cost, r.node_flow.copy()))
        cap = cap - r.node_flow
    return out


# ------------------------------------------------------------------ the R4 draws
def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & (2**64 - 1)))


def rng_h(seed: int, inst: int, rnd: int, gid: int, stream: int) -> int:
    return int(lib().orc_rng_h(seed & (2**64 - 1), inst, rnd, gid, stream))


def pick(x: int, m: int) -> int:
    return int(lib().orc_pick(x & (2**64 - 1), m))


class McRounds:
    """Multi-data-node synchronous rounds (MC-SYNC): K data nodes with
    their own src / snk costs ([K][n]) and supplies ([K]) on I's relays and links."""

    def __init__(self, I: Instance, srcs, snks, supplies, seed=0, inst_id=0, T0=1.7, alpha=0.95,
                 objective=OBJ_SUM, W=5, deny_after=3):
        self.I = I
        self.K = len(supplies)
        self.src = np.ascontiguousarray(np.asarray(srcs, np.int32).reshape(self.K, I.n))
        self.snk = np.ascontiguousarray(np.asarray(snks, np.int32).reshape(self.K, I.n))
        self.M = np.ascontiguousarray(np.asarray(supplies, np.int64).reshape(self.K))
        self.Mmax = max(1, int(self.M.max()))
        c = I.c()
        self.h = lib().orc_mc_rounds_create(ctypes.byref(c), self.K, _ptr(self.src), _ptr(self.snk), _ptr(self.M),
                                            seed, inst_id, T0, alpha, objective, W, deny_after)
        if not self.h:
            raise ValueError("orc_mc_rounds_create rejected the parameters")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_mc_rounds_destroy(self.h)
            self.h = None

    def run(self, max_rounds, digests=False):
        rr = ctypes.c_int32()
        F = np.zeros(self.K, np.int64)
        C = np.zeros(self.K, np.int64)
        dg = ctypes.c_int32()
        d = np.zeros(max(max_rounds, 1), np.uint64) if digests else None
        lib().orc_mc_rounds_run(self.h, max_rounds, ctypes.byref(rr), _ptr(F), _ptr(C), ctypes.byref(dg), _ptr(d))
        out = dict(rounds=rr.value, F_dec=F, cost_dec=C, dangling=dg.value)
        if digests:
            out["digests"] = d[: rr.value]
        return out

    def export(self):
        I = self.I
        up = np.zeros((I.S, I.n, I.max_cap), np.int32)
        dn = np.zeros_like(up)
        tg = np.zeros_like(up)
        sd = np.zeros((self.K, self.Mmax), np.int32)
        su = np.zeros_like(sd)
        k = np.zeros((I.S, I.n), np.int32)
        dw = np.zeros_like(k)
        q = ctypes.c_int32()
        r = ctypes.c_int64()
        lib().orc_mc_rounds_export(self.h, _ptr(up), _ptr(dn), _ptr(tg), _ptr(sd), _ptr(su), _ptr(k), _ptr(dw),
                                   ctypes.byref(q), ctypes.byref(r))
        return dict(up=up, down=dn, tag=tg, src_down=sd, snk_up=su, kacc=k, deny=dw, quiet=q.value, round=r.value)

    def import_state(self, st: dict):
        """Install a state in export()'s layouts (ValueError unless a valid tagged pairing)."""
        c = lambda k: None if st.get(k) is None else np.ascontiguousarray(np.asarray(st[k], np.int32).reshape(-1))  # noqa: E731
        arrs = [c("up"), c("down"), c("tag"), c("src_down"), c("snk_up"), c("kacc"), c("deny")]
        rc = lib().orc_mc_rounds_import(self.h, *[_ptr(a) for a in arrs], int(st.get("quiet", 0)), int(st.get("round", 0)))
        if rc != 0:
            raise ValueError("orc_mc_rounds_import: not a valid tagged pairing")

    def digest(self) -> int:
        return int(lib().orc_mc_rounds_digest(self.h))

