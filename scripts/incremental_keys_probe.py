"""Would keeping the exact solve's keys across augmentations pay (K1c, "key reuse")?

A numpy model of the canonical SSP on a dense layered instance (stress distributions, smaller shape):
per augmentation it compares the keys that really change with two sets that are safe to reset (every
node outside them provably keeps its key):
  closure -- the heads of the saturated path arcs and their descendants along tight arcs;
  hops    -- every node with at least as many hops as the first saturated head.
It also checks the two facts the reuse would rest on: keys never decrease across augmentations, and
every changed key lies in the reset set.
  python scripts/incremental_keys_probe.py S n M [closure|hops]"""
import numpy as np, sys
rng = np.random.default_rng(1)
S, n, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
HB = 20
MODE = sys.argv[4] if len(sys.argv) > 4 else "closure"
INF = np.int64(1) << 62
W = rng.integers(1, 101, (S - 1, n, n)).astype(np.int64)  # W[s][v][u]
src = rng.integers(1, 101, n).astype(np.int64); snk = rng.integers(1, 101, n).astype(np.int64)
cap = rng.integers(1, 21, (S, n)).astype(np.int64)
g = np.zeros((S, n), np.int64); f = np.zeros((S - 1, n, n), np.int64)  # f[s][u][v]
sf = np.zeros(n, np.int64); kf = np.zeros(n, np.int64)
Wk = (W << HB) + 1  # [s][v][u]

def keys():
    kin = np.full((S, n), INF); kout = np.full((S, n), INF); t = INF
    kin[0] = (src << HB) + 1
    for it in range(10000):
        ch = False
        for s in range(S):
            if s > 0:
                cand = (kout[s - 1][None, :] + Wk[s - 1]).min(1)
                m = cand < kin[s]; kin[s][m] = cand[m]; ch |= m.any()
            c2 = np.where(g[s] < cap[s], kin[s] + 1, INF); m = c2 < kout[s]; kout[s][m] = c2[m]; ch |= m.any()
        tc = (kout[S - 1] + (snk << HB) + 1).min()
        if tc < t: t = tc; ch = True
        if t < INF:
            c3 = np.where(kf > 0, t - (snk << HB) + 1, INF); m = c3 < kout[S - 1]; kout[S - 1][m] = c3[m]; ch |= m.any()
        for s in range(S - 1, -1, -1):
            c4 = np.where(g[s] > 0, kout[s] + 1, INF); m = c4 < kin[s]; kin[s][m] = c4[m]; ch |= m.any()
            if s > 0:
                # reverse arcs in[s][v] -> out[s-1][u] where f[s-1][u][v] > 0 : kin[s][v] - W<<HB + 1
                cand = np.where(f[s - 1] > 0, kin[s][None, :] - (W[s - 1].T << HB) + 1, INF).min(1)
                m = cand < kout[s - 1]; kout[s - 1][m] = cand[m]; ch |= m.any()
        kin = np.minimum(kin, INF); kout = np.minimum(kout, INF)
        if not ch: return kin, kout, t, it
    raise RuntimeError

def tight_closure(kin, kout, t, seeds_in, seeds_out, seed_t):
    """descendants of the seeds along tight arcs of the current residual graph (old keys)"""
    Ain = np.zeros((S, n), bool); Aout = np.zeros((S, n), bool); At = seed_t
    for (s, i) in seeds_in: Ain[s, i] = True
    for (s, i) in seeds_out: Aout[s, i] = True
    phases = 0
    while True:
        ch = False; phases += 1
        for s in range(S):
            if s > 0:  # out[s-1][u] -> in[s][v] tight
                T = (kout[s - 1][None, :] + Wk[s - 1] == kin[s][:, None]) & Aout[s - 1][None, :] & (kout[s - 1] < INF)[None, :]
                m = T.any(1) & ~Ain[s]; Ain[s] |= m; ch |= m.any()
            m = Ain[s] & (g[s] < cap[s]) & (kin[s] + 1 == kout[s]) & ~Aout[s]; Aout[s] |= m; ch |= m.any()
        if not At and (Aout[S - 1] & (kout[S - 1] + (snk << HB) + 1 == t)).any(): At = True; ch = True
        if At:
            m = (kf > 0) & (t - (snk << HB) + 1 == kout[S - 1]) & ~Aout[S - 1]; Aout[S - 1] |= m; ch |= m.any()
        for s in range(S - 1, -1, -1):
            m = Aout[s] & (g[s] > 0) & (kout[s] + 1 == kin[s]) & ~Ain[s]; Ain[s] |= m; ch |= m.any()
            if s > 0:
                T = (f[s - 1] > 0) & (kin[s][None, :] - (W[s - 1].T << HB) + 1 == kout[s - 1][:, None]) & Ain[s][None, :]
                m = T.any(1) & ~Aout[s - 1]; Aout[s - 1] |= m; ch |= m.any()
        if not ch: return Ain, Aout, At, phases

F = 0; A = 0; prev = None; stats = []
while F < M:
    kin, kout, t, it = keys()
    if t >= INF: break
    if prev is not None:
        pin, pout, pt, Ain, Aout, At, _ = prev
        chin = (kin != pin); chout = (kout != pout)
        assert (kin >= pin).all() and (kout >= pout).all() and t >= pt
        assert not (chin & ~Ain).any() and not (chout & ~Aout).any() and (t == pt or At)
        lay = np.nonzero(Ain.any(1) | Aout.any(1))[0]
        stats.append((chin.sum(), chout.sum(), Ain.sum(), Aout.sum(), len(lay), it, prev[-1]))
    # trace (lowest index predecessor), path as list of nodes ('in'|'out', s, i)
    path = []; x = ('t', 0, 0); kx = t
    while x[0] != 's':
        path.append(x)
        if x[0] == 't':
            c = np.nonzero((kout[S - 1] + (snk << HB) + 1 == kx))[0]; x = ('out', S - 1, c[0]); kx = kout[S - 1][c[0]]; continue
        typ, s, i = x
        if typ == 'in':
            if s == 0 and (src[i] << HB) + 1 == kx: x = ('s', 0, 0); continue
            if s > 0:
                c = np.nonzero(kout[s - 1] + Wk[s - 1][i] == kx)[0]
                if len(c): x = ('out', s - 1, c[0]); kx = kout[s - 1][c[0]]; continue
            assert g[s][i] > 0 and kout[s][i] + 1 == kx; x = ('out', s, i); kx = kout[s][i]; continue
        if g[s][i] < cap[s][i] and kin[s][i] + 1 == kx: x = ('in', s, i); kx = kin[s][i]; continue
        if s < S - 1:
            c = np.nonzero((f[s][i] > 0) & (kin[s + 1] - (W[s][:, i] << HB) + 1 == kx))[0]
            if len(c): x = ('in', s + 1, c[0]); kx = kin[s + 1][c[0]]; continue
        assert kf[i] > 0 and t - (snk[i] << HB) + 1 == kx; x = ('t', 0, 0); kx = t
    path.append(('s', 0, 0)); path.reverse()
    # residuals / bottleneck
    arcs = list(zip(path[:-1], path[1:])); rc = []
    for a, b in arcs:
        if a[0] == 's' or b[0] == 't': rc.append(M - F if b[0] == 't' or a[0] == 's' else 0)
        elif a[0] == 'in' and b[0] == 'out' and a[1] == b[1]: rc.append(cap[a[1]][a[2]] - g[a[1]][a[2]])
        elif a[0] == 'out' and b[0] == 'in' and a[1] == b[1]: rc.append(g[a[1]][a[2]])
        elif a[0] == 'out' and b[0] == 'in': rc.append(M)
        elif a[0] == 'in' and b[0] == 'out': rc.append(f[b[1]][b[2]][a[2]])
        elif a[0] == 't': rc.append(kf[b[2]])
    d = min(min(rc), M - F)
    seeds_in, seeds_out, seed_t = [], [], False
    for (a, b), r in zip(arcs, rc):
        sat = r == d
        if a[0] == 's': continue
        if b[0] == 't': continue
        if a[0] == 'in' and b[0] == 'out' and a[1] == b[1]: g[a[1]][a[2]] += d
        elif a[0] == 'out' and b[0] == 'in' and a[1] == b[1]: g[a[1]][a[2]] -= d
        elif a[0] == 'out' and b[0] == 'in': f[a[1]][a[2]][b[2]] += d; sat = False
        elif a[0] == 'in' and b[0] == 'out': f[b[1]][b[2]][a[2]] -= d
        elif a[0] == 't': kf[b[2]] -= d
        if sat:
            if b[0] == 'in': seeds_in.append((b[1], b[2]))
            elif b[0] == 'out': seeds_out.append((b[1], b[2]))
    # sink/src arcs
    kf[path[-2][2]] += d if path[-2][0] == 'out' else 0
    sf[path[1][2]] += d
    F += d; A += 1
    if MODE == "hops":
        msk = (1 << HB) - 1
        hmin = min([kin[a, b] & msk for a, b in seeds_in] + [kout[a, b] & msk for a, b in seeds_out])
        Ain, Aout, At, ph = (kin & msk) >= hmin, (kout & msk) >= hmin, True, 0
    else:
        Ain, Aout, At, ph = tight_closure(kin, kout, t, seeds_in, seeds_out, seed_t)
    prev = (kin, kout, t, Ain, Aout, At, ph)
st = np.array(stats)
print(f"S={S} n={n} M={M} A={A} F={F}")
print("changed in/out  median", np.median(st[:, 0]), np.median(st[:, 1]), "mean", st[:, 0].mean(), st[:, 1].mean())
print(MODE, "reset set in/out  median", np.median(st[:, 2]), np.median(st[:, 3]), "mean", st[:, 2].mean(), st[:, 3].mean())
print("layers touched median", np.median(st[:, 4]), "BF sweeps median", np.median(st[:, 5]), "closure sweeps", np.median(st[:, 6]))
print("total nodes", 2 * S * n)
