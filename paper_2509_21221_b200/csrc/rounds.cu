// Decentralized neighbour-exchange flow rounds, synchronous semantics.
//
// PAPER.md:241-263 (Request Flow / Request Change / Request Redirect, simulated annealing,
// steady state) and :269 (DENY).  One team of TPI threads per instance, persistent over an
// atomic instance queue; every phase is relay-parallel and phases are separated by team
// barriers, so each phase reads the snapshot the definition names:
//   R0a self-pairing (round-start costs) | R0 cost-to-sink back to front + advertisements |
//   R1 one Request Flow per node | R2 grants in requester order | R3 commit |
//   R4 Change / Redirect / DENY proposals on the post-R3 state (counter RNG, integer
//   annealing thresholds) | R5 deterministic reservations (64-bit atomicMin, order free) |
//   R6 commit winners | R7 quiet counter, optional state digest.
// Round state lives in global memory (L1/L2 resident for the team); reservation minima are
// read with ld.global.cg because they are produced by L2 atomics.
#include "common.cuh"

namespace gwtf {

namespace {

constexpr int64_t INF = INT64_MAX;
constexpr uint64_t RES_NONE = ~0ull;
enum { K_NONE = 0, K_CHANGE = 1, K_REDIRECT = 2, K_DENY = 3 };

__device__ __forceinline__ uint64_t mix(uint64_t z) {  // splitmix64 finalizer
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t pick(uint64_t x, uint32_t m) {
  return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32);
}
__device__ __forceinline__ int64_t sadd(int64_t a, int64_t b) { return (a == INF || b == INF) ? INF : a + b; }

struct Inst {
  const Problem* P;
  int S, n, ld, MC, Sn;
  int64_t M;
  int inst;
  int32_t *up, *down, *src_down, *snk_up, *kacc, *deny;
  int64_t *scost, *adv_cost;
  int32_t *adv_slot, *req_slot, *req_target, *prop;
  uint64_t *pkey, *res;
  int64_t* ptouch;
  const int32_t *tile, *src, *snk, *cap;
  const uint8_t* alive;

  __device__ int capE(int v) const { return alive[v] ? cap[v] : 0; }
  __device__ int st(int p) const { return (up[p] != kNone ? 2 : 0) | (down[p] != kNone ? 1 : 0); }
  // d(a, b) between nodes; -1 = data node D.  Missing / absent = INF.
  __device__ int64_t d(int a, int b) const {
    int32_t c = kAbsent;
    if (a < 0) {
      if (b >= 0 && b < n) c = src[b];
    } else if (b < 0) {
      if (a / n == S - 1) c = snk[a % n];
    } else {
      const int sa = a / n;
      if (b / n == sa + 1) c = tile[((size_t)sa * n + (b % n)) * ld + (a % n)];
    }
    return c == kAbsent ? INF : (int64_t)c;
  }
  __device__ int64_t res_up(int32_t p) const { return p >= 0 ? p : (int64_t)Sn * MC + (-2 - p); }
  __device__ int64_t res_dn(int32_t p) const { return p >= 0 ? p : (int64_t)Sn * MC + P->Mmax + (-2 - p); }
  __device__ void set_up_of(int32_t p, int32_t v) { if (p >= 0) up[p] = v; else snk_up[-2 - p] = v; }
  __device__ void set_down_of(int32_t p, int32_t v) { if (p >= 0) down[p] = v; else src_down[-2 - p] = v; }
  __device__ uint64_t h(uint64_t round, int gid, int stream) const {
    return mix(mix(mix(mix(P->seed) ^ (uint64_t)(P->inst_base + inst)) ^ round) ^ ((uint64_t)gid * 4 + stream));
  }
};

struct SlotScan {
  int first_in, first_free, npaired;
  bool has_out;
};
__device__ __forceinline__ SlotScan scan_slots(const Inst& I, int v) {
  SlotScan r{-1, -1, 0, false};
  const int c = I.capE(v);
  for (int j = 0; j < c; ++j) {
    const int p = v * I.MC + j, t = I.st(p);
    if (t == 2 && r.first_in < 0) r.first_in = p;
    if (t == 0 && r.first_free < 0) r.first_free = p;
    if (t == 1) r.has_out = true;
    if (t == 3) r.npaired++;
  }
  return r;
}
__device__ __forceinline__ int nth_paired(const Inst& I, int v, int q) {
  const int c = I.capE(v);
  for (int j = 0; j < c; ++j) {
    const int p = v * I.MC + j;
    if (I.st(p) == 3) { if (q == 0) return p; --q; }
  }
  return -1;
}

template <int TPI>
__device__ void compute_costs(const Team<TPI>& T, const Inst& I) {
  for (int s = I.S - 1; s >= 0; --s) {
    for (int t = T.tid; t < I.n * I.MC; t += TPI) {
      const int v = s * I.n + t / I.MC, j = t % I.MC, p = v * I.MC + j;
      int64_t c = INF;
      if (j < I.capE(v)) {
        const int32_t dn = I.down[p];
        if (dn == kNone) c = INF;
        else if (dn <= -2) c = I.d(v, -1);
        else c = sadd(I.d(v, dn / I.MC), I.scost[dn]);
      }
      I.scost[p] = c;
    }
    T.sync();
  }
}

__device__ uint64_t digest_elem(uint64_t pos, uint64_t val) { return mix(mix(pos) ^ val); }

template <int TPI>
__global__ void __launch_bounds__(256) rounds_kernel(const Problem P, const RoundsOut o) {
  __shared__ uint64_t sh_u64[8][2];
  __shared__ int sh_i32[8][4];
  __shared__ int sh_inst[8];
  const Team<TPI> T{(int)(threadIdx.x % TPI), (int)(threadIdx.x / TPI)};
  const int lane = threadIdx.x & 31;
  const int S = P.S, n = P.n, MC = P.MC, Sn = S * n;
  const int nres = Sn * MC + 2 * (int)P.Mmax;

  for (;;) {
    if (T.tid == 0) sh_inst[T.id] = atomicAdd(&P.counters[1], 1);
    T.sync();
    const int b = sh_inst[T.id];
    if (b >= P.B) break;
    Inst I;
    I.P = &P; I.S = S; I.n = n; I.ld = P.ld; I.MC = MC; I.Sn = Sn; I.inst = b;
    I.M = P.supply[b];
    I.up = P.up + (size_t)b * Sn * MC;
    I.down = P.down + (size_t)b * Sn * MC;
    I.src_down = P.src_down + (size_t)b * P.Mmax;
    I.snk_up = P.snk_up + (size_t)b * P.Mmax;
    I.kacc = P.kacc + (size_t)b * Sn;
    I.deny = P.deny + (size_t)b * Sn;
    I.scost = P.scost + (size_t)b * Sn * MC;
    I.adv_cost = P.adv_cost + (size_t)b * Sn;
    I.adv_slot = P.adv_slot + (size_t)b * Sn;
    I.req_slot = P.req_slot + (size_t)b * (Sn + 1);
    I.req_target = P.req_target + (size_t)b * (Sn + 1);
    I.prop = P.prop + (size_t)b * Sn * 6;
    I.pkey = P.prop_key + (size_t)b * Sn;
    I.ptouch = P.prop_touch + (size_t)b * Sn * 4;
    I.res = P.res + (size_t)b * nres;
    I.tile = P.tile + (size_t)b * (S - 1) * n * P.ld;
    I.src = P.src + (size_t)b * n;
    I.snk = P.snk + (size_t)b * n;
    I.cap = P.cap + (size_t)b * Sn;
    I.alive = P.alive + (size_t)b * Sn;
    const int M = (int)I.M;

    for (int k = T.tid; k < nres; k += TPI) __stcg(&I.res[k], RES_NONE);
    int quiet = 0;  // quiet = 0 at the start of every call (DESIGN.md 2.3 R7)
    uint64_t round = (uint64_t)P.round[b];
    int r = 0;
    T.sync();
    while (r < o.max_rounds) {
      int changed = 0;
      // ---------- R0a self-pairing (costs of the round-start state) ----------
      int cand = 0;
      for (int v = T.tid; v < Sn; v += TPI) {
        if (!I.alive[v]) continue;
        const SlotScan sc = scan_slots(I, v);
        cand |= (sc.first_in >= 0 && sc.has_out);
      }
      if (T.sync_or(cand)) {
        compute_costs(T, I);
        for (int v = T.tid; v < Sn; v += TPI) {
          if (!I.alive[v]) continue;
          int x = -1, oo = -1;
          for (int j = 0; j < I.capE(v); ++j) {
            const int p = v * MC + j, t = I.st(p);
            if (t == 2 && x < 0) x = p;
            if (t == 1 && (oo < 0 || I.scost[p] < I.scost[oo])) oo = p;
          }
          if (x < 0 || oo < 0) continue;
          const int32_t cdn = I.down[oo];
          I.down[x] = cdn;
          I.set_up_of(cdn, x);
          I.down[oo] = kNone;
          changed = 1;
        }
        T.sync();
      }
      // ---------- R0 cost to sink + advertisements ----------
      compute_costs(T, I);
      for (int v = T.tid; v < Sn; v += TPI) {
        int64_t bc = INF;
        int bj = -1;
        if (I.alive[v]) {
          for (int j = 0; j < I.capE(v); ++j) {
            const int p = v * MC + j;
            if (I.st(p) == 1 && (bj < 0 || I.scost[p] < bc)) { bc = I.scost[p]; bj = j; }
          }
        }
        I.adv_cost[v] = bc;
        I.adv_slot[v] = bj;
      }
      // data node: lowest unpaired SRC slot, any free SNK slot
      if (T.tid == 0) { sh_i32[T.id][0] = INT_MAX; sh_i32[T.id][1] = 0; }
      T.sync();
      {
        int fs = INT_MAX, anyfree = 0;
        for (int k = T.tid; k < M; k += TPI) {
          if (I.src_down[k] == kNone && k < fs) fs = k;
          anyfree |= I.snk_up[k] == kNone;
        }
        if (fs != INT_MAX) atomicMin(&sh_i32[T.id][0], fs);
        if (anyfree) atomicOr(&sh_i32[T.id][1], 1);
      }
      T.sync();
      const int d_rslot = sh_i32[T.id][0];
      const int dsink_free = sh_i32[T.id][1];
      // ---------- R1 requests (one per node) ----------
      for (int rr = T.tid; rr <= Sn; rr += TPI) {
        int32_t rs = kNone, tg = -2;
        if (rr == Sn) {  // the data node
          if (d_rslot != INT_MAX) {
            int64_t bc = INF;
            for (int j = 0; j < n; ++j) {
              const int64_t dj = I.d(-1, j);
              if (!I.alive[j] || dj == INF || I.adv_cost[j] == INF) continue;
              if (dj + I.adv_cost[j] < bc) { bc = dj + I.adv_cost[j]; tg = j; }
            }
            if (tg != -2) rs = -2 - d_rslot;
          }
        } else if (I.alive[rr]) {
          const SlotScan sc = scan_slots(I, rr);
          int32_t x = kNone;
          if (sc.first_in >= 0) x = sc.first_in;
          else if (!sc.has_out && sc.first_free >= 0) x = sc.first_free;
          if (x != kNone) {
            const int s = rr / n;
            if (s == S - 1) {
              if (I.d(rr, -1) != INF && dsink_free) tg = -1;
            } else {
              int64_t bc = INF;
              for (int jj = 0; jj < n; ++jj) {
                const int j = (s + 1) * n + jj;
                if (!I.alive[j] || I.adv_cost[j] == INF) continue;
                const int64_t dj = I.d(rr, j);
                if (dj == INF) continue;
                if (dj + I.adv_cost[j] < bc) { bc = dj + I.adv_cost[j]; tg = j; }
              }
            }
            if (tg != -2) rs = x;
          }
        }
        I.req_slot[rr] = rs;
        I.req_target[rr] = tg;
      }
      T.sync();
      // ---------- R2 grants: rank among same-target requesters in ascending gid ----------
      // (the grant is parked in prop[rr*6+5]; the data node's in sh_i32[.][2])
      for (int rr = T.tid; rr <= Sn; rr += TPI) {
        const int tg = I.req_target[rr];
        int32_t grant = kNone;
        if (tg >= 0) {
          int rank = 0;
          if (rr != Sn) {
            if (I.req_target[Sn] == tg) ++rank;  // D orders before all relays
            const int s0 = (rr / n) * n;
            for (int q = s0; q < rr; ++q) rank += I.req_target[q] == tg;
          }
          const int64_t ac = I.adv_cost[tg];
          for (int j = 0; j < I.capE(tg); ++j) {
            const int p = tg * MC + j;
            if (I.st(p) == 1 && I.scost[p] == ac) { if (rank == 0) { grant = p; break; } --rank; }
          }
        } else if (tg == -1) {
          int rank = 0;
          for (int q = (S - 1) * n; q < rr; ++q) rank += I.req_target[q] == -1;
          for (int k = 0; k < M; ++k)
            if (I.snk_up[k] == kNone) { if (rank == 0) { grant = -2 - k; break; } --rank; }
        }
        if (rr == Sn) sh_i32[T.id][2] = grant;
        else I.prop[rr * 6 + 5] = grant;
      }
      T.sync();
      // ---------- R3 commit grants ----------
      for (int rr = T.tid; rr <= Sn; rr += TPI) {
        const int32_t grant = rr == Sn ? sh_i32[T.id][2] : I.prop[rr * 6 + 5];
        if (grant == kNone) continue;
        const int32_t rs = I.req_slot[rr];
        if (rr == Sn) I.src_down[-2 - rs] = grant;
        else { I.down[rs] = grant; I.deny[rr] = 0; }
        I.set_up_of(grant, rs);
        changed = 1;
      }
      T.sync();
      // ---------- R4 proposals by idle relays (post-R3 state) ----------
      for (int p = T.tid; p < Sn; p += TPI) {
        int kind = K_NONE;
        int32_t x = kNone, y = kNone, z = kNone;
        int64_t t0 = -1, t1 = -1, t2 = -1, t3 = -1;
        uint64_t key = RES_NONE;
        if (I.alive[p] && I.req_target[p] == -2) {
          const SlotScan sc = scan_slots(I, p);
          const int s = p / n, i = p % n;
          if (sc.first_in >= 0) {
            const int dw = I.deny[p] + 1;
            I.deny[p] = dw;
            if (dw >= P.deny_after) {
              kind = K_DENY;
              x = sc.first_in;
              t0 = x;
              t1 = I.res_up(I.up[x]);
              key = (uint64_t)p;  // delta = -inf
            }
          } else if (n >= 2) {
            uint32_t qi = pick(I.h(round, p, 0), (uint32_t)(n - 1));
            if ((int)qi >= i) qi += 1;
            const int q = s * n + (int)qi;
            const int nq = I.alive[q] ? scan_slots(I, q).npaired : 0;
            if (nq > 0) {
              int64_t delta = 0;
              bool ok = false;
              if (sc.first_free >= 0 && !sc.has_out) {  // Request Redirect
                y = nth_paired(I, q, (int)pick(I.h(round, p, 2), (uint32_t)nq));
                const int a = I.up[y] >= 0 ? I.up[y] / MC : -1, c = I.down[y] >= 0 ? I.down[y] / MC : -1;
                const int64_t dax = I.d(a, p), dxc = I.d(p, c), dab = I.d(a, q), dbc = I.d(q, c);
                if (dax != INF && dxc != INF && dab != INF && dbc != INF) {
                  delta = P.objective == 0 ? (dax + dxc) - (dab + dbc) : max(dax, dxc) - max(dab, dbc);
                  kind = K_REDIRECT;
                  z = sc.first_free;
                  t0 = y; t1 = I.res_up(I.up[y]); t2 = I.res_dn(I.down[y]); t3 = z;
                  ok = true;
                }
              } else if (sc.npaired > 0) {  // Request Change
                x = nth_paired(I, p, (int)pick(I.h(round, p, 1), (uint32_t)sc.npaired));
                y = nth_paired(I, q, (int)pick(I.h(round, p, 2), (uint32_t)nq));
                const int j1 = I.down[x] >= 0 ? I.down[x] / MC : -1, j2 = I.down[y] >= 0 ? I.down[y] / MC : -1;
                if (j1 != j2) {
                  const int64_t a1 = I.d(p, j2), a2 = I.d(q, j1), b1 = I.d(p, j1), b2 = I.d(q, j2);
                  if (a1 != INF && a2 != INF && b1 != INF && b2 != INF) {
                    delta = P.objective == 0 ? (a1 + a2) - (b1 + b2) : max(a1, a2) - max(b1, b2);
                    kind = K_CHANGE;
                    t0 = x; t1 = y; t2 = I.res_dn(I.down[x]); t3 = I.res_dn(I.down[y]);
                    ok = true;
                  }
                }
              }
              if (ok) {
                bool accept = delta < 0;
                if (delta > 0 && delta < P.thr_width) {  // annealing
                  const int kk = min(I.kacc[p], P.thr_K);
                  accept = (I.h(round, p, 3) >> 32) < (uint64_t)P.thr[(size_t)kk * P.thr_width + delta];
                }
                if (accept) key = ((uint64_t)(delta + (1ll << 40)) << 22) | (uint64_t)p;
                else kind = K_NONE;
              }
            }
          }
        }
        if (key == RES_NONE) kind = K_NONE;
        I.prop[p * 6 + 0] = kind;
        I.prop[p * 6 + 1] = x;
        I.prop[p * 6 + 2] = y;
        I.prop[p * 6 + 3] = z;
        I.pkey[p] = key;
        I.ptouch[p * 4 + 0] = t0;
        I.ptouch[p * 4 + 1] = t1;
        I.ptouch[p * 4 + 2] = t2;
        I.ptouch[p * 4 + 3] = t3;
        // ---------- R5 reservations ----------
        if (kind != K_NONE) {
          atomicMin((unsigned long long*)&I.res[t0], (unsigned long long)key);
          atomicMin((unsigned long long*)&I.res[t1], (unsigned long long)key);
          if (t2 >= 0) atomicMin((unsigned long long*)&I.res[t2], (unsigned long long)key);
          if (t3 >= 0) atomicMin((unsigned long long*)&I.res[t3], (unsigned long long)key);
        }
      }
      T.sync();
      // ---------- R6 commit the proposals that hold every slot they touch ----------
      for (int p = T.tid; p < Sn; p += TPI) {
        const int kind = I.prop[p * 6 + 0];
        if (kind == K_NONE) continue;
        const uint64_t key = I.pkey[p];
        bool win = true;
        for (int q = 0; q < 4; ++q) {
          const int64_t t = I.ptouch[p * 4 + q];
          if (t >= 0) win = win && __ldcg(&I.res[t]) == key;
        }
        if (!win) continue;
        const int32_t x = I.prop[p * 6 + 1], y = I.prop[p * 6 + 2], z = I.prop[p * 6 + 3];
        if (kind == K_CHANGE) {
          const int32_t dx = I.down[x], dy = I.down[y];
          I.down[x] = dy;
          I.down[y] = dx;
          I.set_up_of(dy, x);
          I.set_up_of(dx, y);
          I.kacc[p] += 1;
        } else if (kind == K_REDIRECT) {
          const int32_t a = I.up[y], c = I.down[y];
          I.up[z] = a;
          I.down[z] = c;
          I.set_down_of(a, z);
          I.set_up_of(c, z);
          I.up[y] = kNone;
          I.down[y] = kNone;
          I.kacc[p] += 1;
        } else {
          const int32_t a = I.up[x];
          I.up[x] = kNone;
          I.set_down_of(a, kNone);
          I.deny[p] = 0;
        }
        changed = 1;
      }
      T.sync();
      for (int p = T.tid; p < Sn; p += TPI) {  // release the reservations for the next round
        if (I.prop[p * 6 + 0] == K_NONE) continue;
        for (int q = 0; q < 4; ++q) {
          const int64_t t = I.ptouch[p * 4 + q];
          if (t >= 0) __stcg(&I.res[t], RES_NONE);
        }
      }
      // ---------- R7 ----------
      const int any = T.sync_or(changed);
      quiet = any ? 0 : quiet + 1;
      round += 1;
      if (o.digests) {
        if (T.tid == 0) sh_u64[T.id][0] = 0;
        T.sync();
        uint64_t acc = 0;
        const int nslot = Sn * MC;
        for (int p = T.tid; p < nslot; p += TPI) {
          const int32_t u = I.up[p], dn = I.down[p];
          const uint64_t eu = u == kNone ? 0 : (u >= 0 ? 1 + (uint64_t)u : (1ull << 40) + (uint64_t)(-2 - u));
          const uint64_t ed = dn == kNone ? 0 : (dn >= 0 ? 1 + (uint64_t)dn : (1ull << 41) + (uint64_t)(-2 - dn));
          const uint64_t state = (u != kNone ? 2 : 0) | (dn != kNone ? 1 : 0);
          acc += digest_elem(3ull * p, state) + digest_elem(3ull * p + 1, eu) + digest_elem(3ull * p + 2, ed);
        }
        const uint64_t b1 = 3ull * nslot, b2 = b1 + M, b3 = b2 + M, b4 = b3 + 2ull * Sn;
        for (int k = T.tid; k < M; k += TPI) {
          const int32_t sd = I.src_down[k], su = I.snk_up[k];
          acc += digest_elem(b1 + k, sd == kNone ? 0 : 1 + (uint64_t)sd);
          acc += digest_elem(b2 + k, su == kNone ? 0 : 1 + (uint64_t)su);
        }
        for (int v = T.tid; v < Sn; v += TPI) {
          acc += digest_elem(b3 + 2ull * v, (uint64_t)(uint32_t)I.kacc[v]);
          acc += digest_elem(b3 + 2ull * v + 1, (uint64_t)(uint32_t)I.deny[v]);
        }
        if (T.tid == 0) acc += digest_elem(b4, (uint64_t)(uint32_t)quiet);
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) atomicAdd((unsigned long long*)&sh_u64[T.id][0], (unsigned long long)acc);
        T.sync();
        if (T.tid == 0) o.digests[(size_t)b * o.max_rounds + r] = sh_u64[T.id][0];
      }
      ++r;
      if (quiet >= P.W) break;
    }
    if (o.digests)
      for (int k = r + T.tid; k < o.max_rounds; k += TPI) o.digests[(size_t)b * o.max_rounds + k] = 0;
    // ---------- results: complete SRC -> SNK chains and dangling outflows ----------
    if (T.tid == 0) { sh_u64[T.id][0] = 0; sh_u64[T.id][1] = 0; sh_i32[T.id][3] = 0; }
    T.sync();
    {
      unsigned long long f = 0, c = 0;
      for (int k = T.tid; k < M; k += TPI) {
        int32_t p = I.src_down[k];
        if (p == kNone) continue;
        int64_t cc = I.d(-1, p / MC);
        int guard = 0;
        bool ok = true;
        while (p >= 0 && ++guard <= S + 1) {
          const int32_t nx = I.down[p];
          if (nx == kNone) { ok = false; break; }
          cc = sadd(cc, I.d(p / MC, nx <= -2 ? -1 : nx / MC));
          p = nx;
        }
        if (ok && p <= -2 && cc != INF) { f += 1; c += (unsigned long long)cc; }
      }
      int dg = 0;
      for (int p = T.tid; p < Sn * MC; p += TPI) dg += I.st(p) == 1;
      for (int off = 16; off > 0; off >>= 1) {
        f += __shfl_xor_sync(0xffffffffu, f, off);
        c += __shfl_xor_sync(0xffffffffu, c, off);
        dg += __shfl_xor_sync(0xffffffffu, dg, off);
      }
      if (lane == 0) {
        atomicAdd((unsigned long long*)&sh_u64[T.id][0], f);
        atomicAdd((unsigned long long*)&sh_u64[T.id][1], c);
        atomicAdd(&sh_i32[T.id][3], dg);
      }
    }
    T.sync();
    if (T.tid == 0) {
      if (o.rounds_run) o.rounds_run[b] = r;
      if (o.F_dec) o.F_dec[b] = (int64_t)sh_u64[T.id][0];
      if (o.cost_dec) o.cost_dec[b] = (int64_t)sh_u64[T.id][1];
      if (o.dangling) o.dangling[b] = sh_i32[T.id][3];
      P.quiet[b] = quiet;
      P.round[b] = (int64_t)round;
    }
    T.sync();
  }
}

__global__ void init_round_state_kernel(const Problem P) {
  const size_t Sn = (size_t)P.S * P.n;
  const size_t nslot = (size_t)P.B * Sn * P.MC;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (size_t t = t0; t < nslot; t += stride) { P.up[t] = kNone; P.down[t] = kNone; }
  for (size_t t = t0; t < (size_t)P.B * P.Mmax; t += stride) { P.src_down[t] = kNone; P.snk_up[t] = kNone; }
  for (size_t t = t0; t < (size_t)P.B * Sn; t += stride) { P.kacc[t] = 0; P.deny[t] = 0; }
  for (size_t t = t0; t < (size_t)P.B; t += stride) { P.quiet[t] = 0; P.round[t] = 0; }
}

template <int TPI>
cudaError_t launch_rounds_tpi(const Problem& P, const RoundsOut& o, cudaStream_t st, int num_sms) {
  const int teams = 256 / TPI > 8 ? 8 : 256 / TPI;
  auto k = rounds_kernel<TPI>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, teams * TPI, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  long long grid = (long long)per_sm * num_sms;
  const long long need = (P.B + teams - 1) / teams;
  if (grid > need) grid = need;
  k<<<(int)grid, teams * TPI, 0, st>>>(P, o);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_init_round_state(const Problem& P, cudaStream_t st) {
  init_round_state_kernel<<<148 * 4, 256, 0, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_rounds(const Problem& P, const RoundsOut& o, cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemsetAsync(P.counters + 1, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const int Sn = P.S * P.n;
  if (Sn <= 128) return launch_rounds_tpi<32>(P, o, st, num_sms);
  if (Sn <= 512) return launch_rounds_tpi<64>(P, o, st, num_sms);
  if (Sn <= 4096) return launch_rounds_tpi<128>(P, o, st, num_sms);
  return launch_rounds_tpi<256>(P, o, st, num_sms);
}

}  // namespace gwtf
