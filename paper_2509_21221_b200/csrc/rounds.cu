// Decentralized neighbour-exchange flow rounds, synchronous semantics.
//
// PAPER.md:241-263 (Request Flow / Request Change / Request Redirect, simulated annealing,
// steady state) and :269 (DENY).  One team of TPI threads per instance, persistent over an
// atomic instance queue; every phase is relay-parallel (thread t owns relays t, t+TPI, ...)
// and phases are separated by team barriers, so each phase reads the snapshot the
// definition names:
//   summaries | R0a self-pairing (round-start costs) | R0 cost-to-sink back to front +
//   advertisements | R1 one Request Flow per node | R2 grants in requester order | R3 commit |
//   summaries | R4 Change / Redirect / DENY proposals on the post-R3 state (counter RNG,
//   integer annealing thresholds) + R5 deterministic reservations (64-bit atomicMin, order
//   free) | R6 commit winners | R7 quiet counter, optional state digest.
// Index arithmetic uses multiply-shift division (no runtime integer division on the hot
// path).  The per-instance state either lives in global memory (L1/L2 resident; reservation
// minima read with ld.global.cg since they are produced by L2 atomics) or is staged in
// shared memory (tiles by TMA bulk copy) when it fits.
#include <cooperative_groups.h>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace gwtf {

namespace {

constexpr int64_t INF = INT64_MAX;
constexpr uint64_t RES_NONE = ~0ull;
enum { K_NONE = 0, K_CHANGE = 1, K_REDIRECT = 2, K_DENY = 3 };
enum { ST_FREE = 0, ST_OUT = 1, ST_IN = 2, ST_PAIRED = 3 };

int getenv_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// q = x / d for 0 <= x < 2^31 by multiply-shift (Granlund-Montgomery)
struct FastDiv {
  uint32_t d, mul, shr;
  __host__ __device__ void init(uint32_t div) {
    d = div;
    shr = 0;
    while ((1u << shr) < div) ++shr;
    mul = div == 1 ? 0u : (uint32_t)(((1ull << 32) * ((1ull << shr) - div)) / div + 1);
  }
  __device__ __forceinline__ int div(int x) const {
    return d == 1 ? x : (int)((__umulhi((uint32_t)x, mul) + (uint32_t)x) >> shr);
  }
};

__device__ __forceinline__ uint64_t mix(uint64_t z) {  // splitmix64 finalizer
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t pick(uint64_t x, uint32_t m) {
  return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32);
}
__device__ __forceinline__ int64_t sadd(int64_t a, int64_t b) { return (a == INF || b == INF) ? INF : a + b; }
__device__ __forceinline__ int64_t cst(int32_t c) { return c == kAbsent ? INF : (int64_t)c; }

// per-relay slot summary: first IN slot, first FREE slot (63 = none), #PAIRED, has OUT
struct Summ {
  uint32_t w;
  __device__ int first_in() const { return (int)(w & 63u); }
  __device__ int first_free() const { return (int)((w >> 6) & 63u); }
  __device__ int npaired() const { return (int)((w >> 12) & 63u); }
  __device__ bool has_out() const { return (w >> 18) & 1u; }
  __device__ bool has_in() const { return first_in() != 63; }
};

struct Inst {
  const Problem* P;
  int S, n, ld, MC, Sn, M, inst;
  FastDiv dn, dmc;
  int32_t *up, *down, *src_down, *snk_up, *kacc, *deny;
  int64_t *scost, *adv_cost;
  int32_t *req_slot, *req_target, *grant, *prop, *ptouch, *capv;
  uint32_t* summ;
  // incremental bookkeeping (K2): slots whose down pointer changed since the costs were
  // last brought up to date (flag + list), relays whose summary / advertisement is stale (flag +
  // list), the advertiser bitmask per stage [S][W] and its population count per stage
  int32_t *mflag, *mlist, *rflag, *rlist, *advcnt, *lcnt;
  uint32_t* advm;
  uint32_t* pmask;  // per relay: bit j = slot j is PAIRED (max_cap <= 32), maintained with summ
  uint32_t* omask;  // per relay: bit j = slot j is OUT
  int32_t* first_req;  // per target relay: lowest requester gid of the round (INT_MAX: none)
  int32_t* lcd;        // per slot: cost of the link to its down pointer's node (kAbsent: none / absent)
  int W;
  uint64_t *pkey, *res;
  const int32_t *tile, *src, *snk;
  const uint8_t* alive;
  uint64_t hpre;  // mix(mix(mix(seed) ^ inst) ^ round), uniform over the round
  uint64_t hinst;  // mix(mix(seed) ^ inst), fixed per instance

  __device__ int st(int p) const { return (up[p] != kNone ? 2 : 0) | (down[p] != kNone ? 1 : 0); }
  __device__ int relay(int32_t p) const { return dmc.div(p); }           // slot index -> gid
  // one instance's tile has (S-1) n ld < 2^31 entries (create: S <= 64, n <= 4096): 32-bit indices
  __device__ int64_t c_link(int s, int u, int v) const { return cst(tile[(uint32_t)((s * n + v) * ld + u)]); }
  // d(a, b) between nodes; -1 = data node D.  Missing / absent = INF.
  __device__ int64_t d(int a, int b) const {
    if (a < 0) return (b >= 0 && b < n) ? cst(src[b]) : INF;
    const int sa = dn.div(a);
    if (b < 0) return sa == S - 1 ? cst(snk[a - sa * n]) : INF;
    const int sb = dn.div(b);
    return sb == sa + 1 ? c_link(sa, a - sa * n, b - sb * n) : INF;
  }
  __device__ int32_t res_up(int32_t p) const { return p >= 0 ? p : Sn * MC + (-2 - p); }
  __device__ int32_t res_dn(int32_t p) const { return p >= 0 ? p : Sn * MC + (int32_t)P->Mmax + (-2 - p); }
  __device__ void set_up_of(int32_t p, int32_t v) { if (p >= 0) up[p] = v; else snk_up[-2 - p] = v; }
  __device__ void set_down_of(int32_t p, int32_t v) { if (p >= 0) down[p] = v; else src_down[-2 - p] = v; }
  __device__ void set_round(uint64_t round) {
    hpre = mix(hinst ^ round);
  }
  __device__ uint64_t h(int gid, int stream) const { return mix(hpre ^ ((uint64_t)gid * 4 + stream)); }

  __device__ uint32_t summarize(int v) const {
    uint32_t fi = 63, ff = 63, np = 0, ho = 0;
    const int c = capv[v], base = v * MC;
    _Pragma("unroll 1") for (int j = 0; j < c; ++j) {
      const int t = st(base + j);
      if (t == ST_IN && fi == 63) fi = j;
      if (t == ST_FREE && ff == 63) ff = j;
      np += t == ST_PAIRED;
      ho |= t == ST_OUT;
    }
    return fi | (ff << 6) | (np << 12) | (ho << 18);
  }
  // R0 for one relay: cost to sink of each usable slot by walking its down chain (the
  // back-to-front recursion cost(slot) = d(v, node(down)) + cost(down) unrolled; no barriers);
  // returns adv(v) = min cost over its OUT slots
  __device__ int64_t relay_costs(int v) const {
    const int s0 = dn.div(v), i0 = v - s0 * n, c = capv[v];
    int64_t best = INF;
    _Pragma("unroll 1") for (int j = 0; j < c; ++j) {
      const int p0 = v * MC + j;
      int32_t p = down[p0];
      int64_t cc = p == kNone ? INF : 0;
      int s = s0, i = i0;
      while (p != kNone) {
        if (p <= -2) { cc = sadd(cc, cst(snk[i])); break; }
        const int w = relay(p), wi = w - (s + 1) * n;
        cc = sadd(cc, c_link(s, i, wi));
        s += 1;
        i = wi;
        p = down[p];
        if (p == kNone) cc = INF;
      }
      scost[p0] = cc;
      if (up[p0] == kNone && down[p0] != kNone && cc < best) best = cc;
    }
    return best;
  }
  // chain walk of one slot (unusable slots get INF)
  __device__ void slot_cost(int p0) const {
    const int v = relay(p0), j = p0 - v * MC;
    int64_t cc = INF;
    if (j < capv[v]) {
      int32_t p = down[p0];
      if (p != kNone) {
        cc = 0;
        int s = dn.div(v), i = v - s * n;
        while (true) {
          if (p <= -2) { cc = sadd(cc, cst(snk[i])); break; }
          const int w = relay(p), wi = w - (s + 1) * n;
          cc = sadd(cc, c_link(s, i, wi));
          s += 1;
          i = wi;
          p = down[p];
          if (p == kNone) { cc = INF; break; }
        }
      }
    }
    scost[p0] = cc;
  }
  // adv(v) from the maintained OUT-slot mask (refresh() first)
  __device__ int64_t adv_of(int v) const {
    int64_t bc = INF;
    for (uint32_t t = omask[v]; t; t &= t - 1) {
      const int64_t c = scost[v * MC + __ffs(t) - 1];
      if (c < bc) bc = c;
    }
    return bc;
  }
  __device__ int64_t relay_adv(int v) const {
    int64_t bc = INF;
    const int c = capv[v];
    _Pragma("unroll 1") for (int j = 0; j < c; ++j) {
      const int p = v * MC + j;
      if (up[p] == kNone && down[p] != kNone && scost[p] < bc) bc = scost[p];
    }
    return bc;
  }
  // summary and PAIRED-slot mask of relay v, stored
  __device__ void refresh(int v) const {
    uint32_t fi = 63, ff = 63, np = 0, ho = 0, pm = 0, om = 0;
    const int c = capv[v], base = v * MC;
    _Pragma("unroll 4") for (int j = 0; j < c; ++j) {  // 4 slots' loads in flight
      const int t = st(base + j);
      if (t == ST_IN && fi == 63) fi = j;
      if (t == ST_FREE && ff == 63) ff = j;
      np += t == ST_PAIRED;
      pm |= (uint32_t)(t == ST_PAIRED) << j;
      om |= (uint32_t)(t == ST_OUT) << j;
      ho |= t == ST_OUT;
    }
    summ[v] = fi | (ff << 6) | (np << 12) | (ho << 18);
    pmask[v] = pm;
    omask[v] = om;
  }
  // the q-th PAIRED slot of relay v (slot order), from the maintained mask
  __device__ int nth_paired_m(int v, int q) const {
    uint32_t m = pmask[v];
    for (; q > 0; --q) m &= m - 1;
    return m ? v * MC + __ffs(m) - 1 : -1;
  }
  // link cost from slot p's node to its down pointer's node (an SNK pointer: the sink cost)
  __device__ int32_t link_down(int32_t p) const {
    const int32_t d1 = down[p];
    if (d1 == kNone) return kAbsent;
    const int v = relay(p), s = dn.div(v), i = v - s * n;
    if (d1 <= -2) return snk[i];
    return tile[((size_t)s * n + (relay(d1) - (s + 1) * n)) * ld + i];
  }
  // a slot whose down pointer just changed: its link cost is refreshed and it is listed for the
  // next cost update (walk_marks)
  __device__ void mark_slot(int32_t p) const {
    if (p < 0) return;
    lcd[p] = link_down(p);
    if (atomicExch(&mflag[p], 1) == 0) mlist[atomicAdd(&lcnt[0], 1)] = p;
  }
  __device__ void mark_relay(int v) const {
    if (atomicExch(&rflag[v], 1) == 0) rlist[atomicAdd(&lcnt[1], 1)] = v;
  }
  // cost to sink of slot p from its down pointer (valid when scost[down p] is up to date)
  __device__ int64_t cost_from(int32_t p) const {
    const int32_t d1 = down[p];
    if (d1 == kNone) return INF;
    return d1 <= -2 ? cst(lcd[p]) : sadd(cst(lcd[p]), scost[d1]);
  }
  // the advertisement of v and its bit in the stage's advertiser mask (count kept in advcnt)
  __device__ void set_adv(int v, int64_t a) const {
    const int64_t old = adv_cost[v];
    adv_cost[v] = a;
    if ((a != INF) == (old != INF)) return;
    const int s = dn.div(v), i = v - s * n;
    uint32_t* w = advm + (size_t)s * W + (i >> 5);
    if (a != INF) { atomicOr(w, 1u << (i & 31)); atomicAdd(&advcnt[s], 1); }
    else { atomicAnd(w, ~(1u << (i & 31))); atomicSub(&advcnt[s], 1); }
  }
  __device__ int nth_paired(int v, int q) const {
    const int c = capv[v], base = v * MC;
    _Pragma("unroll 1") for (int j = 0; j < c; ++j)
      if (st(base + j) == ST_PAIRED) { if (q == 0) return base + j; --q; }
    return -1;
  }
};

// A team that spans a thread-block cluster of C CTAs x 1,024 threads (stress-sized instances:
// 64 x 1,024 relays would leave one CTA with 256 relays per thread).  Barriers are cluster
// barriers (release/acquire; the acquire invalidates L1, so plain global loads after a barrier
// see every CTA's writes); the OR vote goes through per-CTA DSMEM slots read by every CTA.
template <int C>
struct ClusterTeam {
  static constexpr int kTPI = C * 1024;
  int tid, id;
  uint32_t* vslot;  // this CTA's two vote slots (shared memory)
  uint32_t vid;     // vote counter (uniform over the cluster)
  __device__ __forceinline__ void sync() const { cg::this_cluster().sync(); }
  __device__ int sync_or(int p) {
    ++vid;
    if (p) vslot[vid & 1] = vid;  // stamp (idempotent); the cluster barrier orders it before the reads
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    int res = 0;
    for (int q = 0; q < C; ++q) res |= cl.map_shared_rank(vslot, q)[vid & 1] == vid;
    return res;
  }
};
template <int TPI>
struct TeamOf {  // adapter giving Team<TPI> the same interface
  static constexpr int kTPI = TPI;
  Team<TPI> t;
  int tid, id;
  __device__ __forceinline__ void sync() const { t.sync(); }
  __device__ __forceinline__ int sync_or(int p) const { return t.sync_or(p); }
};

template <class TT>
__device__ void compute_costs(TT& T, const Inst& I) {
  constexpr int TPI = TT::kTPI;
  const int per = I.n * I.MC;
  for (int s = I.S - 1; s >= 0; --s) {
    _Pragma("unroll 1") for (int t = T.tid; t < per; t += TPI) {
      const int i = I.dmc.div(t), j = t - i * I.MC, v = s * I.n + i, p = v * I.MC + j;
      int64_t c = INF;
      if (j < I.capv[v]) {
        const int32_t dn = I.down[p];
        if (dn <= -2) c = cst(I.snk[i]);
        else if (dn >= 0) {
          const int w = I.relay(dn);
          c = sadd(I.c_link(s, i, w - (s + 1) * I.n), I.scost[dn]);
        }
      }
      I.scost[p] = c;
    }
    T.sync();
  }
}

__device__ uint64_t digest_elem(uint64_t pos, uint64_t val) { return mix(mix(pos) ^ val); }

// ---- per-team workspace layout ---------------------------------------------------------
__host__ __device__ inline size_t al16r(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline bool rounds_tile_in_smem(const Problem& P) {
  return (size_t)(P.S > 1 ? P.S - 1 : 0) * P.n * P.ld * 4 <= 16384;
}
struct RoundsLayout {
  size_t res, scost, adv_cost, pkey, up, down, src_down, snk_up, kacc, deny, req_slot, req_target, grant, prop,
      ptouch, capv, summ, mflag, mlist, rflag, rlist, advm, advcnt, pmask, omask, first_req, lcd, lcnt, tile, mbar, cells, total;
};
// smem: everything of one instance; otherwise only the per-instance scratch (the state
// arrays then live in the handle's global buffers)
__host__ __device__ inline RoundsLayout rounds_layout(const Problem& P, bool smem) {
  RoundsLayout L;
  size_t o = 0;
  const size_t Sn = (size_t)P.S * P.n, ns = Sn * P.MC, M = (size_t)P.Mmax;
  L.res = o; o += al16r((ns + 2 * M) * 8);
  L.scost = o; o += al16r(ns * 8);
  L.adv_cost = o; o += al16r(Sn * 8);
  L.pkey = o; o += al16r(Sn * 8);
  L.up = o; if (smem) o += al16r(ns * 4);
  L.down = o; if (smem) o += al16r(ns * 4);
  L.src_down = o; if (smem) o += al16r(M * 4);
  L.snk_up = o; if (smem) o += al16r(M * 4);
  L.kacc = o; if (smem) o += al16r(Sn * 4);
  L.deny = o; if (smem) o += al16r(Sn * 4);
  L.req_slot = o; o += al16r((Sn + 1) * 4);
  L.req_target = o; o += al16r((Sn + 1) * 4);
  L.grant = o; o += al16r((Sn + 1) * 4);
  L.prop = o; o += al16r(Sn * 4 * 4);
  L.ptouch = o; o += al16r(Sn * 4 * 4);
  L.capv = o; o += al16r(Sn * 4);
  L.summ = o; o += al16r(Sn * 4);
  L.mflag = o; o += al16r(ns * 4);
  L.mlist = o; o += al16r((ns + 16) * 4);
  L.rflag = o; o += al16r(Sn * 4);
  L.rlist = o; o += al16r(Sn * 4);
  L.advm = o; o += al16r((size_t)P.S * ((P.n + 31) / 32) * 4);
  L.advcnt = o; o += al16r((size_t)P.S * 4);
  L.pmask = o; o += al16r(Sn * 4);
  L.omask = o; o += al16r(Sn * 4);
  L.first_req = o; o += al16r(Sn * 4);
  L.lcd = o; o += al16r(ns * 4);
  L.lcnt = o; o += 16;
  L.tile = o; if (smem && rounds_tile_in_smem(P)) o += al16r((size_t)(P.S > 1 ? P.S - 1 : 0) * P.n * P.ld * 4);
  L.mbar = o; o += 16;
  L.cells = o; o += 64;  // the cluster team's reduction cells
  L.total = o;
  return L;
}

template <bool kSmem>
__device__ __forceinline__ uint64_t ld_res(const uint64_t* p) {
  if constexpr (kSmem) return *(volatile const uint64_t*)p;
  else return __ldcg(p);
}
template <bool kSmem>
__device__ __forceinline__ void st_res(uint64_t* p, uint64_t v) {
  if constexpr (kSmem) *p = v;
  else __stcg(p, v);
}

// Team reduction cells: shared memory for CTA teams, the team workspace (global, L2 atomics)
// for cluster teams.  [0..1] u64 sums, [0..3] i32 min/or/sum, instance index.
struct Red {
  unsigned long long* u64;
  int* i32;
  int* inst;
};

template <class TT, bool kSmem>
__device__ __forceinline__ void rounds_body(const Problem& P, const RoundsOut& o, const size_t ws_bytes, TT& T,
                                            uint8_t* base, Red red, uint8_t* dsm, int* tma_init,
                                            uint32_t* tma_phase_of) {
  constexpr int TPI = TT::kTPI;
  const int lane = threadIdx.x & 31;
  const int S = P.S, n = P.n, MC = P.MC, Sn = S * n;
  const int nres = Sn * MC + 2 * (int)P.Mmax;
  const RoundsLayout Lr = rounds_layout(P, kSmem);
  unsigned long long* const sh_u64 = red.u64;
  int* const sh_i32 = red.i32;

  for (;;) {
    if (T.tid == 0) *(volatile int*)red.inst = atomicAdd(&P.counters[1], 1);
    T.sync();
    const int b = *(volatile int*)red.inst;
    T.sync();  // every thread of the team has read it before it can be rewritten
    if (b >= P.B) break;
    Inst I;
    I.P = &P; I.S = S; I.n = n; I.ld = P.ld; I.MC = MC; I.Sn = Sn; I.inst = b;
    I.hinst = mix(mix(P.seed) ^ (uint64_t)(P.inst_base + b));
    I.dn.init((uint32_t)n);
    I.dmc.init((uint32_t)(MC > 0 ? MC : 1));
    I.M = (int)P.supply[b];
    I.up = P.up + (size_t)b * Sn * MC;
    I.down = P.down + (size_t)b * Sn * MC;
    I.src_down = P.src_down + (size_t)b * P.Mmax;
    I.snk_up = P.snk_up + (size_t)b * P.Mmax;
    I.kacc = P.kacc + (size_t)b * Sn;
    I.deny = P.deny + (size_t)b * Sn;
    I.tile = P.tile + (size_t)b * (S - 1) * n * P.ld;
    I.src = P.src + (size_t)b * n;
    I.snk = P.snk + (size_t)b * n;
    I.alive = P.alive + (size_t)b * Sn;
    I.res = (uint64_t*)(base + Lr.res);
    I.scost = (int64_t*)(base + Lr.scost);
    I.adv_cost = (int64_t*)(base + Lr.adv_cost);
    I.pkey = (uint64_t*)(base + Lr.pkey);
    I.req_slot = (int32_t*)(base + Lr.req_slot);
    I.req_target = (int32_t*)(base + Lr.req_target);
    I.grant = (int32_t*)(base + Lr.grant);
    I.prop = (int32_t*)(base + Lr.prop);
    I.ptouch = (int32_t*)(base + Lr.ptouch);
    I.capv = (int32_t*)(base + Lr.capv);
    I.summ = (uint32_t*)(base + Lr.summ);
    I.mflag = (int32_t*)(base + Lr.mflag);
    I.mlist = (int32_t*)(base + Lr.mlist);
    I.rflag = (int32_t*)(base + Lr.rflag);
    I.rlist = (int32_t*)(base + Lr.rlist);
    I.advm = (uint32_t*)(base + Lr.advm);
    I.advcnt = (int32_t*)(base + Lr.advcnt);
    I.lcnt = (int32_t*)(base + Lr.lcnt);
    I.pmask = (uint32_t*)(base + Lr.pmask);
    I.omask = (uint32_t*)(base + Lr.omask);
    I.first_req = (int32_t*)(base + Lr.first_req);
    I.lcd = (int32_t*)(base + Lr.lcd);
    I.W = (n + 31) / 32;
    const int M = I.M;
    const int32_t* cap_g = P.cap + (size_t)b * Sn;
    _Pragma("unroll 1") for (int k = T.tid; k < Sn; k += TPI) I.capv[k] = I.alive[k] ? cap_g[k] : 0;
    int32_t* g_up = I.up;
    int32_t* g_down = I.down;
    int32_t* g_src_down = I.src_down;
    int32_t* g_snk_up = I.snk_up;
    int32_t* g_kacc = I.kacc;
    int32_t* g_deny = I.deny;
    if constexpr (kSmem) {  // stage the round state (and small tiles, by TMA) in shared memory
      uint64_t* mbar = (uint64_t*)(base + Lr.mbar);
      I.up = (int32_t*)(base + Lr.up);
      I.down = (int32_t*)(base + Lr.down);
      I.src_down = (int32_t*)(base + Lr.src_down);
      I.snk_up = (int32_t*)(base + Lr.snk_up);
      I.kacc = (int32_t*)(base + Lr.kacc);
      I.deny = (int32_t*)(base + Lr.deny);
      const int32_t* gtile = I.tile;
      const bool tile_smem = rounds_tile_in_smem(P);
      if (tile_smem) I.tile = (const int32_t*)(base + Lr.tile);
      const uint32_t tbytes = tile_smem ? (uint32_t)((size_t)(S - 1) * n * P.ld * 4) : 0u;
      if (T.tid == 0 && tbytes) {
        if (tma_init[T.id] == 0) { mbar_init(mbar, 1); fence_barrier_init(); tma_init[T.id] = 1; }
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(mbar, tbytes);
        for (uint32_t off = 0; off < tbytes; off += 32768u)
          bulk_g2s(base + Lr.tile + off, (const uint8_t*)gtile + off, tbytes - off < 32768u ? tbytes - off : 32768u,
                   mbar);
      }
      _Pragma("unroll 1") for (int k = T.tid; k < Sn * MC; k += TPI) { I.up[k] = g_up[k]; I.down[k] = g_down[k]; }
      _Pragma("unroll 1") for (int k = T.tid; k < M; k += TPI) { I.src_down[k] = g_src_down[k]; I.snk_up[k] = g_snk_up[k]; }
      _Pragma("unroll 1") for (int k = T.tid; k < Sn; k += TPI) { I.kacc[k] = g_kacc[k]; I.deny[k] = g_deny[k]; }
      T.sync();
      if (tbytes) {  // barrier init visible; every thread waits on the transaction barrier
        const uint32_t ph = tma_phase_of[T.id];
        mbar_wait(mbar, ph);
        T.sync();
        if (T.tid == 0) tma_phase_of[T.id] = ph ^ 1u;
      }
    }

    _Pragma("unroll 1") for (int k = T.tid; k < nres; k += TPI) st_res<kSmem>(&I.res[k], RES_NONE);
    int quiet = 0;  // quiet = 0 at the start of every call (DESIGN.md 2.3 R7)
    const int cost_mode = P.rounds_cost_mode;
    uint64_t round = (uint64_t)P.round[b];
    int r = 0;
    const int W = I.W;
    const int lane_w = T.tid >> 5, nwarps = TPI / 32;  // warp index / count inside the team
#ifdef GWTF_DEV_FLAGS
    // development builds (GWTF_DEBUG_FLAGS & 16): leader-thread cycles per phase into stats[1200 + k]
    const bool prof = (P.debug & 16) && T.tid == 0 && T.id == 0 && blockIdx.x == 0;
    unsigned long long tl = clock64();
#define RMARK(k)                                                                       \
  do {                                                                                 \
    if (prof) {                                                                        \
      const unsigned long long t_ = clock64();                                         \
      atomicAdd(&P.stats[1200 + (k)], t_ - tl);                                        \
      tl = t_;                                                                         \
    }                                                                                  \
  } while (0)
#define WSTAT(k, v) do { if (P.debug & 16) atomicAdd(&P.stats[1220 + (k)], (unsigned long long)(v)); } while (0)
#else
#define RMARK(k) do {} while (0)
#define WSTAT(k, v) do {} while (0)
#endif
    // ---- incremental bookkeeping (K2) ----
    // walkers: every marked slot that has no marked slot below it in its chain (chains are disjoint
    // paths of down pointers) recomputes its own cost and every cost above it, bottom-up; below the
    // lowest mark nothing changed, so each chain is brought up to date by exactly one walker.  The
    // relay at the top of a chain (an OUT slot's owner) gets its advertisement refreshed.
    auto walk_marks = [&]() {
      const int nm = *(volatile int*)&I.lcnt[0];
      _Pragma("unroll 1") for (int k = T.tid; k < nm; k += TPI) {
        const int32_t p = I.mlist[k];
        bool lowest = true;
        _Pragma("unroll 1") for (int32_t q = I.down[p]; q >= 0;) {
          const int32_t qn = I.down[q];  // issued together with the flag load: one latency per step
          WSTAT(3, 1);
          if (*(volatile int32_t*)&I.mflag[q]) { lowest = false; break; }
          q = qn;
        }
        WSTAT(0, 1);
        if (!lowest) continue;
        WSTAT(1, 1);
        int32_t x = p;
        int64_t c = p - I.relay(p) * MC < I.capv[I.relay(p)] ? I.cost_from(p) : INF;
        int32_t u = I.up[x];
        // software-pipelined: the next up pointer and this hop's link cost are loaded together
        _Pragma("unroll 1") for (;;) {
          if (u < 0) {
            I.scost[x] = c;
            if (u == kNone) I.mark_relay(I.relay(x));
            break;
          }
          const int32_t un = I.up[u];
          WSTAT(2, 1);
          const int32_t w = I.lcd[u];  // u's down link is the link u -> x
          I.scost[x] = c;
          c = sadd(cst(w), c);
          x = u;
          u = un;
        }
      }
    };
    // after a barrier: clear the slot marks; refresh summaries (and advertisements) of the listed relays
    // (returns the list lengths it read: the reset in the next phase uses them, not the counters)
    auto flush_relays = [&](int& nm, int& nr) {
      nm = *(volatile int*)&I.lcnt[0];
      _Pragma("unroll 1") for (int k = T.tid; k < nm; k += TPI) I.mflag[I.mlist[k]] = 0;
      nr = *(volatile int*)&I.lcnt[1];
      _Pragma("unroll 1") for (int k = T.tid; k < nr; k += TPI) {
        const int v = I.rlist[k];
        I.refresh(v);
        I.set_adv(v, I.adv_of(v));
      }
    };
    // after the next barrier: empty both lists
    auto reset_lists = [&](int nr) {
      _Pragma("unroll 1") for (int k = T.tid; k < nr; k += TPI) I.rflag[I.rlist[k]] = 0;
      if (T.tid == 0) { I.lcnt[0] = 0; I.lcnt[1] = 0; }
    };
    T.sync();
    bool prev_quiet = false;  // the last round changed nothing (the first round of a call always runs)
    while (r < o.max_rounds) {
      int changed = 0;
      I.set_round(round);
      // after a quiet round the slot state is what it was at that round's start (only the deny
      // counters moved, and R0-R3 do not read them): R0a..R3 would recompute the same costs, the
      // same requests and again no grant, so the round starts at R4 (its RNG is the only input
      // that differs); scost, adv_cost and req_* still hold the previous round's values
      if (!prev_quiet) {
      if (r == 0) {
        // ---------- first round of the call: every cost, summary and advertisement from scratch
        // (the state may come from a churn, an import or another call) ----------
        _Pragma("unroll 1") for (int k = T.tid; k < Sn * MC; k += TPI) I.mflag[k] = 0;
        _Pragma("unroll 1") for (int k = T.tid; k < Sn; k += TPI) { I.rflag[k] = 0; I.adv_cost[k] = INF; I.first_req[k] = INT_MAX; }
        _Pragma("unroll 1") for (int k = T.tid; k < S * W; k += TPI) I.advm[k] = 0u;
        _Pragma("unroll 1") for (int k = T.tid; k < S; k += TPI) I.advcnt[k] = 0;
        if (T.tid == 0) { I.lcnt[0] = 0; I.lcnt[1] = 0; }
        _Pragma("unroll 1") for (int k = T.tid; k < Sn * MC; k += TPI) I.lcd[k] = I.link_down(k);
        if (cost_mode == 1) {
          _Pragma("unroll 1") for (int t = T.tid; t < Sn * MC; t += TPI) I.slot_cost(t);
          T.sync();
        } else if (cost_mode == 2) {
          _Pragma("unroll 1") for (int v = T.tid; v < Sn; v += TPI) I.relay_costs(v);
          T.sync();
        } else {
          compute_costs<TT>(T, I);  // stage-synchronous back-to-front recursion (ends with a barrier)
        }
        _Pragma("unroll 1") for (int v = T.tid; v < Sn; v += TPI) {
          I.refresh(v);
          I.set_adv(v, I.adv_of(v));
        }
        T.sync();
      } else {
        // ---------- bring the costs up to date with the previous round's R3 / R6 changes ----------
        walk_marks();
        T.sync();
        int nm, nr;
        flush_relays(nm, nr);
        T.sync();
        reset_lists(nr);
      }
      RMARK(0);
      // ---------- R0a candidates: a relay holding an IN and an OUT slot ----------
      if (T.tid == 0) { sh_i32[0] = INT_MAX; sh_i32[1] = 0; }
      int cand = 0;
      _Pragma("unroll 1") for (int v = T.tid; v < Sn; v += TPI) {
        const uint32_t w = I.summ[v];
        cand |= (w & 63u) != 63u && ((w >> 18) & 1u);
      }
      const int any_cand = T.sync_or(cand);
      RMARK(1);
      if (any_cand) {
        // ---------- R0a self-pairing, costs of the round-start state (scost is up to date) ----------
        _Pragma("unroll 1") for (int v = T.tid; v < Sn; v += TPI) {
          const Summ sm{I.summ[v]};
          if (!sm.has_in() || !sm.has_out() || !I.alive[v]) continue;
          const int x = v * MC + sm.first_in();
          int oo = -1;
          for (int j = 0; j < I.capv[v]; ++j) {
            const int p = v * MC + j;
            if (I.st(p) == ST_OUT && (oo < 0 || I.scost[p] < I.scost[oo])) oo = p;
          }
          const int32_t cdn = I.down[oo];
          I.down[x] = cdn;
          I.set_up_of(cdn, x);
          I.down[oo] = kNone;
          I.mark_slot(x);
          I.mark_slot(oo);
          I.mark_relay(v);
          changed = 1;
        }
        T.sync();
        walk_marks();
        T.sync();
        int nm, nr;
        flush_relays(nm, nr);
        T.sync();
        reset_lists(nr);
        RMARK(2);
      }
      // ---------- data-node slots ----------
      {
        int fs = INT_MAX, anyfree = 0;
        _Pragma("unroll 1") for (int k = T.tid; k < M; k += TPI) {
          if (I.src_down[k] == kNone && k < fs) fs = k;
          anyfree |= I.snk_up[k] == kNone;
        }
        if (fs != INT_MAX) atomicMin(&sh_i32[0], fs);
        if (anyfree) atomicOr(&sh_i32[1], 1);
      }
      T.sync();
      RMARK(3);
      const int d_rslot = *(volatile int*)&sh_i32[0];
      const int dsink_free = *(volatile int*)&sh_i32[1];
      // ---------- R1 requests (one per node): argmin over the next stage's advertisers only
      // (the advertiser bitmask, in ascending position: the same lowest-j tie-break as a full scan
      // that skips INF advertisements) ----------
      // warp-uniform iteration (the warp operations below need every lane); the last warp also
      // carries the data node (rr == Sn)
      _Pragma("unroll 1") for (int rb = T.tid - lane; rb <= Sn; rb += TPI) {
        const int rr = rb + lane;
        int32_t rs = kNone, tg = -2;
        // requester slot: (a) the lowest IN slot, (b) the lowest FREE slot of a stable relay
        int32_t x = kNone;
        int s = 0, i = 0;
        if (rr < Sn) {
          s = I.dn.div(rr);
          i = rr - s * n;
          if (I.alive[rr]) {
            const Summ sm{I.summ[rr]};
            if (sm.has_in()) x = rr * MC + sm.first_in();                                   // (a)
            else if (!sm.has_out() && sm.first_free() != 63) x = rr * MC + sm.first_free();  // (b)
          }
        }
        const bool want = x != kNone && s < S - 1;
        // a warp whose lanes all sit in one stage walks that stage's advertisers together
        // (coalesced link loads, 4 advertisers in flight); otherwise every lane walks alone
        const int s0 = __shfl_sync(0xffffffffu, s, 0);
        const bool uni = __all_sync(0xffffffffu, rr < Sn && s == s0);
        const bool anyw = __any_sync(0xffffffffu, want);
        int64_t bc = INF;
        int tgw = -2;
        if (uni) {
          if (anyw && s0 < S - 1 && *(volatile int32_t*)&I.advcnt[s0 + 1] > 0) {
            const int32_t* col = I.tile + (size_t)s0 * n * I.ld + i;  // C[s][v][i], v = 0..n-1
            const int64_t* av = I.adv_cost + (s0 + 1) * n;
            const uint32_t* am = I.advm + (size_t)(s0 + 1) * W;
            _Pragma("unroll 1") for (int w = 0; w < W; ++w) {
              uint32_t bits = am[w];
              while (bits) {
                int jv[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  jv[t] = bits ? w * 32 + __ffs(bits) - 1 : -1;
                  bits &= bits - 1;
                }
                int32_t cv[4];
                int64_t avv[4];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                  if (jv[t] >= 0) { cv[t] = col[(uint32_t)(jv[t] * I.ld)]; avv[t] = av[jv[t]]; }
#pragma unroll
                for (int t = 0; t < 4; ++t)
                  if (jv[t] >= 0 && cv[t] != kAbsent && cv[t] + avv[t] < bc) { bc = cv[t] + avv[t]; tgw = (s0 + 1) * n + jv[t]; }
              }
            }
          }
        } else if (want && *(volatile int32_t*)&I.advcnt[s + 1] > 0) {
          const int32_t* col = I.tile + (size_t)s * n * I.ld + i;
          const int64_t* av = I.adv_cost + (s + 1) * n;
          const uint32_t* am = I.advm + (size_t)(s + 1) * W;
          _Pragma("unroll 1") for (int w = 0; w < W; ++w) {
            uint32_t bits = am[w];
            while (bits) {
              const int jj = w * 32 + __ffs(bits) - 1;
              bits &= bits - 1;
              const int32_t c = col[(size_t)jj * I.ld];
              if (c == kAbsent) continue;
              const int64_t aj = av[jj];
              if (c + aj < bc) { bc = c + aj; tgw = (s + 1) * n + jj; }
            }
          }
        }
        if (want) tg = tgw;
        else if (x != kNone && s == S - 1 && I.snk[i] != kAbsent && dsink_free) tg = -1;
        if (tg != -2) rs = x;
        if (rr == Sn && d_rslot != INT_MAX && *(volatile int32_t*)&I.advcnt[0] > 0) {
          // the data node requests for its lowest unpaired SRC slot (stage-0 advertisers)
          int64_t bd = INF;
          _Pragma("unroll 1") for (int w = 0; w < W; ++w) {
            uint32_t bits = I.advm[w];
            while (bits) {
              const int j = w * 32 + __ffs(bits) - 1;
              bits &= bits - 1;
              const int64_t dj = cst(I.src[j]), aj = I.adv_cost[j];
              if (dj == INF || !I.alive[j]) continue;
              if (dj + aj < bd) { bd = dj + aj; tg = j; }
            }
          }
          if (tg != -2) rs = -2 - d_rslot;
        }
        if (rr <= Sn) {
          I.req_slot[rr] = rs;
          I.req_target[rr] = tg;
          if (tg >= 0) atomicMin(&I.first_req[tg], rr);
        }
      }
      T.sync();
      RMARK(4);
      // ---------- R2 + R3: each target serves its requesters in ascending gid and commits ----------
      // (a target's eligibility only reads its own OUT slots, which only it modifies; requester
      // slots are IN/FREE slots written by exactly one target, so the fused commit equals
      // "all grants on the pre-R3 state, then all commits").  One thread per advertiser (the
      // bitmask): with one eligible slot -- the usual case -- the lowest-gid requester (first_req,
      // an atomicMin of R1) takes it; with several, the requesters are walked in gid order.
      auto commit_grant = [&](int qq, int32_t pslot) {
        const int32_t rs = I.req_slot[qq];
        I.down[rs] = pslot;
        I.up[pslot] = rs;
        I.deny[qq] = 0;
        I.mark_slot(rs);
        I.mark_relay(qq);
        changed = 1;
      };
      _Pragma("unroll 1") for (int w = T.tid; w < S * W; w += TPI) {
        uint32_t bits = I.advm[w];
        const int s = w / W, wb = (w - s * W) * 32;
        while (bits) {
          const int i = wb + __ffs(bits) - 1;
          bits &= bits - 1;
          const int j = s * n + i;
          const int q1 = I.first_req[j];
          if (q1 == INT_MAX) continue;  // nobody asked
          I.first_req[j] = INT_MAX;     // ready for the next round
          const int64_t ac = I.adv_cost[j];
          uint32_t el = 0;  // eligible: OUT slots with cost == adv(j), in slot order
          for (uint32_t t = I.omask[j]; t; t &= t - 1) {
            const int jj = __ffs(t) - 1;
            if (I.scost[j * MC + jj] == ac) el |= 1u << jj;
          }
          if (!el) continue;
          I.mark_relay(j);
          if (s == 0) {  // the data node is the only requester of stage-0 relays
            const int32_t pslot = j * MC + __ffs(el) - 1;
            const int32_t rs = I.req_slot[Sn];
            I.src_down[-2 - rs] = pslot;
            I.up[pslot] = rs;
            changed = 1;
            continue;
          }
          if (__popc(el) == 1) {
            commit_grant(q1, j * MC + __ffs(el) - 1);
          } else {
            _Pragma("unroll 1") for (int qq = q1; qq < s * n && el; ++qq) {
              if (I.req_target[qq] != j) continue;
              commit_grant(qq, j * MC + __ffs(el) - 1);
              el &= el - 1;
            }
          }
        }
      }
      // D-sink: free SNK slots in index order to last-stage requesters in gid order (last warp:
      // the requesters and the free SNK slots are both taken 32 at a time with ballots)
      if (dsink_free && lane_w == nwarps - 1) {
        int next = 0, fcb = 0;
        uint32_t fm = 0;
        bool full = false;
        _Pragma("unroll 1") for (int q0 = (S - 1) * n; q0 < Sn && !full; q0 += 32) {
          const int q = q0 + lane;
          uint32_t m = __ballot_sync(0xffffffffu, q < Sn && I.req_target[q] == -1);
          while (m) {
            const int qq = q0 + __ffs(m) - 1;
            m &= m - 1;
            while (fm == 0u && next < M) {
              const int k = next + lane;
              fm = __ballot_sync(0xffffffffu, k < M && I.snk_up[k] == kNone);
              fcb = next;
              next += 32;
            }
            if (fm == 0u) { full = true; break; }
            const int k = fcb + __ffs(fm) - 1;
            fm &= fm - 1;
            if (lane == 0) {
              const int32_t rs = I.req_slot[qq];
              I.down[rs] = -2 - k;
              I.snk_up[k] = rs;
              I.deny[qq] = 0;
              I.mark_slot(rs);
              I.mark_relay(qq);
              changed = 1;
            }
          }
        }
      }
      T.sync();
      RMARK(5);
      // ---------- summaries of the relays R3 touched (R4 reads the post-R3 state) ----------
      {
        const int nr = *(volatile int*)&I.lcnt[1];
        _Pragma("unroll 1") for (int k = T.tid; k < nr; k += TPI) I.refresh(I.rlist[k]);
      }
      T.sync();
      RMARK(6);
      }  // !prev_quiet
      // ---------- R4 proposals by idle relays (post-R3 state) + R5 reservations ----------
      _Pragma("unroll 1") for (int p = T.tid; p < Sn; p += TPI) {
        int kind = K_NONE;
        int32_t x = kNone, y = kNone, z = kNone;
        int32_t t0 = -1, t1 = -1, t2 = -1, t3 = -1;
        uint64_t key = RES_NONE;
        if (I.alive[p] && I.req_target[p] == -2) {
          const Summ sm{I.summ[p]};
          const int s = I.dn.div(p), i = p - s * n;
          if (sm.has_in()) {  // DENY after deny_after idle rounds holding unpaired inflow
            const int dw = I.deny[p] + 1;
            I.deny[p] = dw;
            if (dw >= P.deny_after) {
              kind = K_DENY;
              x = p * MC + sm.first_in();
              t0 = x;
              t1 = I.res_up(I.up[x]);
              key = (uint64_t)p;  // delta = -inf
            }
          } else if (n >= 2) {
            uint32_t qi = pick(I.h(p, 0), (uint32_t)(n - 1));
            if ((int)qi >= i) qi += 1;
            const int q = s * n + (int)qi;
            const int nq = I.alive[q] ? Summ{I.summ[q]}.npaired() : 0;
            if (nq > 0) {
              int64_t delta = 0;
              bool ok = false;
              if (sm.first_free() != 63 && !sm.has_out()) {  // Request Redirect
                y = I.nth_paired_m(q, (int)pick(I.h(p, 2), (uint32_t)nq));
                const int a = I.up[y] >= 0 ? I.relay(I.up[y]) : -1;
                const int c = I.down[y] >= 0 ? I.relay(I.down[y]) : -1;
                // the existing links a -> q and q -> c are y's up / down links (stored costs)
                const int64_t dax = I.d(a, p), dxc = I.d(p, c);
                const int64_t dab = I.up[y] >= 0 ? cst(I.lcd[I.up[y]]) : I.d(a, q), dbc = cst(I.lcd[y]);
                if (dax != INF && dxc != INF && dab != INF && dbc != INF) {
                  delta = P.objective == 0 ? (dax + dxc) - (dab + dbc) : max(dax, dxc) - max(dab, dbc);
                  kind = K_REDIRECT;
                  z = p * MC + sm.first_free();
                  t0 = y; t1 = I.res_up(I.up[y]); t2 = I.res_dn(I.down[y]); t3 = z;
                  ok = true;
                }
              } else if (sm.npaired() > 0) {  // Request Change
                x = I.nth_paired_m(p, (int)pick(I.h(p, 1), (uint32_t)sm.npaired()));
                y = I.nth_paired_m(q, (int)pick(I.h(p, 2), (uint32_t)nq));
                const int j1 = I.down[x] >= 0 ? I.relay(I.down[x]) : -1;
                const int j2 = I.down[y] >= 0 ? I.relay(I.down[y]) : -1;
                if (j1 != j2) {
                  // p -> j1 and q -> j2 are the existing links of x and y (stored costs)
                  const int64_t a1 = I.d(p, j2), a2 = I.d(q, j1), b1 = cst(I.lcd[x]), b2 = cst(I.lcd[y]);
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
                  accept = (I.h(p, 3) >> 32) < (uint64_t)P.thr[(size_t)kk * P.thr_width + delta];
                }
                if (accept) key = ((uint64_t)(delta + (1ll << 40)) << 22) | (uint64_t)p;
                else kind = K_NONE;
              }
            }
          }
        }
        if (key == RES_NONE) kind = K_NONE;
        I.prop[p * 4 + 0] = kind;
        if (kind != K_NONE) {
          I.prop[p * 4 + 1] = x;
          I.prop[p * 4 + 2] = y;
          I.prop[p * 4 + 3] = z;
          I.pkey[p] = key;
          I.ptouch[p * 4 + 0] = t0;
          I.ptouch[p * 4 + 1] = t1;
          I.ptouch[p * 4 + 2] = t2;
          I.ptouch[p * 4 + 3] = t3;
          atomicMin((unsigned long long*)&I.res[t0], (unsigned long long)key);
          atomicMin((unsigned long long*)&I.res[t1], (unsigned long long)key);
          if (t2 >= 0) atomicMin((unsigned long long*)&I.res[t2], (unsigned long long)key);
          if (t3 >= 0) atomicMin((unsigned long long*)&I.res[t3], (unsigned long long)key);
        }
      }
      T.sync();
      RMARK(7);
      // ---------- R6 commit the proposals that hold every slot they touch ----------
      _Pragma("unroll 1") for (int p = T.tid; p < Sn; p += TPI) {
        const int kind = I.prop[p * 4 + 0];
        if (kind == K_NONE) continue;
        const uint64_t key = I.pkey[p];
        bool win = true;
        _Pragma("unroll 1") for (int q = 0; q < 4; ++q) {
          const int32_t t = I.ptouch[p * 4 + q];
          if (t >= 0) win = win && ld_res<kSmem>(&I.res[t]) == key;
        }
        if (!win) continue;
        const int32_t x = I.prop[p * 4 + 1], y = I.prop[p * 4 + 2], z = I.prop[p * 4 + 3];
        // every slot whose down pointer changes is marked (its cost and the costs above it are
        // brought up to date at the next round's start); relays whose slot states change are listed
        if (kind == K_CHANGE) {
          const int32_t dx = I.down[x], dy = I.down[y];
          I.down[x] = dy;
          I.down[y] = dx;
          I.set_up_of(dy, x);
          I.set_up_of(dx, y);
          I.kacc[p] += 1;
          I.mark_slot(x);
          I.mark_slot(y);
        } else if (kind == K_REDIRECT) {
          const int32_t a = I.up[y], c = I.down[y];
          I.up[z] = a;
          I.down[z] = c;
          I.set_down_of(a, z);
          I.set_up_of(c, z);
          I.up[y] = kNone;
          I.down[y] = kNone;
          I.kacc[p] += 1;
          I.mark_slot(z);
          I.mark_slot(y);
          I.mark_slot(a);
          I.mark_relay(p);
          I.mark_relay(I.relay(y));
        } else {
          const int32_t a = I.up[x];
          I.up[x] = kNone;
          I.set_down_of(a, kNone);
          I.deny[p] = 0;
          I.mark_slot(a);
          I.mark_relay(p);
          if (a >= 0) I.mark_relay(I.relay(a));
        }
        changed = 1;
      }
      T.sync();
      RMARK(8);
      _Pragma("unroll 1") for (int p = T.tid; p < Sn; p += TPI) {  // release the reservations for the next round
        if (I.prop[p * 4 + 0] == K_NONE) continue;
        _Pragma("unroll 1") for (int q = 0; q < 4; ++q) {
          const int32_t t = I.ptouch[p * 4 + q];
          if (t >= 0) st_res<kSmem>(&I.res[t], RES_NONE);
        }
      }
      // ---------- R7 ----------
      const int any = T.sync_or(changed);
      RMARK(9);
      quiet = any ? 0 : quiet + 1;
      prev_quiet = !any;
      round += 1;
      if (o.digests) {
        if (T.tid == 0) sh_u64[0] = 0;
        T.sync();
        uint64_t acc = 0;
        const int nslot = Sn * MC;
        _Pragma("unroll 1") for (int p = T.tid; p < nslot; p += TPI) {
          const int32_t u = I.up[p], dn = I.down[p];
          const uint64_t eu = u == kNone ? 0 : (u >= 0 ? 1 + (uint64_t)u : (1ull << 40) + (uint64_t)(-2 - u));
          const uint64_t ed = dn == kNone ? 0 : (dn >= 0 ? 1 + (uint64_t)dn : (1ull << 41) + (uint64_t)(-2 - dn));
          const uint64_t state = (u != kNone ? 2 : 0) | (dn != kNone ? 1 : 0);
          acc += digest_elem(3ull * p, state) + digest_elem(3ull * p + 1, eu) + digest_elem(3ull * p + 2, ed);
        }
        const uint64_t b1 = 3ull * nslot, b2 = b1 + M, b3 = b2 + M, b4 = b3 + 2ull * Sn;
        _Pragma("unroll 1") for (int k = T.tid; k < M; k += TPI) {
          const int32_t sd = I.src_down[k], su = I.snk_up[k];
          acc += digest_elem(b1 + k, sd == kNone ? 0 : 1 + (uint64_t)sd);
          acc += digest_elem(b2 + k, su == kNone ? 0 : 1 + (uint64_t)su);
        }
        _Pragma("unroll 1") for (int v = T.tid; v < Sn; v += TPI) {
          acc += digest_elem(b3 + 2ull * v, (uint64_t)(uint32_t)I.kacc[v]);
          acc += digest_elem(b3 + 2ull * v + 1, (uint64_t)(uint32_t)I.deny[v]);
        }
        if (T.tid == 0) acc += digest_elem(b4, (uint64_t)(uint32_t)quiet);
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) atomicAdd(&sh_u64[0], (unsigned long long)acc);
        T.sync();
        if (T.tid == 0) o.digests[(size_t)b * o.max_rounds + r] = *(volatile unsigned long long*)&sh_u64[0];
      }
      ++r;
      if (quiet >= P.W) break;
    }
#undef RMARK
#undef WSTAT
    if (o.digests)
      _Pragma("unroll 1") for (int k = r + T.tid; k < o.max_rounds; k += TPI) o.digests[(size_t)b * o.max_rounds + k] = 0;
    // ---------- results: complete SRC -> SNK chains and dangling outflows ----------
    if (T.tid == 0) { sh_u64[0] = 0; sh_u64[1] = 0; sh_i32[3] = 0; }
    T.sync();
    {
      unsigned long long f = 0, c = 0;
      _Pragma("unroll 1") for (int k = T.tid; k < M; k += TPI) {
        int32_t p = I.src_down[k];
        if (p == kNone) continue;
        int64_t cc = cst(I.src[I.relay(p)]);
        int guard = 0;
        bool ok = true;
        while (p >= 0 && ++guard <= S + 1) {
          const int32_t nx = I.down[p];
          if (nx == kNone) { ok = false; break; }
          cc = sadd(cc, I.d(I.relay(p), nx <= -2 ? -1 : I.relay(nx)));
          p = nx;
        }
        if (ok && p <= -2 && cc != INF) { f += 1; c += (unsigned long long)cc; }
      }
      int dg = 0;
      _Pragma("unroll 1") for (int p = T.tid; p < Sn * MC; p += TPI) dg += I.st(p) == ST_OUT;
      for (int off = 16; off > 0; off >>= 1) {
        f += __shfl_xor_sync(0xffffffffu, f, off);
        c += __shfl_xor_sync(0xffffffffu, c, off);
        dg += __shfl_xor_sync(0xffffffffu, dg, off);
      }
      if (lane == 0) {
        atomicAdd(&sh_u64[0], f);
        atomicAdd(&sh_u64[1], c);
        atomicAdd(&sh_i32[3], dg);
      }
    }
    T.sync();
    if constexpr (kSmem) {
      _Pragma("unroll 1") for (int k = T.tid; k < Sn * MC; k += TPI) { g_up[k] = I.up[k]; g_down[k] = I.down[k]; }
      _Pragma("unroll 1") for (int k = T.tid; k < M; k += TPI) { g_src_down[k] = I.src_down[k]; g_snk_up[k] = I.snk_up[k]; }
      _Pragma("unroll 1") for (int k = T.tid; k < Sn; k += TPI) { g_kacc[k] = I.kacc[k]; g_deny[k] = I.deny[k]; }
    }
    if (T.tid == 0) {
      if (o.rounds_run) o.rounds_run[b] = r;
      if (o.F_dec) o.F_dec[b] = (int64_t)*(volatile unsigned long long*)&sh_u64[0];
      if (o.cost_dec) o.cost_dec[b] = (int64_t)*(volatile unsigned long long*)&sh_u64[1];
      if (o.dangling) o.dangling[b] = *(volatile int*)&sh_i32[3];
      P.quiet[b] = quiet;
      P.round[b] = (int64_t)round;
    }
    T.sync();
  }
}

template <int TPI, bool kSmem>
__global__ void __launch_bounds__(256, 4) rounds_kernel(const Problem P, const RoundsOut o, const size_t ws_bytes) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ unsigned long long sh_u64[8][2];
  __shared__ int sh_i32[8][4];
  __shared__ int sh_inst[8];
  __shared__ int tma_init[8];
  __shared__ uint32_t tma_phase_of[8];
  if (threadIdx.x < 8) { tma_init[threadIdx.x] = 0; tma_phase_of[threadIdx.x] = 0; }
  __syncthreads();
  TeamOf<TPI> T{{(int)(threadIdx.x % TPI), (int)(threadIdx.x / TPI)}, (int)(threadIdx.x % TPI), (int)(threadIdx.x / TPI)};
  const int teams_per_cta = blockDim.x / TPI;
  uint8_t* base = kSmem ? dsm + (size_t)T.id * ws_bytes
                        : P.ws_rounds + (size_t)(blockIdx.x * teams_per_cta + T.id) * ws_bytes;
  rounds_body<TeamOf<TPI>, kSmem>(P, o, ws_bytes, T, base, Red{sh_u64[T.id], sh_i32[T.id], &sh_inst[T.id]}, dsm,
                                  tma_init, tma_phase_of);
}

// cluster tier of the rounds: one cluster of C CTAs x 1,024 threads per instance, state and
// scratch in the global workspace (one per cluster; its last 64 bytes hold the reduction cells)
template <int C>
__global__ void __launch_bounds__(1024, 1) rounds_cluster_kernel(const Problem P, const RoundsOut o, const size_t ws_bytes) {
  __shared__ uint32_t vslot[2];
  if (threadIdx.x < 2) vslot[threadIdx.x] = 0;
  cg::cluster_group cl = cg::this_cluster();
  ClusterTeam<C> T{(int)(cl.block_rank() * 1024 + threadIdx.x), 0, vslot, 0u};
  uint8_t* base = P.ws_rounds + (size_t)(blockIdx.x / C) * ws_bytes;
  uint8_t* cells = base + rounds_layout(P, false).cells;
  cl.sync();
  rounds_body<ClusterTeam<C>, false>(P, o, ws_bytes, T, base,
                                     Red{(unsigned long long*)cells, (int*)(cells + 16), (int*)(cells + 32)},
                                     nullptr, nullptr, nullptr);
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
cudaError_t launch_rounds_tpi(const Problem& P, const RoundsOut& o, cudaStream_t st, int num_sms, bool smem) {
  const size_t ws = rounds_layout(P, smem).total;
  const size_t limit = 200 * 1024;
  int teams = TPI >= 256 ? 1 : 256 / TPI;
  if (teams > 8) teams = 8;
  if (smem)
    while (teams > 1 && teams * ws > limit) --teams;
  const size_t dyn = smem ? teams * ws : 0;
  auto k = smem ? rounds_kernel<TPI, true> : rounds_kernel<TPI, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, teams * TPI, dyn);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  long long grid = (long long)per_sm * num_sms;
  const long long need = (P.B + teams - 1) / teams;
  if (grid > need) grid = need;
  if (!smem && grid * teams > P.ws_rounds_teams) grid = P.ws_rounds_teams / teams;
  if (grid < 1) grid = 1;
  k<<<(int)grid, teams * TPI, dyn, st>>>(P, o, ws);
  return cudaGetLastError();
}

template <int C>
cudaError_t launch_rounds_cluster(const Problem& P, const RoundsOut& o, cudaStream_t st, int* ncl_out, bool query) {
  const size_t ws = rounds_layout(P, false).total;
  auto k = rounds_cluster_kernel<C>;
  cudaError_t e;
  if (C > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(1024);
  cfg.gridDim = dim3(C);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
  if (e != cudaSuccess) return e;
  if (ncl < 1) return cudaErrorInvalidConfiguration;
  if (ncl > P.B) ncl = P.B;
  if (ncl > P.ws_rounds_teams) ncl = P.ws_rounds_teams;
  if (ncl_out) *ncl_out = ncl;
  if (query) return cudaSuccess;
  cfg.gridDim = dim3(ncl * C);
  return cudaLaunchKernelEx(&cfg, k, P, o, ws);
}

// instances with more relay slots than a 256-thread team handles well run on clusters
bool rounds_use_cluster(const Problem& P) {
  const int f = getenv_int("GWTF_ROUNDS_CLUSTER", -1);
  if (f >= 0) return f > 0;
  return (long long)P.S * P.n * std::max(P.MC, 1) > 32768;
}

// cluster size of the rounds: smallest waves x (relays per thread + fixed barrier cost)
int rounds_cluster_size(const Problem& P) {
  if (const char* f = getenv("GWTF_ROUNDS_CLUSTER_SIZE")) return atoi(f);
  if (P.rounds_cluster_pref > 0) return P.rounds_cluster_pref;
  int best = 0;
  long long best_cost = 0;
  for (int C : {16, 8, 4, 2}) {
    int ncl = 0;
    cudaError_t e = C == 16 ? launch_rounds_cluster<16>(P, RoundsOut{}, nullptr, &ncl, true)
                  : C == 8  ? launch_rounds_cluster<8>(P, RoundsOut{}, nullptr, &ncl, true)
                  : C == 4  ? launch_rounds_cluster<4>(P, RoundsOut{}, nullptr, &ncl, true)
                            : launch_rounds_cluster<2>(P, RoundsOut{}, nullptr, &ncl, true);
    if (e != cudaSuccess || ncl < 1) { cudaGetLastError(); continue; }
    const long long waves = (P.B + ncl - 1) / ncl;
    const long long per = ((long long)P.S * P.n + C * 1024 - 1) / (C * 1024);
    const long long cost = waves * (per + 2);
    if (best == 0 || cost < best_cost) { best = C; best_cost = cost; }
  }
  return best;
}

}  // namespace

size_t rounds_ws_bytes(const Problem& P, bool smem) { return rounds_layout(P, smem).total; }

int rounds_tpi(const Problem& P) {
  const int Sn = P.S * P.n;
  const int tpi = Sn <= 32 ? 32 : Sn <= 64 ? 64 : Sn <= 128 ? 128 : 256;  // ~one relay per thread
  return getenv_int("GWTF_ROUNDS_TPI", tpi);
}

bool rounds_use_smem(const Problem& P) {
  return rounds_layout(P, true).total <= 200 * 1024 && getenv_int("GWTF_ROUNDS_GLOBAL", 0) == 0;
}

cudaError_t launch_init_round_state(const Problem& P, cudaStream_t st) {
  init_round_state_kernel<<<148 * 4, 256, 0, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_rounds(const Problem& P0, const RoundsOut& o, cudaStream_t st, int num_sms) {
  Problem P = P0;
  P.rounds_cost_mode = getenv_int("GWTF_ROUNDS_COSTS", 0);
  cudaError_t e = cudaMemsetAsync(P.counters + 1, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const int tpi = rounds_tpi(P);
  const bool smem = rounds_use_smem(P);
  if (!smem && rounds_use_cluster(P)) {
    const int C = rounds_cluster_size(P);
    if (C == 16) return launch_rounds_cluster<16>(P, o, st, nullptr, false);
    if (C == 8) return launch_rounds_cluster<8>(P, o, st, nullptr, false);
    if (C == 4) return launch_rounds_cluster<4>(P, o, st, nullptr, false);
    if (C == 2) return launch_rounds_cluster<2>(P, o, st, nullptr, false);
  }
  if (tpi <= 32) return launch_rounds_tpi<32>(P, o, st, num_sms, smem);
  if (tpi <= 64) return launch_rounds_tpi<64>(P, o, st, num_sms, smem);
  if (tpi <= 128) return launch_rounds_tpi<128>(P, o, st, num_sms, smem);
  return launch_rounds_tpi<256>(P, o, st, num_sms, smem);
}

}  // namespace gwtf
