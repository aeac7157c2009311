// Warm-start rerouting after churn (PAPER.md:188 reroute after a failure,
// :274-288 crash handling).  Starting from a pre-churn assignment (dense layouts of
// gwtf_flow_get_assignment), on the handle's current (churned) graph:
//   1. strip the units the churned graph cannot carry (dead relay, relay over capacity, link /
//      src / snk arc now ABSENT), one unit path at a time;
//   2. cancel negative residual cycles: Bellman-Ford from a virtual root, a change in pass N
//      proves a cycle, the predecessor walk extracts it and its bottleneck is pushed;
//   3. resume successive shortest paths (Bellman-Ford from s*, signed costs) until F = M or t*
//      is unreachable.
// One CTA per instance (grid-stride over the batch).  A pass relaxes every residual arc of the
// node-split stage graph in parallel; a node's label is one 64-bit word, biased distance << 24 |
// residual-arc id, lowered with atomicMin, so a label and its predecessor are always consistent
// (every cycle of the predecessor graph is then negative).  Labels live in a per-instance global
// scratch row (L1/L2 resident for the shapes this serves).  The flow arrays are updated in place.
//
// Arc numbering (forward arc e; residual arc r = 2e forward, 2e+1 backward):
//   e in [0, n)                      src arc     D -> in(0,i)         cap M, cost src[i]
//   e in [n, n+Sn)                   relay arc   in(s,i) -> out(s,i)  cap alive ? cap : 0, cost 0
//   e in [n+Sn, n+Sn+(S-1)n^2)       link arc    out(s,u) -> in(s+1,v) (dest-major s,v,u), cap M
//   e in [n+Sn+(S-1)n^2, E)          snk arc     out(S-1,i) -> D      cap M, cost snk[i]
// Nodes: 0 = s*, 1 = t*, in(s,i) = 2 + 2(s n + i), out(s,i) = in(s,i) + 1.
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>

#include "gwtf_internal.h"

namespace gwtf {

namespace {

constexpr int kThreads = 256;
constexpr int32_t kDeferred = 80;  // status: the instance is re-solved cold (triage or failed repair)
constexpr int kStripList = 256;  // over-capacity arcs listed per instance (more: thread 0 rescans all)
constexpr int kArcBits = 24;
constexpr uint64_t kNoPred = (1ull << kArcBits) - 1;
constexpr int64_t kBias = 1ll << 38;  // |distance| < 2^38 (checked per relaxation)
constexpr uint64_t kLabInf = ~0ull;

struct WarmCtx {
  int S, n, ld, N;
  int64_t E, M;
  const int32_t* tile;   // [S-1][n][ld]
  const int32_t* src;
  const int32_t* snk;
  const int32_t* cap;
  const uint8_t* alive;
  const uint8_t* alive_prev;  // before the last churn: a node arc of a relay alive now and dead then is new
  int32_t* src_f;        // [n]
  int32_t* g;            // [S][n]
  int32_t* arc;          // [S-1][n][n]
  int32_t* snk_f;        // [n]
};

struct ArcV { int from, to; int64_t cap, cost; int32_t* x; };

__device__ __forceinline__ int in_node(const WarmCtx& c, int s, int i) { return 2 + 2 * (s * c.n + i); }

__device__ ArcV arc_of(const WarmCtx& c, int64_t e) {
  ArcV a;
  const int n = c.n, Sn = c.S * c.n;
  if (e < n) {
    const int32_t w = c.src[e];
    a = {0, in_node(c, 0, (int)e), w == kAbsent ? 0 : c.M, w == kAbsent ? 0 : (int64_t)w, c.src_f + e};
  } else if (e < n + Sn) {
    const int k = (int)(e - n);
    a = {2 + 2 * k, 3 + 2 * k, c.alive[k] ? (int64_t)c.cap[k] : 0, 0, c.g + k};
  } else if (e < n + Sn + (int64_t)(c.S - 1) * n * n) {
    const int k = (int)(e - n - Sn);  // < 2^23 (checked by the host)
    const int q = k / n, u = k - q * n, s = q / n, v = q - s * n;
    const int32_t w = c.tile[((size_t)s * n + v) * c.ld + u];
    a = {in_node(c, s, u) + 1, in_node(c, s + 1, v), w == kAbsent ? 0 : c.M, w == kAbsent ? 0 : (int64_t)w, c.arc + k};
  } else {
    const int i = (int)(e - n - Sn - (int64_t)(c.S - 1) * n * n);
    const int32_t w = c.snk[i];
    a = {in_node(c, c.S - 1, i) + 1, 1, w == kAbsent ? 0 : c.M, w == kAbsent ? 0 : (int64_t)w, c.snk_f + i};
  }
  return a;
}

// the id of the idx-th forward arc in layer order: src arcs, then per stage s its node arcs and
// (s < S-1) its outgoing link arcs, then the snk arcs -- a pass over the arcs in this order (or in
// reverse) carries a label update through every stage at once
__device__ __forceinline__ int64_t layered_arc(const WarmCtx& c, int64_t idx) {
  const int n = c.n;
  if (idx < n) return idx;
  idx -= n;
  const int64_t blk = (int64_t)n + (int64_t)n * n;  // one stage: n node arcs + n^2 link arcs
  const int64_t full = (int64_t)(c.S - 1) * blk;
  if (idx < full) {
    const int64_t s = idx / blk, r = idx - s * blk;
    return r < n ? n + s * n + r : n + (int64_t)c.S * n + s * n * n + (r - n);
  }
  idx -= full;
  if (idx < n) return n + (int64_t)(c.S - 1) * n + idx;  // node arcs of the last stage
  return idx - n + n + (int64_t)c.S * n + (int64_t)(c.S - 1) * n * n;  // snk arcs
}

// labels are lowered by global atomics (performed at L2): read them around the L1
__device__ __forceinline__ uint64_t ld_lab(const uint64_t* p) { return *(const volatile uint64_t*)p; }
__device__ __forceinline__ int64_t lab_dist(uint64_t L) { return (int64_t)(L >> kArcBits) - kBias; }
__device__ __forceinline__ int lab_pred(uint64_t L) { return (int)(L & kNoPred); }
__device__ __forceinline__ uint64_t lab(int64_t d, uint64_t r) { return ((uint64_t)(d + kBias) << kArcBits) | r; }

// residual arc r -> (from, to, rcap, rcost, x, sign)
__device__ __forceinline__ void res_of(const WarmCtx& c, int64_t r, int& from, int& to, int64_t& rcap, int64_t& rcost,
                                       int32_t*& x, int& sign) {
  const ArcV a = arc_of(c, r >> 1);
  x = a.x;
  if (r & 1) { from = a.to; to = a.from; rcap = *a.x; rcost = -a.cost; sign = -1; }
  else { from = a.from; to = a.to; rcap = a.cap - *a.x; rcost = a.cost; sign = 1; }
}

// One team-wide Bellman-Ford pass over every residual arc.  Returns (block-uniform) whether
// some label changed; *last = a node lowered in this pass.
__device__ bool bf_pass(const WarmCtx& c, uint64_t* labv, int* last, int* changed_sm, int* bad_sm) {
  if (threadIdx.x == 0) *changed_sm = 0;
  __syncthreads();
  int ch = 0;
  for (int64_t r = threadIdx.x; r < 2 * c.E; r += blockDim.x) {
    int from, to, sign;
    int64_t rcap, rcost;
    int32_t* x;
    res_of(c, r, from, to, rcap, rcost, x, sign);
    if (rcap <= 0) continue;
    const uint64_t Lf = ld_lab(&labv[from]);
    if (Lf == kLabInf) continue;
    const int64_t d = lab_dist(Lf) + rcost;
    if (d >= kBias || d <= -kBias) { *bad_sm = 1; continue; }
    const uint64_t cand = lab(d, (uint64_t)r);
    if ((cand >> kArcBits) < (ld_lab(&labv[to]) >> kArcBits)) {
      const uint64_t old = atomicMin((unsigned long long*)&labv[to], (unsigned long long)cand);
      if ((cand >> kArcBits) < (old >> kArcBits)) { ch = 1; *last = to; }
    }
  }
  if (ch) *changed_sm = 1;
  __syncthreads();
  const bool any = *changed_sm != 0;
  __syncthreads();
  return any;
}

// thread 0: remove one unit along a flow path through forward arc e (lowest index upstream and
// downstream).  A conserved flow has a carrying arc on each side of every interior node; false
// if the given assignment is not conserved.
__device__ bool strip_unit(const WarmCtx& c, int64_t e) {
  const int n = c.n, S = c.S;
  const ArcV a = arc_of(c, e);
  *a.x -= 1;
  for (int node = a.from; node != 0;) {  // upstream
    const int k = (node - 2) >> 1, s = k / n, i = k % n;
    if (node & 1) { c.g[k] -= 1; node = node - 1; continue; }  // out(s,i) <- relay arc
    if (s == 0) { c.src_f[i] -= 1; node = 0; continue; }
    int u = 0;
    while (u < n && c.arc[((size_t)(s - 1) * n + i) * n + u] <= 0) ++u;
    if (u == n) return false;
    c.arc[((size_t)(s - 1) * n + i) * n + u] -= 1;
    node = in_node(c, s - 1, u) + 1;
  }
  for (int node = a.to; node != 1;) {  // downstream
    const int k = (node - 2) >> 1, s = k / n, i = k % n;
    if (!(node & 1)) { c.g[k] -= 1; node = node + 1; continue; }  // in(s,i) -> relay arc
    if (s == S - 1) { c.snk_f[i] -= 1; node = 1; continue; }
    int v = 0;
    while (v < n && c.arc[((size_t)s * n + v) * n + i] <= 0) ++v;
    if (v == n) return false;
    c.arc[((size_t)s * n + v) * n + i] -= 1;
    node = in_node(c, s + 1, v);
  }
  return true;
}

// The general fallback (instances the potential-carrying repair cannot take: a negative residual
// cycle on the kept flow, i.e. some link got cheaper; status 7 from warm_kernel): strip, cancel
// negative cycles (Klein), resume SSP.
__global__ void __launch_bounds__(kThreads) klein_kernel(const Problem P, int32_t* src_f_all, int32_t* g_all,
                                                         int32_t* arc_all, int32_t* snk_f_all, uint64_t* lab_all,
                                                         int32_t* stamp_all, int64_t* F_out, int64_t* cost_out,
                                                         int64_t* stats_out, int32_t* status_out) {
  __shared__ int changed_sm, bad_sm, last_sm, cyc_sm, strip_n;
  __shared__ int strip_list[kStripList];
  __shared__ unsigned long long cost_sm;
  const int S = P.S, n = P.n;
  const int N = 2 + 2 * S * n;
  const int64_t E = 2ll * n + (int64_t)S * n + (int64_t)(S - 1) * n * n;
  for (int b = blockIdx.x; b < P.B; b += gridDim.x) {
    if (status_out[b] != 7 && (status_out[b] < 70 || status_out[b] > 79)) continue;  // solved by the repair
    WarmCtx c;
    c.S = S; c.n = n; c.ld = P.ld; c.N = N; c.E = E; c.M = P.supply[b];
    c.tile = P.tile + (size_t)b * (S - 1) * n * P.ld;
    c.src = P.src + (size_t)b * n;
    c.snk = P.snk + (size_t)b * n;
    c.cap = P.cap + (size_t)b * S * n;
    c.alive = P.alive + (size_t)b * S * n;
    c.src_f = src_f_all + (size_t)b * n;
    c.g = g_all + (size_t)b * S * n;
    c.arc = arc_all + (size_t)b * (S - 1) * n * n;
    c.snk_f = snk_f_all + (size_t)b * n;
    uint64_t* labv = lab_all + (size_t)blockIdx.x * N;
    int32_t* stamp = stamp_all + (size_t)blockIdx.x * N;
    int64_t stripped = 0, cycles = 0, augment = 0;
    int status = 0;
    // ---- 1. strip: the team finds the over-capacity arcs, thread 0 strips their units ----
    // (stripping only lowers flows, so an arc within capacity before the strip stays so)
    if (threadIdx.x == 0) { bad_sm = 0; strip_n = 0; }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      const ArcV a = arc_of(c, e);
      if (*a.x > a.cap) {
        const int slot = atomicAdd(&strip_n, 1);
        if (slot < kStripList) strip_list[slot] = (int)e;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && strip_n > 0) {
      const bool listed = strip_n <= kStripList;
      const int64_t cnt = listed ? strip_n : E;
      for (int64_t j = 0; j < cnt; ++j) {
        const int64_t e = listed ? strip_list[j] : j;
        const ArcV a = arc_of(c, e);
        while (!bad_sm && *a.x > a.cap) {
          if (!strip_unit(c, e)) bad_sm = 4;
          ++stripped;
        }
      }
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x) stamp[k] = -1;
    __syncthreads();
    // ---- 2. negative-cycle cancelling ----
    // Labels are not reset after a cancel: whatever their history, a pass that lowers nothing
    // leaves labels that are feasible potentials of the current residual graph, which proves that
    // no negative cycle is left.  A predecessor cycle found on stale labels is checked (every arc
    // still residual, negative total) before it is pushed; 2N + 8 passes without a usable cycle
    // since the last cancel restart the labels from zero (fresh labels: every predecessor cycle is
    // negative and residual).
    {
      int walk_id = 0, since = 0;
      bool fresh = true;
      for (int k = threadIdx.x; k < N; k += blockDim.x) labv[k] = lab(0, kNoPred);
      __syncthreads();
      while (!bad_sm) {
        const bool ch = bf_pass(c, labv, &last_sm, &changed_sm, &bad_sm);
        if (!ch) break;
        ++since;
        if (threadIdx.x == 0) {  // walk the predecessors of a lowered node; cancel a usable cycle
          ++walk_id;
          int x = last_sm;
          while (stamp[x] != walk_id) {
            stamp[x] = walk_id;
            const int r = lab_pred(ld_lab(&labv[x]));
            if (r == (int)kNoPred) { x = -1; break; }
            int from, to, sign; int64_t rcap, rcost; int32_t* xp;
            res_of(c, r, from, to, rcap, rcost, xp, sign);
            x = from;
          }
          cyc_sm = 0;
          if (x >= 0) {
            const int x0 = x;
            int64_t bott = INT64_MAX, ccost = 0;
            do {
              int from, to, sign; int64_t rcap, rcost; int32_t* xp;
              res_of(c, lab_pred(ld_lab(&labv[x])), from, to, rcap, rcost, xp, sign);
              bott = rcap < bott ? rcap : bott;
              ccost += rcost;
              x = from;
            } while (x != x0);
            if (bott > 0 && ccost < 0) {
              do {
                int from, to, sign; int64_t rcap, rcost; int32_t* xp;
                res_of(c, lab_pred(ld_lab(&labv[x])), from, to, rcap, rcost, xp, sign);
                *xp += (int32_t)(sign * bott);
                x = from;
              } while (x != x0);
              cyc_sm = 1;
            } else if (fresh) {
              bad_sm = 5;  // cannot happen on fresh labels; never loop on it
            }
          }
        }
        __syncthreads();
        if (cyc_sm) {
          ++cycles;
          since = 0;
          fresh = false;
        } else if (since > (fresh ? 4 * N + 8 : 2 * N + 8)) {
          if (fresh) {
            if (threadIdx.x == 0) bad_sm = 2;
          } else {
            for (int k = threadIdx.x; k < N; k += blockDim.x) labv[k] = lab(0, kNoPred);
            since = 0;
            fresh = true;
          }
        }
        __syncthreads();
      }
    }
    // ---- 3. successive shortest paths from the cancelled flow ----
    int64_t F = 0;
    for (int i = 0; i < n; ++i) F += c.src_f[i];
    while (!bad_sm && F < c.M) {
      for (int k = threadIdx.x; k < N; k += blockDim.x) labv[k] = k == 0 ? lab(0, kNoPred) : kLabInf;
      __syncthreads();
      for (int pass = 0; bf_pass(c, labv, &last_sm, &changed_sm, &bad_sm); ++pass)
        if (pass > N) { if (threadIdx.x == 0) bad_sm = 3; __syncthreads(); break; }
      if (bad_sm || ld_lab(&labv[1]) == kLabInf) break;
      if (threadIdx.x == 0) {
        int64_t bott = c.M - F;
        for (int x = 1; x != 0;) {
          int from, to, sign; int64_t rcap, rcost; int32_t* xp;
          res_of(c, lab_pred(ld_lab(&labv[x])), from, to, rcap, rcost, xp, sign);
          bott = rcap < bott ? rcap : bott;
          x = from;
        }
        for (int x = 1; x != 0;) {
          int from, to, sign; int64_t rcap, rcost; int32_t* xp;
          res_of(c, lab_pred(ld_lab(&labv[x])), from, to, rcap, rcost, xp, sign);
          *xp += (int32_t)(sign * bott);
          x = from;
        }
        changed_sm = (int)(bott > 0x7fffffff ? 0x7fffffff : bott);
      }
      __syncthreads();
      F += changed_sm;
      ++augment;
      __syncthreads();
    }
    status = bad_sm;
    // ---- objective of the repaired assignment ----
    if (threadIdx.x == 0) cost_sm = 0;
    __syncthreads();
    long long part = 0;
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      const ArcV a = arc_of(c, e);
      part += (long long)*a.x * a.cost;
    }
    atomicAdd(&cost_sm, (unsigned long long)part);
    __syncthreads();
    if (threadIdx.x == 0) {
      F_out[b] = F;
      cost_out[b] = (int64_t)cost_sm;
      if (stats_out) { stats_out[3 * b] = stripped; stats_out[3 * b + 1] = cycles; stats_out[3 * b + 2] = augment; }
      status_out[b] = status;  // 5 = non-negative cycle (never expected)
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------------------------
// Potential-carrying repair (the default path).  The pre-churn assignment is optimal for the old
// graph, so its residual graph has no negative cycle; a crash, a dropped link or a raised cost
// only removes residual arcs or lowers flows on removed arcs, so the kept part has none either.
//   P. potentials pi: Bellman-Ford from a virtual root over the residual arcs of the kept flow
//      (x' = min(x, cap) on every arc), leaving out the node arcs of rejoined relays (new arcs;
//      alive now, dead before the churn) and the bypass; no convergence within N + 2 passes = a
//      negative cycle (some cost was lowered): status 7, the instance goes to klein_kernel untouched;
//   C. cut: every arc carrying more than its new capacity (dead relay, absent link / src / snk)
//      drops the excess units, which leaves imbalances at its two ends -- the flow is not
//      stripped along whole paths, it is rerouted around the cut ("reroute");
//   V. a rejoined relay's node arc with a negative reduced cost (a shortcut) is saturated;
//   A. successive shortest paths on reduced costs (all >= 0) from the excess nodes to the deficit
//      nodes (multi-source Bellman-Ford, nearest deficit node, bottleneck augment, pi += min(d,
//      d_target)), until balanced; a unit that cannot be rerouted goes back through the bypass
//      s* -> t* (cost BIG > any simple path: the lexicographic max-flow device of SURVEY C3 i);
//   B. successive shortest paths s* -> t* on the real arcs while the bypass still carries units.
//   The result is a min-cost flow of maximum value on the churned graph: (F, cost) equal the cold
//   solve's.  Without churn nothing is cut or saturated and B finds no path: the identity.
// Bypass residual arcs: r = 2E (s* -> t*, cap M - byp, cost BIG) and 2E + 1 (t* -> s*, cap byp).
__device__ __forceinline__ void res2(const WarmCtx& c, int64_t r, int64_t byp, int64_t big, int& from, int& to,
                                     int64_t& rcap, int64_t& rcost, int32_t*& x, int& sign) {
  if (r >= 2 * c.E) {
    x = nullptr;
    if (r == 2 * c.E) { from = 0; to = 1; rcap = c.M - byp; rcost = big; sign = 1; }
    else { from = 1; to = 0; rcap = byp; rcost = -big; sign = -1; }
    return;
  }
  res_of(c, r, from, to, rcap, rcost, x, sign);
}

__global__ void __launch_bounds__(kThreads) warm_kernel(const Problem P, int32_t* src_f_all, int32_t* g_all,
                                                        int32_t* arc_all, int32_t* snk_f_all, uint64_t* lab_all,
                                                        int64_t* pi_all, int32_t* imb_all, int64_t* F_out,
                                                        int64_t* cost_out, int64_t* stats_out, int32_t* status_out) {
  __shared__ int changed_sm, bad_sm, last_sm;
  __shared__ unsigned long long best_sm, cost_sm;
  __shared__ long long byp_sm, delta_sm;
  __shared__ int any_sm;
  const int S = P.S, n = P.n;
  const int N = 2 + 2 * S * n;
  const int64_t E = 2ll * n + (int64_t)S * n + (int64_t)(S - 1) * n * n;
  const int64_t NR = 2 * E + 2;  // residual arcs incl. the bypass pair
  for (int b = blockIdx.x; b < P.B; b += gridDim.x) {
    if (status_out[b] == kDeferred) continue;  // triage: left to the cold solve
    WarmCtx c;
    c.S = S; c.n = n; c.ld = P.ld; c.N = N; c.E = E; c.M = P.supply[b];
    c.tile = P.tile + (size_t)b * (S - 1) * n * P.ld;
    c.src = P.src + (size_t)b * n;
    c.snk = P.snk + (size_t)b * n;
    c.cap = P.cap + (size_t)b * S * n;
    c.alive = P.alive + (size_t)b * S * n;
    c.alive_prev = P.alive_prev + (size_t)b * S * n;
    c.src_f = src_f_all + (size_t)b * n;
    c.g = g_all + (size_t)b * S * n;
    c.arc = arc_all + (size_t)b * (S - 1) * n * n;
    c.snk_f = snk_f_all + (size_t)b * n;
    uint64_t* labv = lab_all + (size_t)blockIdx.x * N;
    int64_t* pi = pi_all + (size_t)blockIdx.x * N;
    int32_t* imb = imb_all + (size_t)blockIdx.x * N;
    // BIG exceeds any simple residual path cost: (2Sn+2) x the largest finite arc cost, + 1
    int64_t maxc = 0;
    if (threadIdx.x == 0) { bad_sm = 0; best_sm = 0; byp_sm = 0; }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      const ArcV a = arc_of(c, e);
      if (a.cost > maxc) maxc = a.cost;
    }
    atomicMax(&best_sm, (unsigned long long)maxc);
    if (threadIdx.x == 0) {
      int64_t F0 = 0;
      for (int i = 0; i < n; ++i) F0 += c.src_f[i];
      byp_sm = c.M - F0;
    }
    __syncthreads();
    const int64_t big = (int64_t)(2 * (int64_t)S * n + 2) * (int64_t)best_sm + 1;
    if (big >= (1ll << 36) || byp_sm < 0) {  // labels hold |distance| < 2^38: leave it to the fallback
      if (threadIdx.x == 0) status_out[b] = 7;
      __syncthreads();
      continue;
    }
    // ---- P. potentials of the kept flow (x' = min(x, cap)), zero-flow node arcs and bypass left out ----
    for (int k = threadIdx.x; k < N; k += blockDim.x) labv[k] = lab(0, kNoPred);
    __syncthreads();
    int passes = 0;
    for (;;) {
      if (threadIdx.x == 0) changed_sm = 0;
      __syncthreads();
      int ch = 0;
      // passes alternate the sweep direction (arc ids run stage by stage): forward and backward
      // chains of label updates each propagate within one pass
      for (int64_t rr = threadIdx.x; rr < 2 * E; rr += blockDim.x) {
        const int64_t q = (passes & 1) ? 2 * E - 1 - rr : rr;  // layered order, alternating direction
        const int64_t r = 2 * layered_arc(c, q >> 1) + (q & 1);
        const ArcV a = arc_of(c, r >> 1);
        const int64_t xk = *a.x < a.cap ? *a.x : a.cap;  // the kept flow
        int from, to;
        int64_t rcap, rcost;
        if (r & 1) { from = a.to; to = a.from; rcap = xk; rcost = -a.cost; }
        else {
          from = a.from; to = a.to; rcap = a.cap - xk; rcost = a.cost;
          if ((r >> 1) >= n && (r >> 1) < n + (int64_t)S * n) {  // a rejoined relay's node arc is new
            const int k = (int)((r >> 1) - n);
            if (c.alive[k] && !c.alive_prev[k]) rcap = 0;
          }
        }
        if (rcap <= 0) continue;
        const int64_t d = lab_dist(ld_lab(&labv[from])) + rcost;
        if (d >= kBias || d <= -kBias) { bad_sm = 1; continue; }
        const uint64_t cand = lab(d, (uint64_t)r);
        if ((cand >> kArcBits) < (ld_lab(&labv[to]) >> kArcBits)) {
          const uint64_t old = atomicMin((unsigned long long*)&labv[to], (unsigned long long)cand);
          if ((cand >> kArcBits) < (old >> kArcBits)) ch = 1;
        }
      }
      if (ch) changed_sm = 1;
      __syncthreads();
      const bool any = changed_sm != 0;
      __syncthreads();
      if (!any || bad_sm) break;
      if (++passes > N + 2) { if (threadIdx.x == 0) bad_sm = 7; __syncthreads(); break; }
    }
    if (bad_sm) {  // a negative cycle on the kept flow (or label overflow): the general fallback
      if (threadIdx.x == 0) status_out[b] = 7;
      __syncthreads();
      continue;
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x) { pi[k] = lab_dist(ld_lab(&labv[k])); imb[k] = 0; }
    __syncthreads();
    // ---- C. cut the units the churned graph cannot carry ----
    long long cut = 0, sat = 0;
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      const ArcV a = arc_of(c, e);
      if (*a.x > a.cap) {
        const int32_t dlt = *a.x - (int32_t)a.cap;
        *a.x = (int32_t)a.cap;
        atomicAdd(&imb[a.from], dlt);
        atomicSub(&imb[a.to], dlt);
        cut += dlt;
      }
    }
    __syncthreads();
    // ---- V. saturate the residual arcs with a negative reduced cost ----
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      if (e < n || e >= n + (int64_t)S * n) continue;  // node arcs only (the rest are certified by P)
      const ArcV a = arc_of(c, e);
      const int k = (int)(e - n);
      if (c.alive[k] && !c.alive_prev[k] && *a.x == 0 && a.cap > 0 && pi[a.from] - pi[a.to] < 0) {
        *a.x = (int32_t)a.cap;
        atomicSub(&imb[a.from], (int)a.cap);
        atomicAdd(&imb[a.to], (int)a.cap);
        ++sat;
      }
    }
    __syncthreads();

    // ---- S. successive shortest paths on reduced costs, excess -> deficit ----
    long long iters = 0;
    bool phaseB = false;
    for (;;) {
      if (threadIdx.x == 0) { any_sm = 0; best_sm = ~0ull; }
      __syncthreads();
      for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const bool src = imb[k] > 0;
        labv[k] = src ? lab(0, kNoPred) : kLabInf;
        if (src) any_sm = 1;
      }
      __syncthreads();
      if (!any_sm) {
        if (phaseB || byp_sm == 0) break;
        // B: the bypass's units become s*'s excess and t*'s deficit; real arcs only from here
        phaseB = true;
        if (threadIdx.x == 0) { imb[0] += (int32_t)byp_sm; imb[1] -= (int32_t)byp_sm; }
        __syncthreads();
        continue;
      }
      const int64_t byp = byp_sm;
      const int64_t nr_now = phaseB ? 2 * E : NR;
      int sp = 0;
      for (;;) {  // Bellman-Ford on reduced costs (non-negative: converges within N passes)
        if (threadIdx.x == 0) changed_sm = 0;
        __syncthreads();
        int ch = 0;
        for (int64_t rr = threadIdx.x; rr < nr_now; rr += blockDim.x) {
          const int64_t q = (sp & 1) ? nr_now - 1 - rr : rr;  // layered order, alternating direction
          const int64_t r = q >= 2 * E ? q : 2 * layered_arc(c, q >> 1) + (q & 1);
          int from, to, sign;
          int64_t rcap, rcost;
          int32_t* xp;
          res2(c, r, byp, big, from, to, rcap, rcost, xp, sign);
          if (r == 2 * E + 1) continue;  // the reverse bypass is never used (B moves its units)
          if (rcap <= 0) continue;
          const uint64_t Lf = ld_lab(&labv[from]);
          if (Lf == kLabInf) continue;
          const int64_t d = lab_dist(Lf) + rcost + pi[from] - pi[to];
          if (d >= kBias) { bad_sm = 1; continue; }
          const uint64_t cand = lab(d, (uint64_t)r);
          if ((cand >> kArcBits) < (ld_lab(&labv[to]) >> kArcBits)) {
            const uint64_t old = atomicMin((unsigned long long*)&labv[to], (unsigned long long)cand);
            if ((cand >> kArcBits) < (old >> kArcBits)) ch = 1;
          }
        }
        if (ch) changed_sm = 1;
        __syncthreads();
        const bool anych = changed_sm != 0;
        __syncthreads();
        if (!anych || bad_sm) break;
        if (++sp > N + 2) { if (threadIdx.x == 0) bad_sm = 3; __syncthreads(); break; }
      }
      if (bad_sm) break;
      // nearest deficit node (distance, node) -- lowest node on ties
      for (int k = threadIdx.x; k < N; k += blockDim.x) {
        if (imb[k] >= 0) continue;
        const uint64_t L = ld_lab(&labv[k]);
        if (L == kLabInf) continue;
        atomicMin(&best_sm, ((unsigned long long)(lab_dist(L) + kBias) << 24) | (unsigned long long)k);
      }
      __syncthreads();
      if (best_sm == ~0ull) {
        if (phaseB) {  // t* unreachable: the units left at s* stay on the bypass (F is maximal)
          if (threadIdx.x == 0) { byp_sm = imb[0]; imb[1] += imb[0]; imb[0] = 0; }
          __syncthreads();
          break;
        }
        if (threadIdx.x == 0) bad_sm = 6;
        __syncthreads();
        break;
      }
      const int tgt = (int)(best_sm & 0xFFFFFF);
      const int64_t dt = (int64_t)(best_sm >> 24) - kBias;
      if (threadIdx.x == 0) {  // trace to the source excess node, bottleneck, augment
        int64_t bott = -(int64_t)imb[tgt];
        int x = tgt, guard = 0;
        while (lab_pred(ld_lab(&labv[x])) != (int)kNoPred && ++guard <= N + 2) {
          int from, to, sign; int64_t rcap, rcost; int32_t* xp;
          res2(c, lab_pred(ld_lab(&labv[x])), byp_sm, big, from, to, rcap, rcost, xp, sign);
          bott = rcap < bott ? rcap : bott;
          x = from;
        }
        const int s0 = x;
        if (guard > N + 2 || imb[s0] <= 0) { bad_sm = 5; }
        else {
          bott = imb[s0] < bott ? imb[s0] : bott;
          for (x = tgt; x != s0;) {
            int from, to, sign; int64_t rcap, rcost; int32_t* xp;
            const int r = lab_pred(ld_lab(&labv[x]));
            res2(c, r, byp_sm, big, from, to, rcap, rcost, xp, sign);
            if (xp) *xp += (int32_t)(sign * bott);
            else byp_sm += sign * bott;
            x = from;
          }
          imb[s0] -= (int32_t)bott;
          imb[tgt] += (int32_t)bott;
          if (phaseB) byp_sm -= bott;  // an s* -> t* path on real arcs takes units off the bypass
        }
        delta_sm = bott;
      }
      __syncthreads();
      if (bad_sm) break;
      for (int k = threadIdx.x; k < N; k += blockDim.x) {  // pi += min(d, d_target)
        const uint64_t L = ld_lab(&labv[k]);
        const int64_t d = L == kLabInf ? dt : lab_dist(L);
        pi[k] += d < dt ? d : dt;
      }
      ++iters;
      __syncthreads();
    }
    // ---- objective of the repaired assignment ----
    if (threadIdx.x == 0) cost_sm = 0;
    __syncthreads();
    long long part = 0;
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      const ArcV a = arc_of(c, e);
      part += (long long)*a.x * a.cost;
    }
    atomicAdd(&cost_sm, (unsigned long long)part);
    __shared__ unsigned long long cut_sm, sat_sm;
    if (threadIdx.x == 0) { cut_sm = 0; sat_sm = 0; }
    __syncthreads();
    atomicAdd(&cut_sm, (unsigned long long)cut);
    atomicAdd(&sat_sm, (unsigned long long)sat);
    __syncthreads();
    if (threadIdx.x == 0) {
      F_out[b] = c.M - byp_sm;
      cost_out[b] = (int64_t)cost_sm;
      if (stats_out) { stats_out[3 * b] = (int64_t)cut_sm; stats_out[3 * b + 1] = (int64_t)sat_sm; stats_out[3 * b + 2] = iters; }
      status_out[b] = bad_sm;
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------------------------
// The same potential-carrying repair with the instance in shared memory (round 2): labels, preds,
// potentials, imbalances, node / src / snk flows and the link flows (int16) of one instance per
// CTA, the link costs read through L1; every Bellman-Ford pass is a layered sweep -- forward arcs
// stage by stage (s* -> in_0, in -> out, out_s -> in_{s+1} as one row minimum per destination,
// out_{S-1} -> t*, the bypass), then reverse arcs back to front -- one block barrier per layer, so a
// pass carries a label across every stage in one direction.  Labels are (distance, pred node):
// the arc between two adjacent nodes is unique, so the pred node names it.  Same phases P, C, V,
// A, B as warm_kernel; an instance that does not fit (or whose kept flow has a negative cycle) is
// left to the next kernel with status 7.
constexpr int64_t kDInf = INT64_MAX / 4;
struct WsLayout { size_t dist, pi, pred, imb, g, srcf, snkf, arcf, red, t16, total; };
// t16_bytes: the instance's 16-bit tile copy staged in shared memory (0: link costs read from L2)
__host__ __device__ inline WsLayout ws_layout(int S, int n, size_t t16_bytes = 0) {
  WsLayout L;
  const size_t N = 2 + 2 * (size_t)S * n, Sn = (size_t)S * n, A = (size_t)(S > 1 ? S - 1 : 0) * n * n;
  size_t o = 0;
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  L.dist = o; o += al(N * 8);
  L.pi = o; o += al(N * 8);
  L.pred = o; o += al(N * 4);
  L.imb = o; o += al(N * 4);
  L.g = o; o += al(Sn * 4);
  L.srcf = o; o += al((size_t)n * 4);
  L.snkf = o; o += al((size_t)n * 4);
  L.arcf = o; o += al(A * 2);
  L.red = o; o += 64;
  L.t16 = o; o += al(t16_bytes);
  L.total = o;
  return L;
}

// a row minimum's candidate and source packed into one key: (cand + 2^44) << 19 | source.  The
// shared-memory repair's labels stay within |d| < 2^44 (path costs < 2^42 by the create bounds, plus two
// potentials) and its node ids below 2^19 (the workspace fits 100 KB), so the packed minimum is the lowest
// candidate and, among equal ones, the lowest source
constexpr uint64_t kPackMask = (1ull << 19) - 1;
__device__ __forceinline__ uint64_t umin64w(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t pack_cand(int64_t cand, int src) {
  return ((uint64_t)(cand + (1ll << 44)) << 19) | (uint64_t)src;
}
__device__ __forceinline__ int64_t unpack_cand(uint64_t k) { return (int64_t)(k >> 19) - (1ll << 44); }

__global__ void __launch_bounds__(kThreads, 2) warm_smem_kernel(const Problem P, int32_t* src_f_all, int32_t* g_all,
                                                             int32_t* arc_all, int32_t* snk_f_all, int64_t* F_out,
                                                             int64_t* cost_out, int64_t* stats_out, int32_t* status_out,
                                                             size_t t16_bytes) {
  extern __shared__ __align__(16) uint8_t wsm[];
  const int S = P.S, n = P.n, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = kThreads / 32;
  const int N = 2 + 2 * S * n, Sn = S * n;
  // the 16-bit tiles in shared memory when the launch reserved room for them
  const bool t16 = P.tile16s != nullptr && t16_bytes > 0;
  const WsLayout L = ws_layout(S, n, t16 ? t16_bytes : 0);
  const uint16_t* tile16 = (const uint16_t*)(wsm + L.t16);
  int64_t* dist = (int64_t*)(wsm + L.dist);
  int64_t* pi = (int64_t*)(wsm + L.pi);
  int32_t* pred = (int32_t*)(wsm + L.pred);
  int32_t* imb = (int32_t*)(wsm + L.imb);
  int32_t* g = (int32_t*)(wsm + L.g);
  int32_t* srcf = (int32_t*)(wsm + L.srcf);
  int32_t* snkf = (int32_t*)(wsm + L.snkf);
  int16_t* arcf = (int16_t*)(wsm + L.arcf);
  unsigned long long* red = (unsigned long long*)(wsm + L.red);
  int* ired = (int*)(red + 4);
  __shared__ unsigned long long dm[4];
  __shared__ unsigned int dfl[2];
  auto IN = [&](int s, int i) { return 2 + 2 * (s * n + i); };
  for (int b = blockIdx.x; b < P.B; b += gridDim.x) {
    if (status_out[b] == kDeferred) continue;  // triage: left to the cold solve
    const int32_t* tile = P.tile + (size_t)b * (S - 1) * n * P.ld;
    const int32_t* src = P.src + (size_t)b * n;
    const int32_t* snk = P.snk + (size_t)b * n;
    const int32_t* cap = P.cap + (size_t)b * Sn;
    const uint8_t* alive = P.alive + (size_t)b * Sn;
    const uint8_t* alive_prev = P.alive_prev + (size_t)b * Sn;
    int32_t* gG = g_all + (size_t)b * Sn;
    int32_t* sG = src_f_all + (size_t)b * n;
    int32_t* kG = snk_f_all + (size_t)b * n;
    int32_t* aG = arc_all + (size_t)b * (S - 1) * n * n;
    const int64_t M = P.supply[b];
    auto capE = [&](int k) -> int32_t { return alive[k] ? cap[k] : 0; };
    auto C = [&](int s, int u, int v) -> int32_t {
      if (t16) {
        const uint32_t c = tile16[((size_t)s * n + v) * P.ld + u];
        return c == 0xFFFFu ? kAbsent : (int32_t)c;
      }
      return __ldg(&tile[((size_t)s * n + v) * P.ld + u]);
    };
    // ---- load, cut (units the churned graph cannot carry), BIG ----
    if (tid == 0) { red[0] = 0; red[1] = 0; red[2] = 0; ired[0] = 0; ired[2] = 0; ired[3] = 0; }
    for (int k = tid; k < N; k += kThreads) imb[k] = 0;
    if (t16) {  // the instance's 16-bit link costs into shared memory (every pass reads them)
      const uint4* s4 = (const uint4*)(P.tile16s + (size_t)b * P.tile16s_stride);
      uint4* d4 = (uint4*)(wsm + L.t16);
      for (size_t k = tid; k < t16_bytes / 16; k += kThreads) d4[k] = s4[k];
    }
    __syncthreads();
    long long cut = 0, F0 = 0;
    int32_t maxc = 0, bigf = 0;
    for (int k = tid; k < n; k += kThreads) {
      int32_t x = sG[k];
      const int32_t c = src[k];
      if (c != kAbsent && c > maxc) maxc = c;
      F0 += x;
      if (c == kAbsent && x > 0) { atomicAdd(&imb[0], x); atomicSub(&imb[IN(0, k)], x); cut += x; x = 0; }
      srcf[k] = x;
      int32_t y = kG[k];
      const int32_t d = snk[k];
      if (d != kAbsent && d > maxc) maxc = d;
      if (d == kAbsent && y > 0) { atomicAdd(&imb[IN(S - 1, k) + 1], y); atomicSub(&imb[1], y); cut += y; y = 0; }
      snkf[k] = y;
    }
    for (int k = tid; k < Sn; k += kThreads) {
      int32_t x = gG[k];
      const int32_t ce = capE(k);
      if (x > ce) { atomicAdd(&imb[2 + 2 * k], x - ce); atomicSub(&imb[3 + 2 * k], x - ce); cut += x - ce; x = ce; }
      g[k] = x;
    }
    for (int64_t e = tid; e < (int64_t)(S - 1) * n * n; e += kThreads) {
      const int s = (int)(e / ((int64_t)n * n)), r = (int)(e - (int64_t)s * n * n), v = r / n, u = r - v * n;
      int32_t x = aG[e];
      const int32_t c = C(s, u, v);
      if (c != kAbsent && c > maxc) maxc = c;
      if (x > 32767) bigf = 1;
      if (c == kAbsent && x > 0) { atomicAdd(&imb[IN(s, u) + 1], x); atomicSub(&imb[IN(s + 1, v)], x); cut += x; x = 0; }
      arcf[e] = (int16_t)x;
    }
    atomicAdd(&red[0], (unsigned long long)F0);
    atomicMax(&red[1], (unsigned long long)maxc);
    if (bigf) atomicOr(&ired[0], 1);
    __syncthreads();
    const int64_t big = (2 * (int64_t)S * n + 2) * (int64_t)red[1] + 1;
    int64_t byp = M - (int64_t)red[0];
    if (ired[0] || M > 32767 || big >= (1ll << 40)) {  // int16 link flows / label range: next kernel
      if (tid == 0) status_out[b] = 70;
      __syncthreads();
      continue;
    }
    // ---- one layered Bellman-Ford pass ----
    // mode 0: potentials (real costs, rejoined relays' node arcs and the bypass left out);
    // mode 1: reduced costs, bypass forward allowed (phase A); mode 2: reduced costs, no bypass (B)
    // layers whose labels changed (bit s of dm[0] / dm[1]: in_s / out_s; dfl bit 0 / 1: s* / t*) in
    // this pass ([0], [1], dfl[0]) and the previous one ([2], [3], dfl[1]): a relaxation whose source
    // layer changed in neither since it last ran cannot lower anything and is skipped (S <= 64)
    const bool track = S <= 64;
    auto mark = [&](int to) {
      if (!track) return;
      if (to < 2) atomicOr(&dfl[0], 1u << to);
      else atomicOr(&dm[to & 1], 1ull << (((to - 2) >> 1) / n));
    };
    auto relax = [&](int to, int64_t cand, int from, int& ch) {
      if (cand < dist[to]) { dist[to] = cand; pred[to] = from; ch = 1; mark(to); }
    };
    auto din = [&](int s) { return !track || (((dm[0] | dm[2]) >> s) & 1ull); };
    auto dout = [&](int s) { return !track || (((dm[1] | dm[3]) >> s) & 1ull); };
    auto dnode = [&](int x) { return !track || ((dfl[0] | dfl[1]) >> x) & 1u; };  // 0: s*, 1: t*
    auto w = [&](int mode, int from, int to, int64_t c) -> int64_t { return mode ? c + pi[from] - pi[to] : c; };
    auto pass = [&](int mode, bool first) -> bool {
      int ch = 0;
      if (tid == 0) {  // this pass's change sets start empty; the previous pass's become "prev"
        dm[2] = first ? ~0ull : dm[0];
        dm[3] = first ? ~0ull : dm[1];
        dfl[1] = first ? 3u : dfl[0];
        dm[0] = 0;
        dm[1] = 0;
        dfl[0] = 0;
      }
      __syncthreads();
      // forward: s* -> in_0
      if (dnode(0))
        for (int i = tid; i < n; i += kThreads)
          if (dist[0] < kDInf && src[i] != kAbsent) relax(IN(0, i), dist[0] + w(mode, 0, IN(0, i), src[i]), 0, ch);
      __syncthreads();
      for (int s = 0; s < S; ++s) {
        if (din(s))
        for (int i = tid; i < n; i += kThreads) {  // in -> out (node arc, residual cap - g)
          const int k = s * n + i, a = IN(s, i);
          if (g[k] >= capE(k) || dist[a] >= kDInf) continue;
          if (mode == 0 && alive[k] && !alive_prev[k]) continue;  // a rejoined relay's arc is new
          relax(a + 1, dist[a] + w(mode, a, a + 1, 0), a, ch);
        }
        __syncthreads();
        if (s + 1 < S && dout(s)) {  // out_s -> in_{s+1}: one row minimum per destination (warp per row)
          for (int v = wid; v < n; v += nw) {
            const int to = IN(s + 1, v);
            uint64_t bk = ~0ull;  // packed (candidate, source): the lowest candidate, then the lowest source
            for (int u = lane; u < n; u += 32) {
              const int fr = IN(s, u) + 1;
              const int32_t c = C(s, u, v);
              if (c == kAbsent || dist[fr] >= kDInf) continue;
              bk = umin64w(bk, pack_cand(dist[fr] + w(mode, fr, to, c), fr));
            }
            for (int off = 16; off > 0; off >>= 1) bk = umin64w(bk, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)bk, off));
            if (lane == 0 && bk != ~0ull) relax(to, unpack_cand(bk), (int)(bk & kPackMask), ch);
          }
          __syncthreads();
        }
      }
      if (tid == 0) {  // out_{S-1} -> t*, then the bypass s* -> t*
        if (dout(S - 1))
        for (int i = 0; i < n; ++i) {
          const int fr = IN(S - 1, i) + 1;
          if (snk[i] != kAbsent && dist[fr] < kDInf) relax(1, dist[fr] + w(mode, fr, 1, snk[i]), fr, ch);
        }
        if (mode == 1 && byp < M && dist[0] < kDInf && dnode(0)) relax(1, dist[0] + w(mode, 0, 1, big), 0, ch);
      }
      __syncthreads();
      // backward: t* -> out_{S-1} (snk flow), then per stage out -> in (node flow) and in_{s} -> out_{s-1}
      if (dnode(1))
      for (int i = tid; i < n; i += kThreads) {
        const int to = IN(S - 1, i) + 1;
        if (snkf[i] > 0 && dist[1] < kDInf) relax(to, dist[1] + w(mode, 1, to, -(int64_t)snk[i]), 1, ch);
      }
      __syncthreads();
      for (int s = S - 1; s >= 0; --s) {
        if (dout(s))
        for (int i = tid; i < n; i += kThreads) {  // out -> in (reverse node arc, residual g)
          const int k = s * n + i, a = IN(s, i);
          if (g[k] > 0 && dist[a + 1] < kDInf) relax(a, dist[a + 1] + w(mode, a + 1, a, 0), a + 1, ch);
        }
        __syncthreads();
        if (s > 0 && din(s)) {  // in_s -> out_{s-1}: reverse link arcs carrying flow (warp per source u)
          for (int u = wid; u < n; u += nw) {
            const int to = IN(s - 1, u) + 1;
            uint64_t bk = ~0ull;
            for (int v = lane; v < n; v += 32) {
              const int fr = IN(s, v);
              if (arcf[((size_t)(s - 1) * n + v) * n + u] <= 0 || dist[fr] >= kDInf) continue;
              bk = umin64w(bk, pack_cand(dist[fr] + w(mode, fr, to, -(int64_t)C(s - 1, u, v)), fr));
            }
            for (int off = 16; off > 0; off >>= 1) bk = umin64w(bk, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)bk, off));
            if (lane == 0 && bk != ~0ull) relax(to, unpack_cand(bk), (int)(bk & kPackMask), ch);
          }
          __syncthreads();
        }
      }
      if (tid == 0 && din(0))  // in_0 -> s* (reverse src arcs)
        for (int i = 0; i < n; ++i)
          if (srcf[i] > 0 && dist[IN(0, i)] < kDInf) relax(0, dist[IN(0, i)] + w(mode, IN(0, i), 0, -(int64_t)src[i]), IN(0, i), ch);
      return __syncthreads_or(ch) != 0;
    };
    // ---- P. potentials of the kept (cut) flow from a virtual root ----
    for (int k = tid; k < N; k += kThreads) { dist[k] = 0; pred[k] = -1; }
    __syncthreads();
    int passes = 0;
    bool conv = true;
    for (bool first = true; pass(0, first); first = false) if (++passes > N + 2) { conv = false; break; }
#ifdef GWTF_DEV_FLAGS
    if ((P.debug & 16) && tid == 0) { atomicAdd(&P.stats[1300], (unsigned long long)passes + 1); atomicAdd(&P.stats[1303], 1ull); }
#endif
    if (!conv) {  // a negative cycle on the kept flow (a lowered cost): the Klein fallback, flows untouched
      if (tid == 0) status_out[b] = 71;
      __syncthreads();
      continue;
    }
    for (int k = tid; k < N; k += kThreads) pi[k] = dist[k];
    __syncthreads();
    // ---- V. saturate rejoined relays' node arcs with a negative reduced cost ----
    long long sat = 0;
    for (int k = tid; k < Sn; k += kThreads) {
      const int a = 2 + 2 * k;
      if (alive[k] && !alive_prev[k] && g[k] == 0 && capE(k) > 0 && pi[a] - pi[a + 1] < 0) {
        g[k] = capE(k);
        imb[a] -= capE(k);
        imb[a + 1] += capE(k);
        ++sat;
      }
    }
    __syncthreads();
    // ---- A / B. successive shortest paths on reduced costs ----
    long long iters = 0;
    bool phaseB = false, bad = false;
    for (;;) {
      if (tid == 0) ired[1] = 0;
      __syncthreads();
      for (int k = tid; k < N; k += kThreads) {
        const bool srcn = imb[k] > 0;
        dist[k] = srcn ? 0 : kDInf;
        pred[k] = -1;
        if (srcn) ired[1] = 1;
      }
      __syncthreads();
      if (!ired[1]) {
        if (phaseB || byp == 0) break;
        phaseB = true;  // B: the bypass's units become s*'s excess and t*'s deficit
        if (tid == 0) { imb[0] += (int32_t)byp; imb[1] -= (int32_t)byp; }
        __syncthreads();
        continue;
      }
      int sp = 0;
      for (bool first = true; pass(phaseB ? 2 : 1, first); first = false) if (++sp > N + 2) { bad = true; break; }
#ifdef GWTF_DEV_FLAGS
      if ((P.debug & 16) && tid == 0) { atomicAdd(&P.stats[1301], (unsigned long long)sp + 1); atomicAdd(&P.stats[1302], 1ull); }
#endif
      if (bad) { if (tid == 0) ired[3] = 74; break; }
      if (tid == 0) red[3] = ~0ull;
      __syncthreads();
      for (int k = tid; k < N; k += kThreads)
        if (imb[k] < 0 && dist[k] < kDInf) atomicMin(&red[3], ((unsigned long long)dist[k] << 20) | (unsigned long long)k);
      __syncthreads();
      const unsigned long long bestv = red[3];
      if (bestv == ~0ull) {
        if (phaseB) {  // t* unreachable: the units left at s* stay on the bypass
          byp = imb[0];
          __syncthreads();
          if (tid == 0) { imb[1] += imb[0]; imb[0] = 0; }
          __syncthreads();
          break;
        }
        if (tid == 0) ired[3] = 72;
        bad = true;
        break;
      }
      const int tgt = (int)(bestv & 0xFFFFF);
      const int64_t dt = dist[tgt];
      if (tid == 0) {  // trace, bottleneck, augment
        int64_t bott = -(int64_t)imb[tgt];
        int x = tgt, guard = 0;
        auto rescap = [&](int fr, int to) -> int64_t {
          if (fr == 0 && to == 1) return M - byp;
          if (fr == 1 && to == 0) return byp;
          if (fr == 0) return kDInf;                                   // src forward
          if (to == 0) return srcf[(fr - 2) / 2];                      // src reverse
          if (to == 1) return kDInf;                                   // snk forward
          if (fr == 1) return snkf[(to - 3) / 2 - (S - 1) * n];        // snk reverse
          const int kf = (fr - 2) / 2, kt = (to - 2) / 2;
          if (kf == kt) return (fr & 1) ? g[kf] : capE(kf) - g[kf];    // node arc reverse / forward
          if (fr & 1) return kDInf;                                    // link forward
          const int sv = kf / n, v = kf % n, u = kt % n;               // link reverse: in_{sv,v} -> out_{sv-1,u}
          return arcf[((size_t)(sv - 1) * n + v) * n + u];
        };
        while (pred[x] >= 0 && ++guard <= N + 2) {
          const int64_t rc = rescap(pred[x], x);
          bott = rc < bott ? rc : bott;
          x = pred[x];
        }
        const int s0 = x;
        if (guard > N + 2 || imb[s0] <= 0 || bott <= 0) {
          ired[2] = 1;
        } else {
          bott = imb[s0] < bott ? imb[s0] : bott;
          for (x = tgt; x != s0; x = pred[x]) {
            const int fr = pred[x], to = x;
            const int32_t d = (int32_t)bott;
            if (fr == 0 && to == 1) byp += bott;
            else if (fr == 1 && to == 0) byp -= bott;
            else if (fr == 0) srcf[(to - 2) / 2] += d;
            else if (to == 0) srcf[(fr - 2) / 2] -= d;
            else if (to == 1) snkf[(fr - 3) / 2 - (S - 1) * n] += d;
            else if (fr == 1) snkf[(to - 3) / 2 - (S - 1) * n] -= d;
            else {
              const int kf = (fr - 2) / 2, kt = (to - 2) / 2;
              if (kf == kt) g[kf] += (fr & 1) ? -d : d;
              else if (fr & 1) { const int su = kf / n; arcf[((size_t)su * n + kt % n) * n + kf % n] += (int16_t)d; }
              else { const int sv = kf / n; arcf[((size_t)(sv - 1) * n + kf % n) * n + kt % n] -= (int16_t)d; }
            }
          }
          imb[s0] -= (int32_t)bott;
          imb[tgt] += (int32_t)bott;
          if (phaseB) byp -= bott;
          red[2] = (unsigned long long)byp;
        }
      }
      __syncthreads();
      if (ired[2]) { if (tid == 0) ired[3] = 73; bad = true; break; }
      byp = (int64_t)red[2];
      for (int k = tid; k < N; k += kThreads) pi[k] += dist[k] < dt ? dist[k] : dt;
      ++iters;
      __syncthreads();
    }
    if (bad) {  // never expected: leave the instance to the fallback (its input flows are untouched)
      if (tid == 0) status_out[b] = ired[3];
      __syncthreads();
      continue;
    }
    // ---- write back, objective ----
    if (tid == 0) { red[0] = 0; red[1] = 0; red[2] = 0; }
    __syncthreads();
    long long part = 0;
    for (int k = tid; k < n; k += kThreads) {
      sG[k] = srcf[k]; kG[k] = snkf[k];
      part += (long long)srcf[k] * (src[k] == kAbsent ? 0 : src[k]) + (long long)snkf[k] * (snk[k] == kAbsent ? 0 : snk[k]);
    }
    for (int k = tid; k < Sn; k += kThreads) gG[k] = g[k];
    for (int64_t e = tid; e < (int64_t)(S - 1) * n * n; e += kThreads) {
      const int s = (int)(e / ((int64_t)n * n)), r = (int)(e - (int64_t)s * n * n), v = r / n, u = r - v * n;
      aG[e] = arcf[e];
      if (arcf[e]) part += (long long)arcf[e] * C(s, u, v);
    }
    atomicAdd(&red[0], (unsigned long long)part);
    atomicAdd(&red[1], (unsigned long long)cut);
    atomicAdd(&red[2], (unsigned long long)sat);
    __syncthreads();
    if (tid == 0) {
      F_out[b] = M - byp;
      cost_out[b] = (int64_t)red[0];
      if (stats_out) { stats_out[3 * b] = (int64_t)red[1]; stats_out[3 * b + 1] = (int64_t)red[2]; stats_out[3 * b + 2] = iters; }
      status_out[b] = 0;
    }
    __syncthreads();
  }
}

}  // namespace

size_t warm_ws_bytes(const Problem& P, int grid) {
  const size_t N = 2 + 2 * (size_t)P.S * P.n;
  return (size_t)grid * N * (8 + 4 + 8 + 4);
}

int warm_grid(const Problem& P) { return (int)std::min<int64_t>(P.B, 148 * 8); }

// status must be a device array of B entries: the repair kernel runs every instance, the fallback
// kernel the ones it marked 7
// Triage (before the repair): the units the churned graph can no longer carry (flow above an
// arc's new capacity: crashed relays, dropped links) against the assignment's flow F0.  A repair
// has to re-route at least those units with one layered search each, while a cold solve of these
// small instances costs about F0 searches of the (faster) exact-solve kernels; an instance with
// kWarmCutShare x cut > F0 is left to the cold solve (status kDeferred, stats {cut, 0, 0}), and so
// is every instance with fewer than kWarmMinLinks links: there the whole cold batch costs a few
// microseconds per instance, less than one repaired instance's chain of layered passes (gpt shape:
// 1,280 links, 16,384 instances cold in 4.4 ms, 730 repaired ones in ~10 ms).
constexpr int kWarmCutShare = 4;
constexpr int64_t kWarmMinLinks = 4096;
__global__ void __launch_bounds__(kThreads) warm_triage_kernel(const Problem P, int32_t* src_f_all, int32_t* g_all,
                                                                int32_t* arc_all, int32_t* snk_f_all,
                                                                int64_t* stats_out, int32_t* status_out, bool repair_all,
                                                                bool smem_repair) {
  __shared__ unsigned long long red[2];
  const int S = P.S, n = P.n;
  const int64_t E = 2ll * n + (int64_t)S * n + (int64_t)(S - 1) * n * n;
  for (int b = blockIdx.x; b < P.B; b += gridDim.x) {
    WarmCtx c;
    c.S = S; c.n = n; c.ld = P.ld; c.N = 2 + 2 * S * n; c.E = E; c.M = P.supply[b];
    c.tile = P.tile + (size_t)b * (S - 1) * n * P.ld;
    c.src = P.src + (size_t)b * n;
    c.snk = P.snk + (size_t)b * n;
    c.cap = P.cap + (size_t)b * S * n;
    c.alive = P.alive + (size_t)b * S * n;
    c.alive_prev = P.alive_prev + (size_t)b * S * n;
    c.src_f = src_f_all + (size_t)b * n;
    c.g = g_all + (size_t)b * S * n;
    c.arc = arc_all + (size_t)b * (S - 1) * n * n;
    c.snk_f = snk_f_all + (size_t)b * n;
    if (threadIdx.x == 0) { red[0] = 0; red[1] = 0; }
    __syncthreads();
    unsigned long long cut = 0, f0 = 0;
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      const ArcV a = arc_of(c, e);
      if (*a.x > a.cap) cut += (unsigned long long)(*a.x - a.cap);
      if (e < n) f0 += (unsigned long long)*a.x;
    }
    atomicAdd(&red[0], cut);
    atomicAdd(&red[1], f0);
    __syncthreads();
    if (threadIdx.x == 0) {
      const bool defer = !repair_all && (!smem_repair || (int64_t)(S - 1) * n * n < kWarmMinLinks ||
                                         (unsigned long long)kWarmCutShare * red[0] > red[1]);
      status_out[b] = defer ? kDeferred : 0;
      // {cut, 0, 0}: a repair overwrites it, a cold solve sets [2] to its augmentations
      if (stats_out) { stats_out[3 * b] = (int64_t)red[0]; stats_out[3 * b + 1] = 0; stats_out[3 * b + 2] = 0; }
    }
    __syncthreads();
  }
}

// instances left to the cold solve: deferred by the triage, or whose repair stopped (7, 70-79)
__global__ void warm_collect_kernel(int32_t B, int32_t* status, int32_t* sel, int32_t* sel_count,
                                    unsigned long long* ctr) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    const int32_t q = status[b];
    if (q == 7 || q >= 70) {
      status[b] = kDeferred;
      sel[atomicAdd(sel_count, 1)] = b;
      atomicAdd(ctr, 1ull);  // gwtf_flow_stats [12]
    }
  }
}

// the cold-solved instances' link flows into the dense [B][S-1][n][n] layout (zero, then scatter
// the positive-arc lists), and their augmentation counts into stats[3b + 2]
__global__ void warm_dense_zero_kernel(const Problem P2, const int32_t* sel, const int32_t* sel_count, int32_t* dense) {
  const int64_t slab = (int64_t)(P2.S - 1) * P2.n * P2.n, cnt = *sel_count;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt * slab; t += (int64_t)gridDim.x * blockDim.x)
    dense[(int64_t)sel[t / slab] * slab + t % slab] = 0;
}
__global__ void warm_dense_scatter_kernel(const Problem P2, const int32_t* sel, const int32_t* sel_count, int32_t* dense,
                                          const int32_t* aug, int64_t* stats_out) {
  const int64_t nb = P2.S - 1, per = nb * P2.Lcap, cnt = *sel_count;
  if (stats_out)
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x)
      stats_out[3 * (int64_t)sel[t] + 2] = aug[sel[t]];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt * per; t += (int64_t)gridDim.x * blockDim.x) {
    const int b = sel[t / per];
    const int64_t r = t % per, sb = r / P2.Lcap, e = r % P2.Lcap;
    const int64_t bs = (int64_t)b * nb + sb;
    if (e >= P2.arc_cnt[bs]) continue;
    const uint32_t ent = P2.arcs[bs * P2.Lcap + e];
    const int u = (int)(ent >> 20), v = (int)((ent >> 8) & 0xFFFu);
    dense[((int64_t)bs * P2.n + v) * P2.n + u] = (int32_t)(ent & 0xFFu);
  }
}

cudaError_t launch_warm(const Problem& P, int32_t* src_f, int32_t* g, int32_t* arc, int32_t* snk_f, void* ws,
                        int64_t* F, int64_t* cost, int64_t* stats, int32_t* status, bool repair_all, cudaStream_t st) {
  const int grid = warm_grid(P);
  const size_t N = 2 + 2 * (size_t)P.S * P.n;
  // the repair runs in shared memory when one instance's state fits (<= 100 KB: at least two CTAs per
  // SM); larger instances (the cluster-tier shapes) are solved cold unless every repair is asked for --
  // one 256-thread CTA per instance over global memory cannot keep up with the cluster tier
  const size_t wsm = ws_layout(P.S, P.n).total;
  const bool smem_repair = wsm <= 100 * 1024 && P.S > 1;
  warm_triage_kernel<<<(int)std::min<int64_t>(P.B, 148 * 8), kThreads, 0, st>>>(P, src_f, g, arc, snk_f, stats, status,
                                                                                     repair_all, smem_repair);
  uint64_t* labv = (uint64_t*)ws;
  int64_t* pi = (int64_t*)(labv + (size_t)grid * N);
  int32_t* imb = (int32_t*)(pi + (size_t)grid * N);
  int32_t* stamp = imb + (size_t)grid * N;
  if (smem_repair) {
    // the 16-bit link costs join the workspace when two CTAs per SM still fit (113 KB each)
    const size_t t16b = P.tile16s ? (size_t)P.tile16s_stride * 2 : 0;
    const size_t t16_bytes = (t16b && ws_layout(P.S, P.n, t16b).total <= 113 * 1024) ? t16b : 0;
    const size_t wsm = ws_layout(P.S, P.n, t16_bytes).total;
    cudaError_t e = cudaFuncSetAttribute(warm_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, warm_smem_kernel, kThreads, wsm);
    if (e != cudaSuccess) return e;
    const int g2 = (int)std::min<int64_t>(P.B, (int64_t)std::max(per_sm, 1) * 148);
    warm_smem_kernel<<<g2, kThreads, wsm, st>>>(P, src_f, g, arc, snk_f, F, cost, stats, status, t16_bytes);
  } else {
    warm_kernel<<<grid, kThreads, 0, st>>>(P, src_f, g, arc, snk_f, labv, pi, imb, F, cost, stats, status);
  }
  if (P.debug & 4096)  // testing (dev builds): the Klein cycle-cancelling fallback instead of the cold solve
    klein_kernel<<<grid, kThreads, 0, st>>>(P, src_f, g, arc, snk_f, labv, stamp, F, cost, stats, status);
  return cudaGetLastError();
}

cudaError_t launch_warm_collect(int32_t B, int32_t* status, int32_t* sel, int32_t* sel_count, unsigned long long* ctr,
                                cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(sel_count, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  warm_collect_kernel<<<(int)std::min<int64_t>((B + 255) / 256, 148 * 4), 256, 0, st>>>(B, status, sel, sel_count, ctr);
  return cudaGetLastError();
}

cudaError_t launch_warm_dense(const Problem& P2, const int32_t* sel, const int32_t* sel_count, int32_t* dense,
                              const int32_t* aug, int64_t* stats, cudaStream_t st) {
  if (P2.S > 1) warm_dense_zero_kernel<<<148 * 8, 256, 0, st>>>(P2, sel, sel_count, dense);
  warm_dense_scatter_kernel<<<148 * 8, 256, 0, st>>>(P2, sel, sel_count, dense, aug, stats);
  return cudaGetLastError();
}

}  // namespace gwtf
