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
#include <stdint.h>

#include "gwtf_internal.h"

namespace gwtf {

namespace {

constexpr int kThreads = 256;
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
    if (status_out[b] != 7) continue;  // solved by warm_kernel
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

}  // namespace

size_t warm_ws_bytes(const Problem& P, int grid) {
  const size_t N = 2 + 2 * (size_t)P.S * P.n;
  return (size_t)grid * N * (8 + 4 + 8 + 4);
}

int warm_grid(const Problem& P) { return (int)std::min<int64_t>(P.B, 148 * 8); }

// status must be a device array of B entries: the repair kernel runs every instance, the fallback
// kernel the ones it marked 7
cudaError_t launch_warm(const Problem& P, int32_t* src_f, int32_t* g, int32_t* arc, int32_t* snk_f, void* ws,
                        int64_t* F, int64_t* cost, int64_t* stats, int32_t* status, cudaStream_t st) {
  const int grid = warm_grid(P);
  const size_t N = 2 + 2 * (size_t)P.S * P.n;
  uint64_t* labv = (uint64_t*)ws;
  int64_t* pi = (int64_t*)(labv + (size_t)grid * N);
  int32_t* imb = (int32_t*)(pi + (size_t)grid * N);
  int32_t* stamp = imb + (size_t)grid * N;
  warm_kernel<<<grid, kThreads, 0, st>>>(P, src_f, g, arc, snk_f, labv, pi, imb, F, cost, stats, status);
  klein_kernel<<<grid, kThreads, 0, st>>>(P, src_f, g, arc, snk_f, labv, stamp, F, cost, stats, status);
  return cudaGetLastError();
}

}  // namespace gwtf
