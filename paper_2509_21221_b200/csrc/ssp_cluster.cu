// Exact solve, cluster tier: one thread-block cluster (up to 16 CTAs, one per SM) per instance,
// for instances whose tiles cannot live in shared memory (e.g. the stress shape: 64 stages x
// 1,024 clients = 252 MB of int32 tiles).  Same canonical SSP as ssp.cu with
// 64-bit (cost, hops) keys; only the data placement differs (K1c):
//   * CTA r of the cluster owns destination rows v in [r*R, r*R+R) of every stage: their in/out
//     keys, node flows and capacities live in its shared memory (read remotely through DSMEM;
//     reverse arcs relax into the owner's keys with a DSMEM 64-bit compare-and-swap min,
//     common.cuh: the generic 64-bit atomicMin is not atomic on remote shared memory);
//   * the dense min-plus relaxation of boundary s streams the CTA's R rows of tile s from HBM
//     in chunks of NW rows (one cp.async.bulk per chunk, one mbarrier per ring slot; the last
//     warp to finish a chunk refills its slot), from a 16-bit copy of the tiles when the costs
//     fit (half the bytes), with 32-bit keys held in registers when the costs allow (IMAD +
//     VIMNMX per weight, not the quarter-rate DPX VIADDMNMX), while the out_s key vector is
//     gathered from the owner CTAs through DSMEM;
//   * after a boundary's first relaxation since the reset, later ones relax only the columns
//     whose out-key changed (owner dirty bits) when there are at most KSP (8-bit columns: KSP8)
//     of them (frontier);
//   * one cluster barrier per boundary step; phase votes and the t* minimum are reduced from
//     per-CTA slots read by every CTA (no remote atomics, no resets);
//   * the leader CTA traces the canonical path; the whole cluster locates the path's arcs in the
//     positive-arc lists (with each entry's weight beside it); the leader augments.  The lists
//     stay in global memory and are only accessed through L2: written by the leader's SM, read
//     by the other SMs of the cluster, whose L1 would otherwise serve stale lines.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace gwtf {

namespace {

constexpr int CT = 512;      // threads per CTA
constexpr int NW = CT / 32;  // warps per CTA: warp w relaxes rows w, w + NW, ... of a boundary
constexpr int NBMAX = 64;    // chunk slots of the TMA ring (one chunk of NW rows per bulk copy)
constexpr int KSP = 32;       // frontier relaxation when at most this many out-keys changed
constexpr int KSP8 = 256;     // ... with the source-major 8-bit columns (warp per column, rows over the lanes)
constexpr int KQ = 4;        // register-resident key chunks per lane (16-bit rows up to 1,024 weights)
constexpr size_t kSmemMax = 227 * 1024;
constexpr uint64_t INF = ~0ull;
constexpr uint64_t kBig = 1ull << 62;  // INF inside the branch-free relaxation

__host__ __device__ inline size_t al16c(size_t x) { return (x + 15) & ~size_t(15); }
// destination rows per CTA: ceil(n / C) rounded up to a multiple of 4, so that a CTA's slice of a
// source-major 8-bit column starts 4-byte aligned (one 32-bit load covers 4 rows)
__host__ __device__ inline int cl_rows(int n, int C) { return (((n + C - 1) / C) + 3) & ~3; }

struct Misc {  // per-CTA control block; the leader's copy is authoritative
  int64_t F, cost;
  uint64_t tpart[2], red64;
  int32_t inst, A, status, pathlen;
  uint32_t votes[2];  // alternating slots: a CTA is at most one phase ahead of the slowest
  uint32_t vin[2][16];  // vote stamps pushed by every CTA of the cluster (parity, source CTA)
  int32_t red32, pred, nrem, ucnt;
  uint32_t p2;  // 1 << H32, read back through a volatile load (see the relaxation)
};

struct ClLayout {
  size_t misc, kin, kout, g, capE, srcf, snkf, kbuf, kb32, aq, dmask, ring, mbar, total;
  int nbc;  // chunk slots of the ring (chunk = NW consecutive rows = one bulk copy)
};
__host__ __device__ inline ClLayout cl_layout(const Problem& P, int C) {
  ClLayout L;
  const size_t R = (size_t)cl_rows(P.n, C), SR = (size_t)P.S * R;
  size_t o = 0;
  L.misc = o; o += al16c(sizeof(Misc));
  L.mbar = o; o += al16c(NBMAX * 8 + NBMAX * 4);  // full barriers + consumed-row counters
  L.kin = o; o += al16c(SR * 8);
  L.kout = o; o += al16c(SR * 8);
  L.g = o; o += al16c(SR);     // node flows and capacities fit int8 (max_cap <= 32)
  L.capE = o; o += al16c(SR);
  L.srcf = o; o += al16c(R * 4);
  L.snkf = o; o += al16c(R * 4);
  const size_t ldk = P.tile8 ? P.ld8 : P.tile16 ? P.ld16 : P.ld;  // key-vector length
  const size_t slot = P.tile8 ? (size_t)P.ld8 : P.tile16 ? (size_t)P.ld16 * 2 : (size_t)P.ld * 4;  // bytes per row
  L.kbuf = o; o += al16c(ldk * 8);
  L.kb32 = o; o += al16c(ldk * 4);
  L.aq = o; o += al16c((size_t)CT * 12);
  L.dmask = o; o += al16c((size_t)P.S * ((R + 31) / 32) * 4);
  // as many chunk slots in flight as fit, up to the ceil(R / NW) chunks a CTA streams per
  // boundary.  Chunks, not rows: a bulk copy costs the TMA unit a fixed ~46 cycles, so 2 KB
  // rows would cap an SM at ~44 B/cycle (scratch probe), 32-64 KB chunks run at ~80 B/cycle.
  const size_t cbytes = slot * NW;
  const size_t fit = o < kSmemMax ? (kSmemMax - o - 16) / cbytes : 0;
  L.nbc = (int)std::min<size_t>(std::min<size_t>(fit, (size_t)NBMAX), (R + NW - 1) / NW);
  if (L.nbc < 1) L.nbc = 1;  // layout too large: total > kSmemMax rejects it
  L.ring = o; o += al16c((size_t)L.nbc * cbytes);
  L.total = o;
  return L;
}

template <int C>
__global__ void __launch_bounds__(CT, 1) ssp_cluster_kernel(const Problem P, const SspOut o) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) uint8_t sm[];
  const int r = (int)cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cid = blockIdx.x / C;
  const int S = P.S, n = P.n, ld = P.ld, Lt = 2 * S + 1, Lcap = P.Lcap;
  const int R = cl_rows(n, C), v0 = r * R, nr = max(0, min(R, n - v0));
  const ClLayout L = cl_layout(P, C);
  Misc* misc = (Misc*)(sm + L.misc);
  uint64_t* mbar = (uint64_t*)(sm + L.mbar);
  int8_t* g = (int8_t*)(sm + L.g);
  int8_t* capE = (int8_t*)(sm + L.capE);
  int32_t* srcf = (int32_t*)(sm + L.srcf);
  int32_t* snkf = (int32_t*)(sm + L.snkf);
  uint64_t* kbuf = (uint64_t*)(sm + L.kbuf);
  uint32_t* kb32 = (uint32_t*)(sm + L.kb32);
  uint32_t* aq = (uint32_t*)(sm + L.aq);  // staged path arcs: list key, boundary, list length
  // out-keys changed since their boundary was last relaxed: bit (s, lv) of the owner, [S][DW]
  const int DW = (R + 31) / 32;
  uint32_t* dmask = (uint32_t*)(sm + L.dmask);
  const bool track = true;
  uint32_t* spu = aq;                       // frontier step: changed columns (reuses aq)
  uint64_t* spk = (uint64_t*)(aq + KSP8);   // ... and their out-keys
  uint64_t* rowmin = kbuf;                  // ... per-row minima (reuses the gather buffer)
  uint8_t* ring = sm + L.ring;
  const int nbc = L.nbc;
  uint32_t* ecnt = (uint32_t*)(mbar + NBMAX);  // per chunk slot: rows consumed (monotonic)
  // streamed rows: the 16-bit tile copy when present (half the bytes), else the int32 tiles
  const bool t8 = P.tile8 != nullptr;  // 8-bit rows (every arc present, costs < 255): a quarter of int32
  const bool t16 = !t8 && P.tile16 != nullptr;
  const int ldk = t8 ? P.ld8 : t16 ? P.ld16 : ld;  // weights per streamed row
  // frontier threshold (testing override GWTF_DEBUG_FLAGS bits 16..23; 8192: dense only)
  int ksp = t8 ? KSP8 : KSP;
  if (P.debug & 8192) ksp = 0;
  else if ((P.debug >> 16) & 0xFF) ksp = min(ksp, (P.debug >> 16) & 0xFF);
  const uint32_t rowbytes = t8 ? (uint32_t)P.ld8 : t16 ? (uint32_t)P.ld16 * 2 : (uint32_t)ld * 4;
  Misc* M0 = cl.map_shared_rank(misc, 0);
  // per-cluster global scratch: path (t* -> s*) and found (gwtf_api.cpp sizes it)
  uint32_t* path = (uint32_t*)(P.ws_cluster + (size_t)cid * 2 * (2 * (size_t)S * n + 4) * 4);
  int32_t* found = (int32_t*)(path + (2 * S * n + 4));  // list index of path arc e (INT_MAX: none)
  // keys of the owned rows: kin[s * R + lv] / kout[s * R + lv] in shared memory (remote: DSMEM)
  uint64_t* kin = (uint64_t*)(sm + L.kin);
  uint64_t* kout = (uint64_t*)(sm + L.kout);
  // remote views of the owners' arrays
  const uint64_t rmag = ((1ull << 32) + R - 1) / R;  // v / R == (v * rmag) >> 32 for v < 2^32 / R
  auto own = [&](int v) { return (int)(((uint64_t)(uint32_t)v * rmag) >> 32); };
  // 32-bit relaxation keys: (cost << H32) + hops + 1 with 2^H32 > 2Sn+2 hops; a
  // boundary step uses them when every finite out-key cost plus the largest arc weight stays
  // below T32, and absent weights / INF keys are clamped to T32 (never a minimum).
  const int H32 = 32 - __clz(2 * S * n + 2);
  const int CB32 = 32 - H32;
  const uint32_t T32 = CB32 >= 4 ? min((1u << (CB32 - 1)) - 1u, (t16 || t8) ? 0xFFFFu : 0xFFFFFFFFu) : 0u;
  auto ldk_in = [&](int s, int v) -> uint64_t { const int q = own(v); return *(cl.map_shared_rank(kin, q) + s * R + (v - q * R)); };
  auto ldk_out = [&](int s, int v) -> uint64_t { const int q = own(v); return *(cl.map_shared_rank(kout, q) + s * R + (v - q * R)); };
  auto rg = [&](int s, int v) -> int8_t* { const int q = own(v); return cl.map_shared_rank(g, q) + s * R + (v - q * R); };
  auto rcap = [&](int s, int v) -> int8_t* { const int q = own(v); return cl.map_shared_rank(capE, q) + s * R + (v - q * R); };
  auto rsrcf = [&](int v) -> int32_t* { const int q = own(v); return cl.map_shared_rank(srcf, q) + (v - q * R); };
  auto rsnkf = [&](int v) -> int32_t* { const int q = own(v); return cl.map_shared_rank(snkf, q) + (v - q * R); };

  if (tid < 32) misc->vin[tid >> 4][tid & 15] = 0u;  // vote ids start at 1 and never repeat in a launch
  if (tid == 0) {
    misc->p2 = 1u << H32;
    for (int b = 0; b < nbc; ++b) { mbar_init(&mbar[b], 1); ecnt[b] = 0; }
    fence_barrier_init();
  }
  // testing (GWTF_DEBUG_FLAGS & 16): leader-thread cycle counts per phase into stats[1100 + k]
  unsigned long long tlast = clock64();
#define TMARK(k)                                                                       \
  do {                                                                                 \
    if ((P.debug & 16) && r == 0 && tid == 0) {                                        \
      const unsigned long long t_ = clock64();                                         \
      atomicAdd(&P.stats[1100 + (k)], t_ - tlast);                                     \
      tlast = t_;                                                                      \
    }                                                                                  \
  } while (0)
  int slot0 = 0;          // ring slot of the next chunk (uniform over the CTA)
  uint64_t php = 0;       // per-slot mbarrier phase parity (uniform over the CTA)
  int pf_s = -1, pf_n = 0;  // boundary whose first pf_n chunks were streamed ahead (uniform)
  // wait out the chunks streamed ahead for a boundary that is not next after all
  auto drain = [&]() {
    for (int k = 0, b = slot0; k < pf_n; ++k, b = b + 1 == nbc ? 0 : b + 1) {
      mbar_wait(&mbar[b], (uint32_t)(php >> b) & 1u);
      php ^= 1ull << b;
    }
    slot0 = (slot0 + pf_n) % nbc;
    pf_s = -1;
    pf_n = 0;
    __syncthreads();  // every warp is past the waits before a slot is re-armed
  };
  uint32_t vote_id = 0;   // phase counter of the votes (uniform over the cluster)
  uint32_t tphase = 0;    // phase counter of the t* reductions
  __syncthreads();

  for (;;) {
    if (r == 0 && tid == 0) {
      int q = atomicAdd(&P.counters[4], 1);
      if (P.sel) q = q < *P.sel_count ? P.sel[q] : P.B;  // subset solve
      misc->inst = q;
    }
    cl.sync();
    const int inst = M0->inst;
    cl.sync();  // every CTA has read the leader's value before any CTA exits or it is rewritten
    if (inst >= P.B) break;
    const int64_t M = P.supply[inst];
    const int32_t maxw = *(volatile int32_t*)&P.counters[6];  // largest finite arc weight (bound)
    const int32_t* tile = P.tile + (size_t)inst * (S - 1) * n * ld;
    const int32_t* src = P.src + (size_t)inst * n;
    const int32_t* snk = P.snk + (size_t)inst * n;
    uint32_t* arcs = P.arcs + (size_t)inst * (S - 1) * Lcap;
    int32_t* arcw = P.arcw + (size_t)inst * (S - 1) * Lcap;  // weight of each list entry (no tile fetch)
    int32_t* cnt = P.arc_cnt + (size_t)inst * (S - 1);
    for (int k = tid; k < S * R; k += CT) {
      const int s = k / R, v = v0 + k % R;
      g[k] = 0;
      capE[k] = (v < n && P.alive[((size_t)inst * S + s) * n + v]) ? (int8_t)P.cap[((size_t)inst * S + s) * n + v] : 0;
    }
    for (int k = tid; k < R; k += CT) { srcf[k] = 0; snkf[k] = 0; }
    if (r == 0) {
      if (tid == 0) { misc->F = 0; misc->cost = 0; misc->A = 0; misc->status = 0; misc->votes[0] = 0; misc->votes[1] = 0; }
      for (int k = tid; k < S - 1; k += CT) __stcg(&cnt[k], 0);
    }
    cl.sync();

    // vote: did any CTA of the cluster change something in this phase?  (cluster barrier)
    auto vote = [&](int ch) -> bool {
      // a thread that changed something stamps its CTA's slot with the vote id (idempotent); the
      // cluster barrier orders every stamp before the reads, so no CTA-level reduction is needed
      // a warp that changed something pushes the stamp into its CTA's slot in every CTA (lane q to
      // CTA q; idempotent) before the barrier, whose skew hides the remote stores; after it every
      // CTA reads its own slots only
      ++vote_id;
      const int p = vote_id & 1;
      if (__any_sync(0xffffffffu, ch) && lane < C) *cl.map_shared_rank(&misc->vin[p][r], lane) = vote_id;
      cl.sync();
      bool res = false;
      for (int q = 0; q < C; ++q) res |= *(volatile uint32_t*)&misc->vin[p][q] == vote_id;
      return res;
    };

    for (;;) {  // successive shortest paths
      const int64_t F = M0->F;
      if (F >= M || M0->status) break;
      for (int k = tid; k < S * R; k += CT) {  // own rows: INF, then s* -> in_0, in_0 -> out_0
        const int s = k / R, lv = k - s * R, v = v0 + lv;
        if (lv >= nr) continue;
        uint64_t ki = INF, ko = INF;
        if (s == 0 && src[v] != kAbsent) {
          ki = ((uint64_t)(uint32_t)src[v] << kHopBits) | 1ull;
          if (g[lv] < capE[lv]) ko = ki + 1;
        }
        kin[k] = ki;
        kout[k] = ko;
      }
      if (track) for (int k = tid; k < S * DW; k += CT) dmask[k] = 0u;
      uint64_t fresh = ~0ull;
      uint64_t tkey = INF;
      uint64_t fwd = S > 1 ? 1ull : 0ull, bwd = 1ull;
      bool tdirty = S == 1, trev = false;
      cl.sync();
      for (;;) {
        // ---- forward: dense min-plus relaxation of the dirty boundaries (streamed tiles) ----
        for (int s = 0; s + 1 < S; ++s) {
          if (!((fwd >> s) & 1ull)) continue;
          fwd &= ~(1ull << s);
          if (r == 0 && tid == 0) atomicAdd(&P.stats[0], 1ull);
          TMARK(9);
          const bool fresh_s = (fresh >> s) & 1ull;
          fresh &= ~(1ull << s);
          if (!fresh_s && ksp > 0 && C * DW <= CT) {
            // ---- frontier relaxation: after its first relaxation since the reset, boundary s only
            // needs the columns u whose out-key changed since (dirty bits of the owners, DSMEM);
            // in_{s+1,v} = min(in_{s+1,v}, out_{s,u} + w(u,v)) over those u is the same fixed point
            if (tid == 0) { misc->ucnt = 0; misc->red32 = 0; }
            __syncthreads();
            uint32_t m = 0;  // one mask word per thread (C * DW <= CT)
            if (tid < C * DW) {
              m = *(cl.map_shared_rank(dmask, tid / DW) + s * DW + (tid % DW));
              if (m) atomicAdd(&misc->red32, __popc(m));
            }
            __syncthreads();
            const int nU = misc->red32;
            if ((P.debug & 2048) && r == 0 && tid == 0)  // testing: histogram of changed columns
              atomicAdd(&P.stats[1200 + (nU == 0 ? 0 : 32 - __clz(nU))], 1ull);
            if (nU <= ksp) {
              if (m) {
                int k = atomicAdd(&misc->ucnt, __popc(m));
                for (; m; m &= m - 1) spu[k++] = (tid / DW) * R + (tid % DW) * 32 + (__ffs(m) - 1);
              }
              for (int j = tid; j < nr; j += CT) rowmin[j] = INF;
              __syncthreads();
              if (!t8) {  // the int32 path reads the keys from shared memory
                for (int i = tid; i < nU; i += CT) spk[i] = ldk_out(s, (int)spu[i]);
                __syncthreads();
              }
              if (t8) {
                // source-major 8-bit columns: warp w takes columns w, w + NW, ... (eight in flight),
                // lane l the CTA's rows 4l .. 4l+3 of each (one aligned 32-bit load); per-lane row
                // minima in registers, one shared-memory atomicMin per (warp, row)
                const uint8_t* colb = P.tile8t + ((size_t)inst * (S - 1) + s) * (size_t)n * P.ld8 + v0;
                for (int jb = 0; jb < nr; jb += 128) {
                  uint64_t rm[4] = {INF, INF, INF, INF};
                  const bool on = jb + 4 * lane < nr;
                  for (int i0 = warp; i0 < nU; i0 += 8 * NW) {
                    // the columns' bytes (HBM) and their out-keys (the owners, one broadcast DSMEM
                    // load per warp) in flight together
                    uint32_t wv[8];
                    uint64_t kv[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                      const int i = i0 + c * NW;
                      const int u = i < nU ? (int)spu[i] : 0;
                      wv[c] = (i < nU && on) ? *(const uint32_t*)(colb + (size_t)u * P.ld8 + jb + 4 * lane) : 0u;
                      kv[c] = i < nU ? ldk_out(s, u) : INF;
                    }
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                      const uint64_t kk = kv[c];
                      if (kk == INF) continue;
#pragma unroll
                      for (int k = 0; k < 4; ++k)  // tile8 holds no absent arc
                        rm[k] = umin64(rm[k], kk + ((uint64_t)((wv[c] >> (8 * k)) & 0xFFu) << kHopBits) + 1ull);
                    }
                  }
#pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    const int j = jb + 4 * lane + k;
                    if (j < nr && rm[k] != INF) atomicMin((unsigned long long*)&rowmin[j], (unsigned long long)rm[k]);
                  }
                }
              } else {
                for (int t = tid; t < nr * nU; t += CT) {
                  const int j = t / nU, i = t - j * nU;
                  const uint64_t k = spk[i];
                  if (k == INF) continue;
                  const int32_t w = tile[((size_t)s * n + v0 + j) * ld + spu[i]];
                  if (w == kAbsent) continue;
                  atomicMin((unsigned long long*)&rowmin[j], (unsigned long long)(k + ((uint64_t)(uint32_t)w << kHopBits) + 1ull));
                }
              }
              __syncthreads();
              int chs = 0;
              for (int j = tid; j < nr; j += CT) {
                const uint64_t best = rowmin[j];
                const int e = (s + 1) * R + j;
                uint64_t kv = kin[e];
                if (best < kv) { kin[e] = best; kv = best; chs = 1; }
                if (kv != INF && g[e] < capE[e] && kv + 1 < kout[e]) {
                  kout[e] = kv + 1;
                  chs = 1;
                  atomicOr(&dmask[(s + 1) * DW + (j >> 5)], 1u << (j & 31));
                }
              }
              if (r == 0 && tid == 0) atomicAdd(&P.stats[11], 1ull);
              TMARK(10);  // frontier relaxation
              const bool vfs = vote(chs);
              for (int k = tid; k < DW; k += CT) dmask[s * DW + k] = 0u;  // every CTA has read it
              TMARK(11);  // frontier vote
              if (vfs) {
                if (s + 1 < S - 1) fwd |= 1ull << (s + 1);
                else tdirty = true;
                bwd |= 1ull << (s + 1);
              }
              continue;
            }
          }
          // chunk k (rows k*NW .. k*NW+NW-1, one per warp) goes to slot (slot0 + k) % nbc; the last
          // warp to finish a chunk refills its slot with chunk k + nbc, or, past the last chunk,
          // with chunk k + nbc - nch of boundary s + 1: the forward sweep's likely next step is
          // streamed across the vote (speculative; a mismatch drains it)
          const int nch = (nr + NW - 1) / NW;
          const uint32_t cbytes = (uint32_t)NW * rowbytes;
          auto rows_of = [&](int sb) -> const uint8_t* {
            if (t8) return P.tile8 + (((size_t)inst * (S - 1) + sb) * n + v0) * P.ld8;
            return t16 ? (const uint8_t*)(P.tile16 + (((size_t)inst * (S - 1) + sb) * n + v0) * P.ld16)
                       : (const uint8_t*)(tile + ((size_t)sb * n + v0) * ld);
          };
          const uint8_t* rows = rows_of(s);
          auto issue_from = [&](const uint8_t* src, int k, int b) {  // chunk k of `src` into slot b
            const uint32_t bytes = (uint32_t)min(NW, nr - k * NW) * rowbytes;
            mbar_arrive_expect_tx(&mbar[b], bytes);
            bulk_g2s(ring + (size_t)b * cbytes, src + (size_t)k * cbytes, bytes, &mbar[b]);
          };
          auto issue = [&](int k, int b) { issue_from(rows, k, b); };
          const bool nostream = P.debug & 64;  // testing: time the compute without the stream
          if (pf_n && pf_s != s) drain();     // the speculation missed
          const int pre = pf_n;                // chunks of this boundary already in flight
          const int nxt = (s + 2 < S && !nostream && !(P.debug & 512) && ((fresh >> (s + 1)) & 1ull)) ? s + 1 : -1;
          const uint8_t* rows_next = nxt >= 0 ? rows_of(nxt) : nullptr;
          pf_s = nxt;
          pf_n = nxt >= 0 ? min(nbc, nch) : 0;
          if (tid == 0 && !nostream) {
            fence_proxy_async_smem();
            for (int k = pre; k < min(nbc, nch); ++k) issue(k, slot0 + k < nbc ? slot0 + k : slot0 + k - nbc);
            for (int k2 = 0; k2 < pf_n && k2 + nch < nbc; ++k2)  // free slots: next boundary now
              issue_from(rows_next, k2, (slot0 + nch + k2) % nbc);
          }
          // lane k of warp w prefetches the keys of the warp's row j = k * NW + w of in/out_{s+1}
          // (consumed by lane k after the row's minimum; rows beyond 32 per warp load late)
          uint64_t pkv = INF, pko = INF;
          int pres = 0;  // in -> out residual of that row
          if (lane < nch && lane * NW + warp < nr) {
            const int jr = lane * NW + warp;
            pkv = kin[(s + 1) * R + jr];
            pko = kout[(s + 1) * R + jr];
            pres = g[(s + 1) * R + jr] < capE[(s + 1) * R + jr];
          }
          TMARK(13);  // stream issue + row-key prefetch
          const uint32_t lim = T32 > (uint32_t)maxw ? T32 - (uint32_t)maxw : 0u;
          int wide = lim == 0u || (P.debug & 32) || (t8 && T32 < 255u);  // testing (32): force the 64-bit path
          const bool kreg8 = t8 && ldk == 16 * 32 * 2;  // 8-bit rows of 1,024 weights
          const bool perm8 = kreg8 && !nostream;          // the register-key layout below
          for (int u0 = 0; u0 < ldk; u0 += 4 * CT) {  // gather out_s from L2 (4 loads in flight)
            uint64_t kk[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int u = u0 + j * CT + tid;
              kk[j] = u < n ? dsmem_ld_u64(dsmem_addr(kout + s * R + (u - own(u) * R), (uint32_t)own(u))) : INF;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int u = u0 + j * CT + tid;
              if (u >= ldk) break;
              kbuf[u] = kk[j] == INF ? kBig : kk[j];
              uint32_t k32 = T32 << H32;
              if (kk[j] != INF) {
                const uint64_t c = kk[j] >> kHopBits, hops = kk[j] & ((1ull << kHopBits) - 1);
                if (c >= lim || hops + 1 >= (1ull << H32)) wide = 1;
                k32 = ((uint32_t)c << H32) + (uint32_t)hops + 1u;
              }
              // 8-bit rows of 1,024 weights: lane l's register keys (columns 16 (l + 32q) + 4t + e) are
              // stored at uint4 (4q + t) * 32 + l, so that the warps' 16-byte loads below are
              // conflict-free (the natural layout puts a lane's pieces 64 B apart: 4-way conflicts)
              kb32[perm8 ? (((((u >> 9) << 2) + ((u >> 2) & 3)) << 5) + ((u >> 4) & 31)) * 4 + (u & 3) : u] = k32;
            }
          }
          wide = __syncthreads_or(wide) && !nostream;
          // 16-bit rows of up to 1,024 weights: every lane keeps the 32-bit keys of its own
          // columns (chunks c = lane + 32q, 8 weights each) in registers for the whole step
          const bool kreg = t16 && ldk <= 8 * 32 * KQ;
          uint4 kr[2 * KQ];
          if (kreg && !wide) {
            const uint4* kv4 = (const uint4*)kb32;
#pragma unroll
            for (int q = 0; q < KQ; ++q) {
              const int c = lane + 32 * q;
              kr[2 * q] = c < ldk / 8 ? kv4[2 * c] : make_uint4(0u, 0u, 0u, 0u);
              kr[2 * q + 1] = c < ldk / 8 ? kv4[2 * c + 1] : make_uint4(0u, 0u, 0u, 0u);
            }
          } else if (kreg8 && !wide) {  // lane chunk c = lane + 32q holds columns 16c .. 16c+15
            const uint4* kv4 = (const uint4*)kb32;
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
              for (int t = 0; t < 4; ++t) kr[4 * q + t] = kv4[(4 * q + t) * 32 + lane];
          }
          TMARK(0);
          int ch = 0;
          // the lane holding row j's prefetched keys applies its minimum (and the fused node arc)
          auto apply = [&](int k, int j, uint64_t best) {
            if (lane != (k & 31)) return;
            const int e = (s + 1) * R + j;
            uint64_t kv = pkv, ko = pko;
            int res = pres;
            if (k >= 32) { kv = kin[e]; ko = kout[e]; res = g[e] < capE[e]; }
            if (best < kv) { kin[e] = best; kv = best; ch = 1; }
            if (kv != INF && res && kv + 1 < ko) {
              kout[e] = kv + 1;
              ch = 1;
              if (track) atomicOr(&dmask[(s + 1) * DW + (j >> 5)], 1u << (j & 31));
            }
          };
          // every lane is done with its row of slot b (its values fed the warp minimum); the last
          // warp to finish the chunk refills the slot through the async proxy
          auto release = [&](int k, int b) {
            php ^= 1ull << b;  // slot b's phase advanced (every thread tracks every chunk)
            const int k2 = k + nbc - nch;  // chunk of the next boundary that reuses slot b
            if (lane == 0 && !nostream && (k + nbc < nch || (k2 >= 0 && k2 < pf_n))) {
              if (atomicAdd(&ecnt[b], 1u) % NW == NW - 1) {  // last reader of the chunk
                __threadfence_block();
                fence_proxy_async_smem();
                if (k + nbc < nch) issue(k + nbc, b);
                else issue_from(rows_next, k2, b);
              }
            }
          };
          const uint32_t p2 = *(volatile const uint32_t*)&misc->p2;  // 2^H32, opaque to ptxas (below)
          if (kreg8 && !wide && !nostream) {
            // 8-bit rows of 1,024 weights (stress): two 16-byte loads per lane, 32 register keys;
            // every byte is masked out (BFE-like LOP / SHF) before the IMAD by 2^H32
            for (int k = 0, b = slot0; k < nch; ++k, b = b + 1 == nbc ? 0 : b + 1) {
              const int j = k * NW + warp;
              if (j < nr) {
                mbar_wait(&mbar[b], (uint32_t)(php >> b) & 1u);
                if (k == 0) TMARK(12);  // first chunk landed
                const uint4* row = (const uint4*)(ring + (size_t)b * cbytes + (size_t)warp * rowbytes) + lane;
                const uint4 w0 = row[0], w1 = row[32];
                uint32_t a0 = 0xFFFFFFFFu, a1 = a0, a2 = a0, a3 = a0;
                auto word = [&](uint32_t wd, const uint4& kk) {
                  a0 = min(a0, (wd & 0xFFu) * p2 + kk.x);
                  a1 = min(a1, ((wd >> 8) & 0xFFu) * p2 + kk.y);
                  a2 = min(a2, ((wd >> 16) & 0xFFu) * p2 + kk.z);
                  a3 = min(a3, (wd >> 24) * p2 + kk.w);
                };
                word(w0.x, kr[0]); word(w0.y, kr[1]); word(w0.z, kr[2]); word(w0.w, kr[3]);
                word(w1.x, kr[4]); word(w1.y, kr[5]); word(w1.z, kr[6]); word(w1.w, kr[7]);
                const uint32_t acc = __reduce_min_sync(0xffffffffu, min(min(a0, a1), min(a2, a3)));
                apply(k, j, (acc >> H32) >= T32 ? INF
                                                : ((uint64_t)(acc >> H32) << kHopBits) | (uint64_t)(acc & ((1u << H32) - 1u)));
              }
              release(k, b);
            }
          } else if (t16 && kreg && H32 >= 16 && ldk == 8 * 32 * KQ && !wide && !nostream) {
            // the stress fast path: 1,024-weight 16-bit rows, register-resident 32-bit keys, no
            // predicates.  (w << H32) + key is one IMAD by p2 (ptxas would otherwise fuse a shift's
            // add with the min into the quarter-rate DPX VIADDMNMX); the low half-word needs no
            // mask (its high bits leave the register), the high one a shift.
            for (int k = 0, b = slot0; k < nch; ++k, b = b + 1 == nbc ? 0 : b + 1) {
              const int j = k * NW + warp;
              if (j < nr) {
                mbar_wait(&mbar[b], (uint32_t)(php >> b) & 1u);
                const uint4* row = (const uint4*)(ring + (size_t)b * cbytes + (size_t)warp * rowbytes) + lane;
                uint4 w[KQ];
#pragma unroll
                for (int q = 0; q < KQ; ++q) w[q] = row[32 * q];
                uint32_t a0 = 0xFFFFFFFFu, a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
                for (int q = 0; q < KQ; ++q) {
                  a0 = min(a0, w[q].x * p2 + kr[2 * q].x);
                  a1 = min(a1, (w[q].x >> 16) * p2 + kr[2 * q].y);
                  a2 = min(a2, w[q].y * p2 + kr[2 * q].z);
                  a3 = min(a3, (w[q].y >> 16) * p2 + kr[2 * q].w);
                  a0 = min(a0, w[q].z * p2 + kr[2 * q + 1].x);
                  a1 = min(a1, (w[q].z >> 16) * p2 + kr[2 * q + 1].y);
                  a2 = min(a2, w[q].w * p2 + kr[2 * q + 1].z);
                  a3 = min(a3, (w[q].w >> 16) * p2 + kr[2 * q + 1].w);
                }
                const uint32_t acc = __reduce_min_sync(0xffffffffu, min(min(a0, a1), min(a2, a3)));
                apply(k, j, (acc >> H32) >= T32 ? INF
                                                : ((uint64_t)(acc >> H32) << kHopBits) | (uint64_t)(acc & ((1u << H32) - 1u)));
              }
              release(k, b);
            }
          } else
          for (int k = 0, b = slot0; k < nch; ++k, b = b + 1 == nbc ? 0 : b + 1) {
            const int j = k * NW + warp;
            if (j < nr) {
            if (!nostream) mbar_wait(&mbar[b], (uint32_t)(php >> b) & 1u);
            const uint8_t* rowb = ring + (size_t)b * cbytes + (size_t)warp * rowbytes;
            uint64_t best;
            if (!wide) {
              // 32-bit: per weight one shift, one add and one min (IADD + VIMNMX, full rate; the fused
              // DPX VIADDMNMX issues at a quarter of that rate on sm_100a); four
              // independent accumulators keep the add-min chains short
              const uint4* kv4 = (const uint4*)kb32;
              uint32_t a0 = 0xFFFFFFFFu, a1 = a0, a2 = a0, a3 = a0;
              if (t8) {  // 8-bit rows (any n): 16 weights per 16-byte load, keys from shared memory
                const uint4* row = (const uint4*)rowb;
                for (int c = lane; c < ldk / 16; c += 32) {
                  const uint4 w = row[c];
                  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    const uint4 kk = kv4[4 * c + t];
                    a0 = min(a0, (ws[t] & 0xFFu) * p2 + kk.x);
                    a1 = min(a1, ((ws[t] >> 8) & 0xFFu) * p2 + kk.y);
                    a2 = min(a2, ((ws[t] >> 16) & 0xFFu) * p2 + kk.z);
                    a3 = min(a3, (ws[t] >> 24) * p2 + kk.w);
                  }
                }
              } else if (t16) {
                // 16-bit rows, pre-clamped (absent = T32): two weights per word, shifted into the
                // cost field; with H32 >= 16 the low weight is one shift, the high one shift + mask
                const uint4* row = (const uint4*)rowb;
                if (kreg && H32 >= 16) {
                  // IMAD + VIMNMX: 3 issue slots per weight against 5 for SHF + VIADDMNMX
#pragma unroll
                  for (int q = 0; q < KQ; ++q) {
                    if (lane + 32 * q < ldk / 8) {
                      const uint4 w = row[lane + 32 * q];
                      a0 = min(a0, w.x * p2 + kr[2 * q].x);          // low half: bits above 32 drop
                      a1 = min(a1, (w.x >> 16) * p2 + kr[2 * q].y);
                      a2 = min(a2, w.y * p2 + kr[2 * q].z);
                      a3 = min(a3, (w.y >> 16) * p2 + kr[2 * q].w);
                      a0 = min(a0, w.z * p2 + kr[2 * q + 1].x);
                      a1 = min(a1, (w.z >> 16) * p2 + kr[2 * q + 1].y);
                      a2 = min(a2, w.w * p2 + kr[2 * q + 1].z);
                      a3 = min(a3, (w.w >> 16) * p2 + kr[2 * q + 1].w);
                    }
                  }
                } else {
#pragma unroll 2
                  for (int c = lane; c < ldk / 8; c += 32) {
                    const uint4 w = row[c];
                    const uint4 ka = kv4[2 * c], kc = kv4[2 * c + 1];
                    a0 = min(a0, (w.x & 0xFFFFu) * p2 + ka.x);
                    a1 = min(a1, (w.x >> 16) * p2 + ka.y);
                    a2 = min(a2, (w.y & 0xFFFFu) * p2 + ka.z);
                    a3 = min(a3, (w.y >> 16) * p2 + ka.w);
                    a0 = min(a0, (w.z & 0xFFFFu) * p2 + kc.x);
                    a1 = min(a1, (w.z >> 16) * p2 + kc.y);
                    a2 = min(a2, (w.w & 0xFFFFu) * p2 + kc.z);
                    a3 = min(a3, (w.w >> 16) * p2 + kc.w);
                  }
                }
              } else {
                const int4* row = (const int4*)rowb;
#pragma unroll 4
                for (int c = lane; c < ld / 4; c += 32) {
                  const int4 w = row[c];
                  const uint4 kq = kv4[c];
                  a0 = min(a0, min((uint32_t)w.x, T32) * p2 + kq.x);
                  a1 = min(a1, min((uint32_t)w.y, T32) * p2 + kq.y);
                  a2 = min(a2, min((uint32_t)w.z, T32) * p2 + kq.z);
                  a3 = min(a3, min((uint32_t)w.w, T32) * p2 + kq.w);
                }
              }
              const uint32_t acc = __reduce_min_sync(0xffffffffu, min(min(a0, a1), min(a2, a3)));
              best = (acc >> H32) >= T32 ? INF
                                         : ((uint64_t)(acc >> H32) << kHopBits) | (uint64_t)(acc & ((1u << H32) - 1u));
            } else {
              // 64-bit branch-free: keys are < 2^62 when finite (DESIGN.md 2.2 bound) and kBig =
              // 2^62 stands for INF in kbuf; absent weights (INT32_MAX, or 0xFFFF -> 2^42 in the
              // 16-bit rows) push a candidate to >= 2^62; nothing overflows 64 bits
              uint64_t acc = kBig, acc2 = kBig;
              if (t8) {  // 8-bit rows hold no absent arc; padding columns carry kBig keys
                const uint32_t* row = (const uint32_t*)rowb;
                for (int c = lane; c < ldk / 4; c += 32) {
                  const uint32_t wd = row[c];  // 4 weights
                  const ulonglong2 k01 = *(const ulonglong2*)(kbuf + 4 * c);
                  const ulonglong2 k23 = *(const ulonglong2*)(kbuf + 4 * c + 2);
                  acc = umin64(acc, k01.x + ((uint64_t)(wd & 0xFFu) << kHopBits) + 1ull);
                  acc2 = umin64(acc2, k01.y + ((uint64_t)((wd >> 8) & 0xFFu) << kHopBits) + 1ull);
                  acc = umin64(acc, k23.x + ((uint64_t)((wd >> 16) & 0xFFu) << kHopBits) + 1ull);
                  acc2 = umin64(acc2, k23.y + ((uint64_t)(wd >> 24) << kHopBits) + 1ull);
                }
              } else if (t16) {
                const uint2* row = (const uint2*)rowb;
                auto w64 = [&](uint32_t h) -> uint64_t { return h == T32 ? (1ull << 42) : (uint64_t)h; };
#pragma unroll 2
                for (int c = lane; c < ldk / 4; c += 32) {
                  const uint2 w = row[c];  // 4 weights
                  const ulonglong2 k01 = *(const ulonglong2*)(kbuf + 4 * c);
                  const ulonglong2 k23 = *(const ulonglong2*)(kbuf + 4 * c + 2);
                  acc = umin64(acc, k01.x + (w64(w.x & 0xFFFFu) << kHopBits) + 1ull);
                  acc2 = umin64(acc2, k01.y + (w64(w.x >> 16) << kHopBits) + 1ull);
                  acc = umin64(acc, k23.x + (w64(w.y & 0xFFFFu) << kHopBits) + 1ull);
                  acc2 = umin64(acc2, k23.y + (w64(w.y >> 16) << kHopBits) + 1ull);
                }
              } else {
                const int4* row = (const int4*)rowb;
#pragma unroll 2
                for (int c = lane; c < ld / 4; c += 32) {
                  const int4 w = row[c];
                  const ulonglong2 k01 = *(const ulonglong2*)(kbuf + 4 * c);
                  const ulonglong2 k23 = *(const ulonglong2*)(kbuf + 4 * c + 2);
                  acc = umin64(acc, k01.x + ((uint64_t)(uint32_t)w.x << kHopBits) + 1ull);
                  acc2 = umin64(acc2, k01.y + ((uint64_t)(uint32_t)w.y << kHopBits) + 1ull);
                  acc = umin64(acc, k23.x + ((uint64_t)(uint32_t)w.z << kHopBits) + 1ull);
                  acc2 = umin64(acc2, k23.y + ((uint64_t)(uint32_t)w.w << kHopBits) + 1ull);
                }
              }
              acc = umin64(acc, acc2);
              for (int off = 16; off > 0; off >>= 1)
                acc = umin64(acc, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)acc, off));
              best = acc >= kBig ? INF : acc;
            }
            apply(k, j, best);
            }
            release(k, b);
          }
          slot0 = (slot0 + nch) % nbc;
          TMARK(1);
          const bool vf = vote(ch);
          if (track) for (int k = tid; k < DW; k += CT) dmask[s * DW + k] = 0u;  // every CTA read it
          TMARK(2);
          if (vf) {
            if (s + 1 < S - 1) fwd |= 1ull << (s + 1);
            else tdirty = true;
            bwd |= 1ull << (s + 1);
          }
        }
        // ---- out_{S-1} -> t* ----
        if (tdirty) {
          tdirty = false;
          // every CTA publishes its partial minimum in its own slot (double-buffered by the
          // phase parity), then every CTA reduces all C slots: no remote atomics, no resets
          const int slot = (int)(++tphase & 1u);
          if (tid == 0) misc->red64 = INF;
          __syncthreads();
          uint64_t tc = INF;
          for (int lv = tid; lv < nr; lv += CT) {
            const int v = v0 + lv;
            const uint64_t k = kout[(S - 1) * R + lv];
            if (snk[v] != kAbsent && k != INF) tc = umin64(tc, k + ((uint64_t)(uint32_t)snk[v] << kHopBits) + 1ull);
          }
          for (int off = 16; off > 0; off >>= 1)
            tc = umin64(tc, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)tc, off));
          if (lane == 0 && tc != INF) atomicMin((unsigned long long*)&misc->red64, (unsigned long long)tc);
          __syncthreads();
          if (tid == 0) misc->tpart[slot] = misc->red64;
          cl.sync();
          uint64_t tn = INF;
          for (int q = 0; q < C; ++q) tn = umin64(tn, cl.map_shared_rank(misc, q)->tpart[slot]);
          if (tn < tkey) { tkey = tn; trev = true; }
        }
        TMARK(3);
        // ---- t* -> out_{S-1} (reverse sink arcs) ----
        if (trev) {
          trev = false;
          int ch = 0;
          if (tkey != INF)
            for (int lv = tid; lv < nr; lv += CT) {
              if (snkf[lv] <= 0) continue;
              const uint64_t c = tkey - ((uint64_t)(uint32_t)snk[v0 + lv] << kHopBits) + 1ull;
              if (c < kout[(S - 1) * R + lv]) {
                kout[(S - 1) * R + lv] = c;
                ch = 1;
                if (track) atomicOr(&dmask[(S - 1) * DW + (lv >> 5)], 1u << (lv & 31));
              }
            }
          if (vote(ch)) bwd |= 1ull << (S - 1);
        }
        TMARK(4);
        // ---- backward: reverse node arcs (owners) + reverse inter-stage arcs (DSMEM atomicMin) ----
        for (int s = S - 1; s >= 0; --s) {
          if (!((bwd >> s) & 1ull)) continue;
          bwd &= ~(1ull << s);
          if (r == 0 && tid == 0) atomicAdd(&P.stats[1], 1ull);
          for (int lv = tid; lv < nr; lv += CT) {
            if (g[s * R + lv] <= 0) continue;
            const uint64_t ko = kout[s * R + lv];
            if (ko != INF && ko + 1 < kin[s * R + lv]) kin[s * R + lv] = ko + 1;
          }
          if (s == 0) { cl.sync(); break; }
          const uint32_t* al = arcs + (size_t)(s - 1) * Lcap;
          // the thread's first list entry is fetched together with the list length (one L2 round
          // trip instead of two; entries past the length are never used)
          const int e0 = r * CT + tid;
          uint32_t ent0 = 0u;
          int32_t w0 = 0;
          if (e0 < Lcap) { ent0 = __ldcg(&al[e0]); w0 = __ldcg(&arcw[(size_t)(s - 1) * Lcap + e0]); }
          const int c = __ldcg(&cnt[s - 1]);
          int ch = 0;
          for (int e = e0; e < c; e += C * CT) {
            const uint32_t ent = e == e0 ? ent0 : __ldcg(&al[e]);
            const int32_t w = e == e0 ? w0 : __ldcg(&arcw[(size_t)(s - 1) * Lcap + e]);
            const int u = (int)(ent >> 20), v = (int)((ent >> 8) & 0xFFFu);
            uint64_t ki = ldk_in(s, v);
            const uint64_t kov = ldk_out(s, v);
            if (*rg(s, v) > 0 && kov != INF && kov + 1 < ki) ki = kov + 1;
            if (ki == INF) continue;
            const uint64_t cand = ki - ((uint64_t)(uint32_t)w << kHopBits) + 1ull;
            const int q = own(u);
            const uint64_t old = dsmem_atomic_min_u64(dsmem_addr(kout + (s - 1) * R + (u - q * R), (uint32_t)q), cand);
            if (track && cand < old) {
              const int lu = u - q * R;
              asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(dsmem_addr(dmask + (s - 1) * DW + (lu >> 5), (uint32_t)q)),
                           "r"(1u << (lu & 31)) : "memory");
            }
            if (cand < old) ch = 1;
          }
          if (vote(ch)) {
            fwd |= 1ull << (s - 1);
            bwd |= 1ull << (s - 1);
          }
        }
        TMARK(5);
        if (r == 0 && tid == 0) atomicAdd(&P.stats[3], 1ull);
        if (!(fwd | bwd) && !tdirty && !trev) break;
      }
      if (tkey == INF) break;  // t* unreachable: F is maximal
      if ((P.debug & 8) && r == 0 && tid == 0) {  // testing: record the key of every augmenting path
        const unsigned long long a = atomicAdd(&P.stats[10], 1ull);
        if (a < 1000) P.stats[1000 + a] = tkey;
      }
      if ((P.debug & 4) && r == 0 && M0->A == (P.debug >> 8)) {  // testing: dump the converged keys
        if (tid == 0) {
          P.stats[8] = tkey;
          for (int s2 = 0; s2 < S && 2 * S * n + 16 < 2000; ++s2)
            for (int i = 0; i < n; ++i) {
              P.stats[16 + (s2 * n + i) * 3 + 0] = ldk_in(s2, i);
              P.stats[16 + (s2 * n + i) * 3 + 1] = ldk_out(s2, i);
              P.stats[16 + (s2 * n + i) * 3 + 2] = (unsigned long long)*rg(s2, i);
            }
          misc->status = 9;
        }
      }
      if ((P.debug & 4) && M0->A == (P.debug >> 8)) { cl.sync(); break; }

      TMARK(9);
      // ---- trace the canonical augmenting path and augment (leader CTA) ----
      if (r == 0) {
        auto key_of = [&](int id) -> uint64_t {
          const int l = id >> 16, p = id & 0xFFFF;
          if (l == 0) return 0ull;
          if (l == Lt) return tkey;
          if (l & 1) return ldk_in((l - 1) >> 1, p);
          return ldk_out((l >> 1) - 1, p);
        };
        int x = Lt << 16, len = 1, err = 0;
        if (tid == 0) path[0] = (uint32_t)x;
        while (x != 0) {
          const int l = x >> 16, p = x & 0xFFFF;
          const uint64_t kx = key_of(x);
          if (tid == 0) misc->red32 = INT_MAX;
          __syncthreads();
          int pred = -1;
          if (l == Lt) {  // lowest i with out_{S-1,i} + (snk_i, 1) == key(t*)
            for (int i = tid; i < n; i += CT) {
              if (snk[i] == kAbsent) continue;
              const uint64_t k = ldk_out(S - 1, i);
              if (k != INF && k + ((uint64_t)(uint32_t)snk[i] << kHopBits) + 1ull == kx) { atomicMin(&misc->red32, i); break; }
            }
            __syncthreads();
            if (misc->red32 != INT_MAX) pred = ((2 * S) << 16) | misc->red32;
          } else if (l & 1) {  // in_{s,i}: s* / lowest tight out_{s-1,u} (recorded arg-min), then out_{s,i}
            const int s = (l - 1) >> 1, i = p;
            if (s == 0) {
              if (src[i] != kAbsent && ((((uint64_t)(uint32_t)src[i]) << kHopBits) | 1ull) == kx) pred = 0;
            } else {  // lowest tight u of row i of boundary s-1: 4 weights and 4 out-keys per thread
              const int4* row4 = (const int4*)(tile + ((size_t)(s - 1) * n + i) * ld);
              for (int c = tid; c < ld / 4; c += CT) {
                const int4 w4 = row4[c];
                const int32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
                uint64_t k4[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) k4[j] = (ws[j] != kAbsent && 4 * c + j < n) ? ldk_out(s - 1, 4 * c + j) : INF;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  if (k4[j] != INF && k4[j] + ((uint64_t)(uint32_t)ws[j] << kHopBits) + 1ull == kx) {
                    atomicMin(&misc->red32, 4 * c + j);
                    break;
                  }
              }
              __syncthreads();
              if (misc->red32 != INT_MAX) pred = ((2 * s) << 16) | misc->red32;
            }
            if (pred < 0) {
              const uint64_t ko = ldk_out(s, i);
              if (*rg(s, i) > 0 && ko != INF && ko + 1 == kx) pred = ((2 * s + 2) << 16) | i;
            }
          } else {  // out_{s,i}: in_{s,i}, then lowest tight reverse in_{s+1,v}, then t*
            const int s = (l >> 1) - 1, i = p;
            const uint64_t ki = ldk_in(s, i);
            if (*rg(s, i) < *rcap(s, i) && ki != INF && ki + 1 == kx) {
              pred = ((2 * s + 1) << 16) | i;
            } else if (s < S - 1) {
              const uint32_t* al = arcs + (size_t)s * Lcap;
              const int c = __ldcg(&cnt[s]);
              for (int e = tid; e < c; e += CT) {
                const uint32_t ent = __ldcg(&al[e]);
                if ((int)(ent >> 20) != i) continue;
                const int v = (int)((ent >> 8) & 0xFFFu);
                const uint64_t k = ldk_in(s + 1, v);
                const int32_t w = __ldcg(&arcw[(size_t)s * Lcap + e]);
                if (k != INF && k + 1ull == kx + ((uint64_t)(uint32_t)w << kHopBits)) atomicMin(&misc->red32, v);
              }
              __syncthreads();
              if (misc->red32 != INT_MAX) pred = ((2 * s + 3) << 16) | misc->red32;
            } else if (*rsnkf(i) > 0 && tkey + 1ull == kx + ((uint64_t)(uint32_t)snk[i] << kHopBits)) {
              pred = Lt << 16;
            }
          }
          __syncthreads();
          if (pred < 0 || len >= 2 * S * n + 2) {
            if (tid == 0 && atomicCAS(&P.stats[9], 0ull, (unsigned long long)inst + 1) == 0ull) {
              P.stats[5] = (unsigned long long)x; P.stats[6] = kx; P.stats[7] = (unsigned long long)len;
              P.stats[8] = tkey;
              for (int s2 = 0; s2 < S && 2 * S * n + 16 < 2000; ++s2)
                for (int i = 0; i < n; ++i) {
                  P.stats[16 + (s2 * n + i) * 3 + 0] = ldk_in(s2, i);
                  P.stats[16 + (s2 * n + i) * 3 + 1] = ldk_out(s2, i);
                  P.stats[16 + (s2 * n + i) * 3 + 2] = (unsigned long long)*rg(s2, i);
                }
            }
            err = 1;
            break;
          }
          if (tid == 0) path[len] = (uint32_t)pred;
          ++len;
          x = pred;
        }
        __syncthreads();
        if (tid == 0) misc->pathlen = err ? -1 : len;
        for (int e = tid; e < len - 1; e += CT) found[e] = INT_MAX;
      }
      cl.sync();

      TMARK(6);
      // ---- locate the path's inter-stage arcs in the positive-arc lists (whole cluster) ----
      // arc e of the path is path[len-1-e] -> path[len-2-e]; the lists are scanned in parallel by
      // all C * CT threads of the cluster, chunk by chunk of CT path arcs staged in shared memory
      const int plen = M0->pathlen;
      for (int e0 = 0; e0 < plen - 1; e0 += CT) {
        const int ne = min(CT, plen - 1 - e0);
        if (tid < ne) {
          const int e = e0 + tid;
          const int u = (int)__ldcg(&path[plen - 1 - e]), v = (int)__ldcg(&path[plen - 2 - e]);
          const int lu = u >> 16, lv = v >> 16, pu = u & 0xFFFF, pv = v & 0xFFFF;
          uint32_t key = 0xFFFFFFFFu;
          int sb = 0, c = 0;
          if (u != 0 && lv != Lt && ((!(lu & 1) && lv == lu + 1) || ((lu & 1) && lv == lu - 1))) {
            const bool fwdarc = !(lu & 1);
            sb = fwdarc ? (lu >> 1) - 1 : (lv >> 1) - 1;
            key = fwdarc ? (((uint32_t)pu << 12) | (uint32_t)pv) : (((uint32_t)pv << 12) | (uint32_t)pu);
            c = __ldcg(&cnt[sb]);
          }
          aq[3 * tid] = key; aq[3 * tid + 1] = (uint32_t)sb; aq[3 * tid + 2] = (uint32_t)c;
        }
        __syncthreads();
#pragma unroll 4
        for (int t = 0; t < ne; ++t) {
          const uint32_t key = aq[3 * t];
          const int c = (int)aq[3 * t + 2];
          const uint32_t* al = arcs + (size_t)aq[3 * t + 1] * Lcap;
          for (int q = r * CT + tid; q < c; q += C * CT)
            if ((__ldcg(&al[q]) >> 8) == key) atomicMin(&found[e0 + t], q);
        }
        __syncthreads();
      }
      cl.sync();

      TMARK(7);
      // ---- bottleneck and augmentation (leader CTA; a simple path touches every g, f_src,
      // f_snk and list entry at most once, so all in-place updates run in parallel) ----
      if (r == 0) {
        const int len = plen, err = plen < 0;
        if (tid == 0) misc->red64 = err ? 0ull : (uint64_t)(M - F);
        __syncthreads();
        if (!err) {
          for (int e = tid; e < len - 1; e += CT) {
            const int u = (int)path[len - 1 - e], v = (int)path[len - 2 - e];
            const int lu = u >> 16, lv = v >> 16, pu = u & 0xFFFF;
            uint64_t rc = INF;
            if (u == 0 || lv == Lt) {
            } else if ((lu & 1) && lv == lu + 1) {
              const int s = (lu - 1) >> 1;
              rc = (uint64_t)(*rcap(s, pu) - *rg(s, pu));
            } else if (!(lu & 1) && lv == lu - 1) {
              rc = (uint64_t)*rg((lu >> 1) - 1, pu);
            } else if ((lu & 1) && lv == lu - 1) {  // reverse inter-stage arc: its flow
              const int q = __ldcg(&found[e]);
              rc = q == INT_MAX ? 0ull : (uint64_t)(__ldcg(&arcs[(size_t)((lv >> 1) - 1) * Lcap + q]) & 0xFFu);
            }
            if (rc != INF) atomicMin((unsigned long long*)&misc->red64, (unsigned long long)rc);
          }
        }
        __syncthreads();
        const long long d = (long long)misc->red64;
        __syncthreads();
        if (err || d <= 0) {
          if (tid == 0) misc->status = err ? 1 : 4;
        } else {
          // (1) node arcs, source/sink arcs and list entries whose flow stays positive; entries
          // whose flow drops to zero are collected and (2) leave their list one by one (swap with
          // the last entry).  A removal moves another entry, so every index is re-checked.
          auto locate = [&](const uint32_t* al, int sb, int q, uint32_t key) -> int {
            const int c = __ldcg(&cnt[sb]);
            if (q < c && (__ldcg(&al[q]) >> 8) == key) return q;
            for (int k = 0; k < c; ++k)
              if ((__ldcg(&al[k]) >> 8) == key) return k;
            return -1;
          };
          for (int e0 = 0; e0 < len - 1; e0 += CT) {
            if (tid == 0) misc->nrem = 0;
            __syncthreads();
            const int e = e0 + tid;
            if (e < len - 1) {
              const int u = (int)path[len - 1 - e], v = (int)path[len - 2 - e];
              const int lu = u >> 16, lv = v >> 16, pu = u & 0xFFFF, pv = v & 0xFFFF;
              if (u == 0) {
                *rsrcf(pv) += (int32_t)d;
              } else if (lv == Lt) {
                *rsnkf(pu) += (int32_t)d;
              } else if ((lu & 1) && lv == lu + 1) {
                *rg((lu - 1) >> 1, pu) += (int8_t)d;
              } else if (!(lu & 1) && lv == lu - 1) {
                *rg((lu >> 1) - 1, pu) -= (int8_t)d;
              } else {
                const bool fwdarc = !(lu & 1);
                const int sb = fwdarc ? (lu >> 1) - 1 : (lv >> 1) - 1;
                const uint32_t key = fwdarc ? (((uint32_t)pu << 12) | (uint32_t)pv) : (((uint32_t)pv << 12) | (uint32_t)pu);
                uint32_t* al = arcs + (size_t)sb * Lcap;
                int q = __ldcg(&found[e]);
                if (q != INT_MAX) q = locate(al, sb, q, key);
                if (q >= 0 && q != INT_MAX) {
                  const uint32_t ent = __ldcg(&al[q]);
                  const int f = (int)(ent & 0xFFu) + (fwdarc ? (int)d : -(int)d);
                  if (f > 0) {
                    __stcg(&al[q], (ent & ~0xFFu) | (uint32_t)f);
                  } else {
                    const int k = atomicAdd(&misc->nrem, 1);
                    aq[3 * k] = key; aq[3 * k + 1] = (uint32_t)sb; aq[3 * k + 2] = (uint32_t)q;
                  }
                } else if (!fwdarc || q < 0) {
                  misc->status = 2;
                }
              }
            }
            __syncthreads();
            if (tid == 0)
              for (int k = 0; k < misc->nrem; ++k) {
                const int sb = (int)aq[3 * k + 1];
                uint32_t* al = arcs + (size_t)sb * Lcap;
                const int q = locate(al, sb, (int)aq[3 * k + 2], aq[3 * k]);
                if (q < 0) { misc->status = 2; continue; }
                const int c = __ldcg(&cnt[sb]);
                __stcg(&al[q], __ldcg(&al[c - 1]));
                __stcg(&arcw[(size_t)sb * Lcap + q], __ldcg(&arcw[(size_t)sb * Lcap + c - 1]));
                __stcg(&cnt[sb], c - 1);
              }
            __syncthreads();
          }
          // (3) new positive arcs are appended (parallel, one atomic slot each)
          for (int e = tid; e < len - 1; e += CT) {
            const int u = (int)path[len - 1 - e], v = (int)path[len - 2 - e];
            const int lu = u >> 16, lv = v >> 16, pu = u & 0xFFFF, pv = v & 0xFFFF;
            if (u == 0 || lv == Lt || !(!(lu & 1) && lv == lu + 1) || __ldcg(&found[e]) != INT_MAX) continue;
            const int sb = (lu >> 1) - 1;
            const int q = atomicAdd(&cnt[sb], 1);
            if (q < Lcap) {
              __stcg(&arcs[(size_t)sb * Lcap + q], ((uint32_t)pu << 20) | ((uint32_t)pv << 8) | (uint32_t)d);
              __stcg(&arcw[(size_t)sb * Lcap + q], tile[((size_t)sb * n + pv) * ld + pu]);
            } else {
              misc->status = 2;
            }
          }
          __syncthreads();
          if (tid == 0) {
            misc->F = F + d;
            misc->cost += (int64_t)d * (int64_t)(tkey >> kHopBits);
            misc->A += 1;
            atomicAdd(&P.stats[2], 1ull);
            atomicAdd(&P.stats[4], (unsigned long long)len);
          }
        }
      }
      TMARK(8);
      cl.sync();
    }

    drain();  // nothing may stay in flight past the instance (or the kernel)
    // ---- results and the canonical assignment ----
    if (r == 0 && tid == 0) {
      o.F[inst] = misc->F;
      o.cost[inst] = misc->cost;
      if (o.A) o.A[inst] = misc->A;
      if (o.status) o.status[inst] = misc->status;
    }
    for (int k = tid; k < S * R; k += CT) {
      const int s = k / R, v = v0 + k % R;
      if (v < n) P.g[((size_t)inst * S + s) * n + v] = g[k];
    }
    for (int lv = tid; lv < nr; lv += CT) {
      P.src_f[(size_t)inst * n + v0 + lv] = srcf[lv];
      P.snk_f[(size_t)inst * n + v0 + lv] = snkf[lv];
    }
    cl.sync();
  }
}

#undef TMARK

template <int C>
cudaError_t launch_c(const Problem& P, const SspOut& o, cudaStream_t st, int* nclusters_out, bool query) {
  const size_t smem = cl_layout(P, C).total;
  if (smem > kSmemMax) return cudaErrorInvalidConfiguration;
  auto k = ssp_cluster_kernel<C>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
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
  cfg.blockDim = dim3(CT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C);
  int ncl = 0;
  e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
  if (e != cudaSuccess) return e;
  if (getenv("GWTF_DEBUG")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)k);
    fprintf(stderr, "[gwtf] C=%d regs %d static smem %zu max dyn %d ptx %d -> clusters %d\n", C, fa.numRegs,
            fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.ptxVersion, ncl);
  }
  if (ncl < 1) return cudaErrorInvalidConfiguration;
  if (ncl > P.B) ncl = P.B;
  if (nclusters_out) *nclusters_out = ncl;
  if (query) return cudaSuccess;
  if (ncl > P.ws_cluster_slots) ncl = P.ws_cluster_slots;  // path scratch slots
  cfg.gridDim = dim3(ncl * C);
  return cudaLaunchKernelEx(&cfg, k, P, o);
}

}  // namespace

size_t ssp_cluster_smem_bytes(const Problem& P, int C) { return cl_layout(P, C).total; }

// Cluster size: the smallest estimated makespan, waves x per-CTA rows, where waves =
// ceil(B / clusters the device hosts at once) and a CTA's step time grows with its R = n / C
// destination rows plus a fixed barrier/gather overhead (~16 rows).  E.g. 8 stress instances:
// clusters of 16 CTAs fit 7 at a time (2 waves), clusters of 10 fit all 8 (1 wave).
int ssp_cluster_size(const Problem& P) {
  int best = 0;
  long long best_cost = 0;
  for (int C : {16, 12, 10, 8, 4, 2}) {
    if (P.n < C || cl_layout(P, C).total > kSmemMax) continue;
    int ncl = 0;
    cudaError_t e;
    switch (C) {
      case 16: e = launch_c<16>(P, SspOut{}, nullptr, &ncl, true); break;
      case 12: e = launch_c<12>(P, SspOut{}, nullptr, &ncl, true); break;
      case 10: e = launch_c<10>(P, SspOut{}, nullptr, &ncl, true); break;
      case 8: e = launch_c<8>(P, SspOut{}, nullptr, &ncl, true); break;
      case 4: e = launch_c<4>(P, SspOut{}, nullptr, &ncl, true); break;
      default: e = launch_c<2>(P, SspOut{}, nullptr, &ncl, true); break;
    }
    if (getenv("GWTF_DEBUG"))
      fprintf(stderr, "[gwtf] cluster size %d: smem %zu B, ring %d chunks, query %s, max active clusters %d\n", C,
              cl_layout(P, C).total, cl_layout(P, C).nbc, cudaGetErrorString(e), ncl);
    if (e != cudaSuccess || ncl < 1) { cudaGetLastError(); continue; }
    const long long waves = (P.B + ncl - 1) / ncl;
    const long long cost = waves * (cl_rows(P.n, C) + 16);
    if (best == 0 || cost < best_cost) { best_cost = cost; best = C; }
  }
  if (const char* f = getenv("GWTF_CLUSTER_SIZE")) best = atoi(f);  // testing override
  return best;
}

cudaError_t launch_ssp_cluster(const Problem& P, const SspOut& o, cudaStream_t st, int C) {
  cudaError_t e = cudaMemsetAsync(P.counters + 4, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  switch (C) {
    case 16: return launch_c<16>(P, o, st, nullptr, false);
    case 12: return launch_c<12>(P, o, st, nullptr, false);
    case 10: return launch_c<10>(P, o, st, nullptr, false);
    case 8: return launch_c<8>(P, o, st, nullptr, false);
    case 4: return launch_c<4>(P, o, st, nullptr, false);
    case 2: return launch_c<2>(P, o, st, nullptr, false);
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace gwtf
