// Exact solve: canonical successive shortest paths for a batch of instances.
//
// One team of TPI threads per instance, persistent over an atomic instance queue.  The
// instance's cost tiles are staged once into shared memory by the TMA bulk-copy engine
// (cp.async.bulk + mbarrier) and every Bellman-Ford sweep of every augmentation then reads
// them from shared memory.  The dominant step is the dense min-plus relaxation of one stage
// boundary,
//     key_in[s+1][v] = min(key_in[s+1][v], min_u key_out[s][u] + (C[s][v][u], 1))
// done by groups of G lanes per destination row v (the dest-major tile row is read as 128-bit
// vectors, 4 sources per lane per load) followed by a shuffle-min across the group.  Keys are
// lexicographic (cost, hops) packed into one integer:
//   * 32-bit keys (k32): cost << H | hops with the tile pre-shifted to (C << H) + 1 in shared
//     memory, so one relaxation is one DPX VIADDMNMX (min(a + b, c)); used when the bound of
//     DESIGN.md 2.2 allows, with a per-instance overflow guard that re-runs the instance with
//   * 64-bit keys: cost << 20 | hops (the global-memory tier and the fallback).
// Bellman-Ford passes track dirty stages: a boundary is re-relaxed only if its sources changed
// since its last relaxation, the backward (reverse-arc) phases likewise.  Reverse residual arcs
// are relaxed from the per-boundary list of positive-flow arcs.  The augmenting path is traced
// by warp 0 with ballots (lowest (layer, position) tight predecessor) and augmented in place.
#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace gwtf {

namespace {

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// ---- key arithmetic --------------------------------------------------------------------
// "w" is a tile/src/snk entry as stored in the team workspace: the raw cost for 64-bit keys,
// the pre-shifted weight (C << H) + 1 for 32-bit keys (kInf32 = absent).
constexpr uint32_t kInf32 = 0x3FFFFFFFu;
constexpr uint32_t kGuard32 = 1u << 29;

template <bool k32>
struct KT;

template <>
struct KT<false> {
  using K = uint64_t;
  static constexpr K INF = ~0ull;
  __device__ static K relax(K acc, K k, int32_t w, int) {
    return (w == kAbsent || k == INF) ? acc : umin64(acc, k + ((uint64_t)(uint32_t)w << kHopBits) + 1ull);
  }
  __device__ static bool absent(int32_t w) { return w == kAbsent; }
  __device__ static K plus(K k, int32_t w) { return k + ((uint64_t)(uint32_t)w << kHopBits) + 1ull; }
  __device__ static K src_key(int32_t w) { return ((uint64_t)(uint32_t)w << kHopBits) | 1ull; }
  // reverse arc of a flow-carrying forward arc of weight w: kin - (c, 0) + (0, 1)
  __device__ static K rev(K kin, int32_t w) { return kin - ((uint64_t)(uint32_t)w << kHopBits) + 1ull; }
  __device__ static bool rev_tight(K kin, int32_t w, K kx) { return kin + 1ull == kx + ((uint64_t)(uint32_t)w << kHopBits); }
  __device__ static int64_t cost(K k, int) { return (int64_t)(k >> kHopBits); }
  __device__ static int32_t prep(int32_t c, int) { return c; }
};

template <>
struct KT<true> {
  using K = uint32_t;
  static constexpr K INF = kInf32;
  // min(k + w, acc) as IMAD (w * one + k, `one` = 1 read through a volatile load) + VIMNMX: ptxas
  // would fuse a plain add with the min into the DPX VIADDMNMX, which issues at a quarter of the
  // integer rate on sm_100a (measured: 32.7 vs 62 add-min pairs/cycle/SM for IADD3 + VIMNMX)
  __device__ static K relax(K acc, K k, int32_t w, int one) { return (K)min(w * one + (int)k, (int)acc); }
  __device__ static bool absent(int32_t w) { return (uint32_t)w == kInf32; }
  __device__ static K plus(K k, int32_t w) { return k + (uint32_t)w; }
  __device__ static K src_key(int32_t w) { return (uint32_t)w; }
  __device__ static K rev(K kin, int32_t w) { return kin + 2u - (uint32_t)w; }
  __device__ static bool rev_tight(K kin, int32_t w, K kx) { return kin + 2u == kx + (uint32_t)w; }
  __device__ static int64_t cost(K k, int H) { return (int64_t)(k >> H); }
  __device__ static int32_t prep(int32_t c, int H) { return c == kAbsent ? (int32_t)kInf32 : (int32_t)(((uint32_t)c << H) + 1u); }
};

template <bool k32>
__device__ __forceinline__ void load_keys4(const typename KT<k32>::K* p, typename KT<k32>::K* k) {
  if constexpr (k32) {
    const uint4 v = *(const uint4*)p;
    k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
  } else {
    const ulonglong2 a = *(const ulonglong2*)p, b = *(const ulonglong2*)(p + 2);
    k[0] = a.x; k[1] = a.y; k[2] = b.x; k[3] = b.y;
  }
}

template <class K>
__device__ __forceinline__ K shfl_min(K v, int off, int width) {
  if constexpr (sizeof(K) == 4) {
    const uint32_t o = __shfl_xor_sync(0xffffffffu, (uint32_t)v, off, width);
    return o < v ? o : v;
  } else {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, off, width);
    return o < v ? o : v;
  }
}

// ---- workspace layout ------------------------------------------------------------------
struct SspLayout {
  size_t misc, tile, kin, kout, g, capE, src, snk, srcf, snkf, arcs, cnt, path, total;
};
// misc block: 0 mbarrier | 8 F | 16 cost | 24 tnew | 32 A | 36 status | 40 inst
// tile_bytes: 4 (int32 tiles) or 2 (the 16-bit copy, Problem::tile16s)
__host__ __device__ inline SspLayout ssp_layout(const Problem& P, bool with_tile, int key_bytes, int tile_bytes = 4) {
  SspLayout L;
  size_t o = 0;
  const size_t Sn = (size_t)P.S * P.n, Sld = (size_t)P.S * P.ld;
  const size_t nb = (size_t)(P.S > 1 ? P.S - 1 : 0);
  L.misc = o; o += 64;
  L.tile = o; if (with_tile) o += al16(nb * P.n * P.ld * tile_bytes);
  L.kin = o; o += al16((Sld + 4) * key_bytes);
  L.kout = o; o += al16((Sld + 4) * key_bytes);
  L.g = o; o += al16(Sn * 4);
  L.capE = o; o += al16(Sn * 4);
  L.src = o; o += al16((size_t)P.n * 4);
  L.snk = o; o += al16((size_t)P.n * 4);
  L.srcf = o; o += al16((size_t)P.n * 4);
  L.snkf = o; o += al16((size_t)P.n * 4);
  L.arcs = o; o += al16(nb * P.Lcap * 4);
  L.cnt = o; o += al16((nb + 1) * 4);
  L.path = o; o += al16((2 * Sn + 4) * 4);
  L.total = o;
  return L;
}

// node ids of the trace: layer << 16 | position
__device__ __forceinline__ int nid(int layer, int pos) { return (layer << 16) | pos; }

// kTB = 2 / 1: the instance's tiles are staged from the 16-bit / 8-bit copy (Problem::tile16s: costs
// < 65535, absent 0xFFFF; Problem::tile8s: costs < 255, absent 0xFF) and widened on use -- a half / a
// quarter of the shared memory, so more instances per SM; kTB = 4: the int32 tiles
template <int TPI, bool kSmem, bool k32, bool kRedo, int kTB>
__global__ void __launch_bounds__(TPI >= 128 ? TPI : 128, TPI >= 128 ? 1536 / TPI : 6) ssp_kernel(const Problem P, const SspOut o, const size_t ws_bytes) {
  using K = typename KT<k32>::K;
  constexpr K INF = KT<k32>::INF;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int sh_one;
  if (threadIdx.x == 0) sh_one = 1;
  __syncthreads();
  const int one = *(volatile int*)&sh_one;
  const Team<TPI> T{(int)(threadIdx.x % TPI), (int)(threadIdx.x / TPI)};
  const int teams_per_cta = blockDim.x / TPI;
  uint8_t* base;
  if constexpr (kSmem) base = smem + (size_t)T.id * ws_bytes;
  else base = P.ws + (size_t)(blockIdx.x * teams_per_cta + T.id) * ws_bytes;
  constexpr bool k16 = kTB == 2, k8 = kTB == 1;
  const SspLayout L = ssp_layout(P, kSmem, sizeof(K), kTB);
  uint64_t* mbar = (uint64_t*)(base + L.misc);
  int64_t* F_p = (int64_t*)(base + L.misc + 8);
  int64_t* cost_p = (int64_t*)(base + L.misc + 16);
  K* tnew = (K*)(base + L.misc + 24);
  int32_t* A_p = (int32_t*)(base + L.misc + 32);
  int32_t* status_p = (int32_t*)(base + L.misc + 36);
  int32_t* inst_p = (int32_t*)(base + L.misc + 40);
  K* kin = (K*)(base + L.kin);
  K* kout = (K*)(base + L.kout);
  int32_t* g = (int32_t*)(base + L.g);
  int32_t* capE = (int32_t*)(base + L.capE);
  int32_t* src = (int32_t*)(base + L.src);
  int32_t* snk = (int32_t*)(base + L.snk);
  int32_t* srcf = (int32_t*)(base + L.srcf);
  int32_t* snkf = (int32_t*)(base + L.snkf);
  uint32_t* arcs = (uint32_t*)(base + L.arcs);
  int32_t* cnt = (int32_t*)(base + L.cnt);
  uint32_t* path = (uint32_t*)(base + L.path);

  const int S = P.S, n = P.n, ld = P.ld, Sn = S * n, Lcap = P.Lcap, H = P.hbits;
  const int chunks = ld / 4;
  int G = 1;
  while (G * 2 <= chunks && G * 2 <= 32) G *= 2;  // lanes per destination row
  const int NG = TPI / G, gi = T.tid / G, li = T.tid % G;
  const int lane = threadIdx.x & 31;
  const int Lt = 2 * S + 1;  // layer of t*
  const size_t tile_elems = (size_t)(S - 1) * n * ld;
  const uint32_t tile_bytes = k16 ? (uint32_t)(P.tile16s_stride * 2) : k8 ? (uint32_t)P.tile8s_stride : (uint32_t)(tile_elems * 4);
  uint32_t phase = 0;
  unsigned long long n_relax = 0, n_back = 0, n_pass = 0;

  if (kSmem && T.tid == 0) {
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  T.sync();

  for (;;) {
    if (T.tid == 0) {
      int q;
      if constexpr (kRedo) {
        q = atomicAdd(&P.counters[3], 1);
        q = q < P.counters[2] ? P.redo[q] : P.B;
      } else {
        q = atomicAdd(&P.counters[0], 1);
        if (P.sel) q = q < *P.sel_count ? P.sel[q] : P.B;
      }
      *inst_p = q;
    }
    T.sync();
    const int inst = *inst_p;
    if (inst >= P.B) break;

    // ---- stage the instance: tiles by TMA bulk copy, the rest by plain loads ----
    const int32_t* gtile = P.tile + (size_t)inst * tile_elems;
    const int32_t* tile = gtile;
    const uint16_t* tile16 = (const uint16_t*)(base + L.tile);  // k16: the staged 16-bit copy
    const uint8_t* tile8 = (const uint8_t*)(base + L.tile);     // k8: the staged 8-bit copy
    if constexpr (kSmem) {
      tile = (const int32_t*)(base + L.tile);
      const uint8_t* gsrc = k16 ? (const uint8_t*)(P.tile16s + (size_t)inst * P.tile16s_stride)
                          : k8 ? P.tile8s + (size_t)inst * P.tile8s_stride : (const uint8_t*)gtile;
      if (T.tid == 0 && tile_bytes) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(mbar, tile_bytes);
        for (uint32_t off = 0; off < tile_bytes; off += 32768u)
          bulk_g2s((uint8_t*)(base + L.tile) + off, gsrc + off, tile_bytes - off < 32768u ? tile_bytes - off : 32768u, mbar);
      }
    }
    // weight of a 16-bit tile entry in the key arithmetic's form: pre-shifted (C << H) + 1 for
    // 32-bit keys, the raw cost for 64-bit keys, absent (0xFFFF) -> the absent code of each
    constexpr uint32_t kAbs = k8 ? 0xFFu : 0xFFFFu;  // the narrow copies' absent code
    auto w16 = [&](uint32_t c) -> int32_t {
      if constexpr (k32) return c == kAbs ? (int32_t)kInf32 : (int32_t)((c << H) + 1u);
      else return c == kAbs ? kAbsent : (int32_t)c;
    };
    auto wgt = [&](size_t idx) -> int32_t {
      if constexpr (k16) return w16(tile16[idx]);
      else if constexpr (k8) return w16(tile8[idx]);
      else return tile[idx];
    };
    const int64_t M = P.supply[inst];
    for (int k = T.tid; k < Sn; k += TPI) {
      g[k] = 0;
      capE[k] = P.alive[(size_t)inst * Sn + k] ? P.cap[(size_t)inst * Sn + k] : 0;
    }
    for (int i = T.tid; i < n; i += TPI) {
      src[i] = KT<k32>::prep(P.src[(size_t)inst * n + i], H);
      snk[i] = KT<k32>::prep(P.snk[(size_t)inst * n + i], H);
      srcf[i] = 0;
      snkf[i] = 0;
    }
    for (int k = T.tid; k < S; k += TPI) cnt[k] = 0;
    if (T.tid == 0) { *F_p = 0; *cost_p = 0; *A_p = 0; *status_p = 0; }
    if (kSmem && tile_bytes) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
      if constexpr (k32 && kTB == 4) {  // pre-shift the weights in place: (C << H) + 1, absent -> INF
        T.sync();
        int32_t* tw = (int32_t*)(base + L.tile);
        for (size_t k = T.tid; k < tile_elems; k += TPI) tw[k] = KT<true>::prep(tw[k], H);
      }
    }
    T.sync();

    // ---- successive shortest paths ----
    for (;;) {
      const int64_t F = *F_p;
      if (F >= M || *status_p) break;
      for (int k = T.tid; k < S * ld + 4; k += TPI) { kin[k] = INF; kout[k] = INF; }
      K tkey = INF;
      T.sync();
      // s* -> in_0 (src arcs), then in_0 -> out_0 where g < cap
      for (int vb = 0; vb < n; vb += NG) {
        const int v = vb + gi;
        if (li == 0 && v < n && !KT<k32>::absent(src[v])) {
          const K c = KT<k32>::src_key(src[v]);
          kin[v] = c;
          if (g[v] < capE[v]) kout[v] = c + 1;
        }
      }
      T.sync();
      uint64_t fwd = S > 1 ? 1ull : 0ull;  // relax(s) pending
      uint64_t bwd = 1ull;                 // backward phase s pending
      bool tdirty = S == 1, trev = false;
      for (;;) {  // Bellman-Ford sweeps to the fixed point, dirty stages only
        // forward: dense min-plus relaxation of the dirty stage boundaries
        for (int s = 0; s + 1 < S; ++s) {
          if (!((fwd >> s) & 1ull)) continue;
          fwd &= ~(1ull << s);
          ++n_relax;
          const int32_t* Ts = tile + (size_t)s * n * ld;
          const K* ko = kout + (size_t)s * ld;
          int ch = 0;
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            K acc = INF;
            if (v < n) {
              if constexpr (k8) {  // 4 weights per 4-byte load, widened
                const uint32_t* row = (const uint32_t*)(tile8 + ((size_t)s * n + v) * ld);
                for (int c = li; c < chunks; c += G) {
                  const uint32_t w = row[c];
                  K kk[4];
                  load_keys4<k32>(ko + 4 * c, kk);
                  acc = KT<k32>::relax(acc, kk[0], w16(w & 0xFFu), one);
                  acc = KT<k32>::relax(acc, kk[1], w16((w >> 8) & 0xFFu), one);
                  acc = KT<k32>::relax(acc, kk[2], w16((w >> 16) & 0xFFu), one);
                  acc = KT<k32>::relax(acc, kk[3], w16(w >> 24), one);
                }
              } else if constexpr (k16) {  // 4 weights per 8-byte load, widened
                const uint2* row = (const uint2*)(tile16 + ((size_t)s * n + v) * ld);
                for (int c = li; c < chunks; c += G) {
                  const uint2 w = row[c];
                  K kk[4];
                  load_keys4<k32>(ko + 4 * c, kk);
                  acc = KT<k32>::relax(acc, kk[0], w16(w.x & 0xFFFFu), one);
                  acc = KT<k32>::relax(acc, kk[1], w16(w.x >> 16), one);
                  acc = KT<k32>::relax(acc, kk[2], w16(w.y & 0xFFFFu), one);
                  acc = KT<k32>::relax(acc, kk[3], w16(w.y >> 16), one);
                }
              } else {
                const int4* row = (const int4*)(Ts + (size_t)v * ld);
                for (int c = li; c < chunks; c += G) {
                  const int4 w = row[c];
                  K kk[4];
                  load_keys4<k32>(ko + 4 * c, kk);
                  acc = KT<k32>::relax(acc, kk[0], w.x, one);
                  acc = KT<k32>::relax(acc, kk[1], w.y, one);
                  acc = KT<k32>::relax(acc, kk[2], w.z, one);
                  acc = KT<k32>::relax(acc, kk[3], w.w, one);
                }
              }
            }
            for (int off = G >> 1; off > 0; off >>= 1) acc = shfl_min<K>(acc, off, G);
            if (v < n && li == 0) {
              const int idx = (s + 1) * ld + v, gidx = (s + 1) * n + v;
              K kv = kin[idx];
              if (acc < kv) { kin[idx] = acc; kv = acc; ch = 1; }
              if (kv != INF && g[gidx] < capE[gidx] && kv + 1 < kout[idx]) { kout[idx] = kv + 1; ch = 1; }
            }
          }
          if (T.sync_or(ch)) {
            if (s + 1 < S - 1) fwd |= 1ull << (s + 1);
            else tdirty = true;
            bwd |= 1ull << (s + 1);
          }
        }
        // out_{S-1} -> t*
        if (tdirty) {
          tdirty = false;
          if (T.tid == 0) *tnew = INF;
          T.sync();
          K tc = INF;
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            if (li == 0 && v < n && !KT<k32>::absent(snk[v])) {
              const K k = kout[(S - 1) * ld + v];
              if (k != INF) tc = tc < KT<k32>::plus(k, snk[v]) ? tc : KT<k32>::plus(k, snk[v]);
            }
          }
          for (int off = 16; off > 0; off >>= 1) tc = shfl_min<K>(tc, off, 32);
          if (lane == 0 && tc != INF) {
            if constexpr (k32) atomicMin((unsigned int*)tnew, (unsigned int)tc);
            else atomicMin((unsigned long long*)tnew, (unsigned long long)tc);
          }
          T.sync();
          const K tn = *tnew;
          if (tn < tkey) { tkey = tn; trev = true; }
        }
        // t* -> out_{S-1} (reverse sink arcs, snk_f > 0)
        if (trev) {
          trev = false;
          int ch = 0;
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            if (li == 0 && v < n && snkf[v] > 0) {
              const int idx = (S - 1) * ld + v;
              const K c = KT<k32>::rev(tkey, snk[v]);
              if (c < kout[idx]) { kout[idx] = c; ch = 1; }
            }
          }
          if (T.sync_or(ch)) bwd |= 1ull << (S - 1);
        }
        // backward: reverse node arcs out_s -> in_s (g > 0) and reverse inter-stage arcs
        // in_s -> out_{s-1} over the positive-flow list of boundary s-1
        for (int s = S - 1; s >= 0; --s) {
          if (!((bwd >> s) & 1ull)) continue;
          bwd &= ~(1ull << s);
          ++n_back;
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            if (li == 0 && v < n) {
              const int idx = s * ld + v;
              const K ko = kout[idx];
              if (g[s * n + v] > 0 && ko != INF && ko + 1 < kin[idx]) kin[idx] = ko + 1;
            }
          }
          if (s == 0) { T.sync(); break; }
          const uint32_t* al = arcs + (size_t)(s - 1) * Lcap;
          const int c = cnt[s - 1];
          int ch = 0;
          for (int e = T.tid; e < c; e += TPI) {
            const uint32_t ent = al[e];
            const int u = (int)(ent >> 20), v = (int)((ent >> 8) & 0xFFFu);
            const int idx = s * ld + v;
            K ki = kin[idx];
            const K kov = kout[idx];
            if (g[s * n + v] > 0 && kov != INF && kov + 1 < ki) ki = kov + 1;
            if (ki == INF) continue;
            const K cand = KT<k32>::rev(ki, wgt(((size_t)(s - 1) * n + v) * ld + u));
            K old;
            if constexpr (k32) old = atomicMin((unsigned int*)&kout[(s - 1) * ld + u], (unsigned int)cand);
            else old = atomicMin((unsigned long long*)&kout[(s - 1) * ld + u], (unsigned long long)cand);
            if (cand < old) ch = 1;
          }
          if (T.sync_or(ch)) {
            fwd |= 1ull << (s - 1);
            bwd |= 1ull << (s - 1);
          }
        }
        ++n_pass;
        if (!(fwd | bwd) && !tdirty && !trev) break;
      }
      if (tkey == INF) break;  // t* unreachable: F is the maximum flow
      if constexpr (k32) {  // overflow guard: every finite key must stay < 2^29
        int big = 0;
        for (int k = T.tid; k < S * ld; k += TPI) {
          big |= (kin[k] != INF && kin[k] >= kGuard32);
          big |= (kout[k] != INF && kout[k] >= kGuard32);
        }
        if (T.sync_or(big || tkey >= kGuard32)) {
          if (T.tid == 0) *status_p = 3;
          T.sync();
          break;
        }
      }

      // ---- trace the canonical augmenting path and augment (warp 0) ----
      if (T.tid < 32) {
        auto key_of = [&](int id) -> K {
          const int l = id >> 16, p = id & 0xFFFF;
          if (l == 0) return (K)0;
          if (l == Lt) return tkey;
          if (l & 1) return kin[((l - 1) >> 1) * ld + p];
          return kout[((l >> 1) - 1) * ld + p];
        };
        const int maxlen = 2 * Sn + 2;
        int x = nid(Lt, 0), len = 1, err = 0;
        if (lane == 0) path[0] = (uint32_t)x;
        while (x != 0) {
          const int l = x >> 16, p = x & 0xFFFF;
          const K kx = key_of(x);
          int pred = -1;
          if (l == Lt) {
            for (int b = 0; b < n && pred < 0; b += 32) {
              const int i = b + lane;
              bool ok = false;
              if (i < n && !KT<k32>::absent(snk[i])) {
                const K k = kout[(S - 1) * ld + i];
                ok = k != INF && KT<k32>::plus(k, snk[i]) == kx;
              }
              const uint32_t m = __ballot_sync(0xffffffffu, ok);
              if (m) pred = nid(2 * S, b + __ffs(m) - 1);
            }
          } else if (l & 1) {  // in_{s,i}: s* or out_{s-1,u} (layer 2s) first, then out_{s,i} (layer 2s+2)
            const int s = (l - 1) >> 1, i = p;
            if (s == 0) {
              if (!KT<k32>::absent(src[i]) && KT<k32>::src_key(src[i]) == kx) pred = 0;
            } else {
              const size_t row = ((size_t)(s - 1) * n + i) * ld;
              for (int b = 0; b < n && pred < 0; b += 32) {
                const int u = b + lane;
                bool ok = false;
                const int32_t w = u < n ? wgt(row + u) : 0;
                if (u < n && !KT<k32>::absent(w)) {
                  const K k = kout[(s - 1) * ld + u];
                  ok = k != INF && KT<k32>::plus(k, w) == kx;
                }
                const uint32_t m = __ballot_sync(0xffffffffu, ok);
                if (m) pred = nid(2 * s, b + __ffs(m) - 1);
              }
            }
            if (pred < 0) {
              const K ko = kout[s * ld + i];
              if (g[s * n + i] > 0 && ko != INF && ko + 1 == kx) pred = nid(2 * s + 2, i);
            }
          } else {  // out_{s,i}: in_{s,i} (2s+1), then in_{s+1,v} reverse (2s+3), then t* reverse
            const int s = (l >> 1) - 1, i = p;
            const K ki = kin[s * ld + i];
            if (g[s * n + i] < capE[s * n + i] && ki != INF && ki + 1 == kx) {
              pred = nid(2 * s + 1, i);
            } else if (s < S - 1) {
              const uint32_t* al = arcs + (size_t)s * Lcap;
              const int c = cnt[s];
              uint32_t best = 0xFFFFFFFFu;
              for (int e = lane; e < c; e += 32) {
                const uint32_t ent = al[e];
                if ((int)(ent >> 20) != i) continue;
                const int v = (int)((ent >> 8) & 0xFFFu);
                const K k = kin[(s + 1) * ld + v];
                if (k != INF && KT<k32>::rev_tight(k, wgt(((size_t)s * n + v) * ld + i), kx)) best = min(best, (uint32_t)v);
              }
              best = __reduce_min_sync(0xffffffffu, best);
              if (best != 0xFFFFFFFFu) pred = nid(2 * s + 3, (int)best);
            } else if (snkf[i] > 0 && KT<k32>::rev_tight(tkey, snk[i], kx)) {
              pred = nid(Lt, 0);
            }
          }
          if (pred < 0 || len >= maxlen) { err = 1; break; }
          if (lane == 0) path[len] = (uint32_t)pred;
          ++len;
          x = pred;
        }
        __syncwarp();
        if (err) {
          if (lane == 0) *status_p = 1;
        } else {
          // bottleneck delta = min(M - F, residual capacities); arc e: path[len-1-e] -> path[len-2-e]
          const int narcs = len - 1;
          long long d = (long long)(M - F);
          for (int e = lane; e < narcs; e += 32) {
            const int u = (int)path[len - 1 - e], v = (int)path[len - 2 - e];
            const int lu = u >> 16, lv = v >> 16, pu = u & 0xFFFF, pv = v & 0xFFFF;
            long long r = LLONG_MAX;
            if (u == 0 || lv == Lt) {
            } else if ((lu & 1) && lv == lu + 1) {
              const int idx = ((lu - 1) >> 1) * n + pu;
              r = capE[idx] - g[idx];
            } else if (!(lu & 1) && lv == lu - 1) {
              r = g[((lu >> 1) - 1) * n + pu];
            } else if ((lu & 1) && lv == lu - 1) {
              const int s = (lv >> 1) - 1;
              const uint32_t key = ((uint32_t)pv << 12) | (uint32_t)pu;
              const uint32_t* al = arcs + (size_t)s * Lcap;
              r = 0;
              for (int q = 0; q < cnt[s]; ++q)
                if ((al[q] >> 8) == key) r = al[q] & 0xFFu;
            }
            d = r < d ? r : d;
          }
          for (int off = 16; off > 0; off >>= 1) {
            const long long t = __shfl_xor_sync(0xffffffffu, d, off);
            d = t < d ? t : d;
          }
          if (d <= 0) {
            if (lane == 0) *status_p = 1;
          } else {
            for (int e = 0; e < narcs; ++e) {
              const int u = (int)path[len - 1 - e], v = (int)path[len - 2 - e];
              const int lu = u >> 16, lv = v >> 16, pu = u & 0xFFFF, pv = v & 0xFFFF;
              if (u == 0) {
                if (lane == 0) srcf[pv] += (int32_t)d;
              } else if (lv == Lt) {
                if (lane == 0) snkf[pu] += (int32_t)d;
              } else if ((lu & 1) && lv == lu + 1) {
                if (lane == 0) g[((lu - 1) >> 1) * n + pu] += (int32_t)d;
              } else if (!(lu & 1) && lv == lu - 1) {
                if (lane == 0) g[((lu >> 1) - 1) * n + pu] -= (int32_t)d;
              } else {
                const bool fwdarc = !(lu & 1);
                const int s = fwdarc ? (lu >> 1) - 1 : (lv >> 1) - 1;
                const uint32_t uu = fwdarc ? pu : pv, vv = fwdarc ? pv : pu;
                const uint32_t key = (uu << 12) | vv;
                uint32_t* al = arcs + (size_t)s * Lcap;
                const int c = cnt[s];
                int found = -1;
                for (int b = 0; b < c && found < 0; b += 32) {
                  const int q = b + lane;
                  const uint32_t m = __ballot_sync(0xffffffffu, q < c && (al[q] >> 8) == key);
                  if (m) found = b + __ffs(m) - 1;
                }
                if (lane == 0) {
                  if (found >= 0) {
                    const int f = (int)(al[found] & 0xFFu) + (fwdarc ? (int)d : -(int)d);
                    if (f > 0) {
                      al[found] = (uu << 20) | (vv << 8) | (uint32_t)f;
                    } else {
                      al[found] = al[c - 1];
                      cnt[s] = c - 1;
                    }
                  } else if (fwdarc && c < Lcap) {
                    al[c] = (uu << 20) | (vv << 8) | (uint32_t)d;
                    cnt[s] = c + 1;
                  } else {
                    *status_p = 2;
                  }
                }
                __syncwarp();
              }
            }
            if (lane == 0) {
              *F_p = F + d;
              *cost_p += (int64_t)d * KT<k32>::cost(tkey, H);
              *A_p += 1;
            }
          }
        }
      }
      T.sync();
    }

    // ---- results and the canonical assignment ----
    T.sync();
    if (T.tid == 0) {
      atomicAdd(&P.stats[0], n_relax);
      atomicAdd(&P.stats[1], n_back);
      atomicAdd(&P.stats[2], (unsigned long long)*A_p);
      atomicAdd(&P.stats[3], n_pass);
    }
    n_relax = n_back = n_pass = 0;
    const int st = *status_p;
    if (k32 && st == 3) {  // key overflow: queue the instance for the 64-bit kernel
      if (T.tid == 0) {
        const int q = atomicAdd(&P.counters[2], 1);
        P.redo[q] = inst;
        atomicAdd(&P.stats[13], 1ull);  // instances re-solved with 64-bit keys (gwtf_flow_stats)
      }
      T.sync();
      continue;
    }
    if (T.tid == 0) {
      o.F[inst] = *F_p;
      o.cost[inst] = *cost_p;
      if (o.A) o.A[inst] = *A_p;
      if (o.status) o.status[inst] = st;
    }
    for (int k = T.tid; k < Sn; k += TPI) P.g[(size_t)inst * Sn + k] = g[k];
    for (int i = T.tid; i < n; i += TPI) {
      P.src_f[(size_t)inst * n + i] = srcf[i];
      P.snk_f[(size_t)inst * n + i] = snkf[i];
    }
    const int nb = S - 1;
    for (int k = T.tid; k < nb * Lcap; k += TPI) P.arcs[(size_t)inst * nb * Lcap + k] = arcs[k];
    for (int k = T.tid; k < nb; k += TPI) P.arc_cnt[(size_t)inst * nb + k] = cnt[k];
    T.sync();
  }
}

template <int TPI, bool kSmem, bool k32, bool kRedo, int kTB = 4>
cudaError_t launch_one(const Problem& P, const SspOut& o, cudaStream_t st, int num_sms) {
  const size_t ws = ssp_layout(P, kSmem, k32 ? 4 : 8, kTB).total;
  auto k = ssp_kernel<TPI, kSmem, k32, kRedo, kTB>;
  if (kSmem) {
    const size_t limit = 227 * 1024;
    int teams = TPI >= 128 ? 1 : 128 / TPI;
    while (teams > 1 && teams * ws > limit) --teams;
    const size_t smem = teams * ws;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, teams * TPI, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    long long grid = (long long)per_sm * num_sms;
    const long long need = kRedo ? (long long)num_sms : (P.B + teams - 1) / teams;
    if (grid > need) grid = need;
    k<<<(int)grid, teams * TPI, smem, st>>>(P, o, ws);
  } else {
    long long grid = P.ws_teams;
    if (!kRedo && grid > P.B) grid = P.B;
    if (grid < 1) grid = 1;
    k<<<(int)grid, TPI, 0, st>>>(P, o, ws);
  }
  return cudaGetLastError();
}

template <int TPI>
cudaError_t launch_tpi(const Problem& P, const SspOut& o, cudaStream_t st, int num_sms, bool smem_tier) {
  if (!smem_tier) return launch_one<256, false, false, false>(P, o, st, num_sms);
  if (P.tile8s) {  // the 8-bit shared-memory tiles
    if (P.hbits == 0) return launch_one<TPI, true, false, false, 1>(P, o, st, num_sms);
    cudaError_t e = launch_one<TPI, true, true, false, 1>(P, o, st, num_sms);
    if (e != cudaSuccess) return e;
    return launch_one<TPI, true, false, true, 1>(P, o, st, num_sms);
  }
  if (P.tile16s) {  // the 16-bit shared-memory tiles
    if (P.hbits == 0) return launch_one<TPI, true, false, false, 2>(P, o, st, num_sms);
    cudaError_t e = launch_one<TPI, true, true, false, 2>(P, o, st, num_sms);
    if (e != cudaSuccess) return e;
    return launch_one<TPI, true, false, true, 2>(P, o, st, num_sms);
  }
  if (P.hbits == 0) return launch_one<TPI, true, false, false>(P, o, st, num_sms);
  cudaError_t e = launch_one<TPI, true, true, false>(P, o, st, num_sms);
  if (e != cudaSuccess) return e;
  // instances whose 32-bit keys could overflow re-run with 64-bit keys (usually none)
  return launch_one<TPI, true, false, true>(P, o, st, num_sms);
}

}  // namespace

size_t ssp_smem_bytes(const Problem& P) { return ssp_layout(P, true, 8).total; }
size_t ssp_global_ws_bytes(const Problem& P) { return ssp_layout(P, false, 8).total; }

int ssp_launch_count(const Problem& P, int force_tier) {
  const bool smem_tier = force_tier == 0 && ssp_smem_bytes(P) <= 227 * 1024;
  if (!smem_tier) return 1;           // cluster tier or global tier: one kernel
  return P.hbits == 0 ? 1 : 2;        // 32-bit keys: the solve and its 64-bit redo launch
}

cudaError_t launch_ssp(const Problem& P, const SspOut& o, cudaStream_t st, int num_sms, int force_tier) {
  // counters [0] ssp queue, [2] redo count, [3] redo queue ([1] is the rounds queue, which may be
  // running concurrently on another stream: gwtf_flow_solve_and_rounds)
  cudaError_t e = cudaMemsetAsync(P.counters, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(P.counters + 2, 0, 2 * sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const bool smem_tier = force_tier == 0 && ssp_smem_bytes(P) <= 227 * 1024;
  if (!smem_tier) {
    if (force_tier != 1 && P.cluster_size > 0) return launch_ssp_cluster(P, o, st, P.cluster_size);
    return launch_tpi<256>(P, o, st, num_sms, false);
  }
  // team size: about one thread per destination row to start with, then doubled while the teams
  // that fit in an SM's shared memory would leave it with fewer than 512 threads
  int tpi = P.n <= 32 ? 32 : P.n <= 64 ? 64 : P.n <= 128 ? 128 : 256;
  const long long teams_per_sm =
      std::max<long long>(1, (long long)(227 * 1024) / (long long)ssp_layout(P, true, 4, P.tile8s ? 1 : P.tile16s ? 2 : 4).total);
  while (tpi < 512 && teams_per_sm * tpi < 512) tpi *= 2;
  // multi-warp teams (named barriers) keep doubling up to 1,024 threads per SM: measured with the
  // 16-bit tiles, llama 64.4 -> 56.5 ms at 256 threads per team, churn 704 -> 574 ms at 512; a
  // single-warp team (gpt: 22 per SM) stays one warp (64 threads measured 2x slower)
  while (tpi >= 64 && tpi < 512 && teams_per_sm * tpi < 1024) tpi *= 2;
  if (const char* f = getenv("GWTF_SSP_TPI")) tpi = atoi(f);  // testing override
  if (tpi <= 32) return launch_tpi<32>(P, o, st, num_sms, true);
  if (tpi <= 64) return launch_tpi<64>(P, o, st, num_sms, true);
  if (tpi <= 128) return launch_tpi<128>(P, o, st, num_sms, true);
  if (tpi <= 256) return launch_tpi<256>(P, o, st, num_sms, true);
  return launch_tpi<512>(P, o, st, num_sms, true);
}

}  // namespace gwtf
