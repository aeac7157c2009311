// Exact solve: canonical successive shortest paths for a batch of instances.
//
// One team of TPI threads per instance, persistent over an atomic instance queue.  The
// instance's cost tiles are staged once into shared memory by the TMA bulk-copy engine
// (cp.async.bulk + mbarrier) and every Bellman-Ford sweep of every augmentation then reads
// them from shared memory.  The dominant step is the dense min-plus relaxation of one
// stage boundary,
//     key_in[s+1][v] = min(key_in[s+1][v], min_u key_out[s][u] + (C[s][v][u], 1))
// done by groups of G lanes per destination row v (the dest-major tile row is read as
// 128-bit vectors, 4 sources per lane per load) followed by a shuffle-min across the group.
// The in->out node arc of v is fused into the owner's write.  Reverse residual arcs are
// relaxed from the per-boundary list of positive-flow arcs.  The augmenting path is traced
// by warp 0 with ballots (lowest (layer, position) tight predecessor) and augmented in place.
#include "common.cuh"

namespace gwtf {

namespace {

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

struct SspLayout {
  size_t misc, tile, kin, kout, g, capE, src, snk, srcf, snkf, arcs, cnt, path, total;
};

// misc block: 0 mbarrier | 8 F | 16 cost | 24 tnew | 32 A | 36 status | 40 inst
__host__ __device__ inline SspLayout ssp_layout(const Problem& P, bool with_tile) {
  SspLayout L;
  size_t o = 0;
  const size_t Sn = (size_t)P.S * P.n;
  const size_t nb = (size_t)(P.S > 1 ? P.S - 1 : 0);
  L.misc = o; o += 64;
  L.tile = o; if (with_tile) o += al16(nb * P.n * P.ld * 4);
  L.kin = o; o += al16((Sn + 4) * 8);
  L.kout = o; o += al16((Sn + 4) * 8);
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

template <int TPI, bool kSmem>
__global__ void __launch_bounds__(256) ssp_kernel(const Problem P, const SspOut o, const size_t ws_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Team<TPI> T{(int)(threadIdx.x % TPI), (int)(threadIdx.x / TPI)};
  const int teams_per_cta = blockDim.x / TPI;
  uint8_t* base;
  if constexpr (kSmem) base = smem + (size_t)T.id * ws_bytes;
  else base = P.ws + (size_t)(blockIdx.x * teams_per_cta + T.id) * ws_bytes;
  const SspLayout L = ssp_layout(P, kSmem);
  uint64_t* mbar = (uint64_t*)(base + L.misc);
  int64_t* F_p = (int64_t*)(base + L.misc + 8);
  int64_t* cost_p = (int64_t*)(base + L.misc + 16);
  uint64_t* tnew = (uint64_t*)(base + L.misc + 24);
  int32_t* A_p = (int32_t*)(base + L.misc + 32);
  int32_t* status_p = (int32_t*)(base + L.misc + 36);
  int32_t* inst_p = (int32_t*)(base + L.misc + 40);
  uint64_t* kin = (uint64_t*)(base + L.kin);
  uint64_t* kout = (uint64_t*)(base + L.kout);
  int32_t* g = (int32_t*)(base + L.g);
  int32_t* capE = (int32_t*)(base + L.capE);
  int32_t* src = (int32_t*)(base + L.src);
  int32_t* snk = (int32_t*)(base + L.snk);
  int32_t* srcf = (int32_t*)(base + L.srcf);
  int32_t* snkf = (int32_t*)(base + L.snkf);
  uint32_t* arcs = (uint32_t*)(base + L.arcs);
  int32_t* cnt = (int32_t*)(base + L.cnt);
  uint32_t* path = (uint32_t*)(base + L.path);

  const int S = P.S, n = P.n, ld = P.ld, Sn = S * n, Lcap = P.Lcap;
  const int chunks = ld / 4;
  int G = 1;
  while (G * 2 <= chunks && G * 2 <= 32) G *= 2;  // lanes per destination row
  const int NG = TPI / G, gi = T.tid / G, li = T.tid % G;
  const int lane = threadIdx.x & 31;
  const int Lt = 2 * S + 1;  // layer of t*
  const size_t tile_elems = (size_t)(S - 1) * n * ld;
  const uint32_t tile_bytes = (uint32_t)(tile_elems * 4);
  uint32_t phase = 0;

  if (kSmem && T.tid == 0) {
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  T.sync();

  for (;;) {
    if (T.tid == 0) *inst_p = atomicAdd(&P.counters[0], 1);
    T.sync();
    const int inst = *inst_p;
    if (inst >= P.B) break;

    // ---- stage the instance: tiles by TMA bulk copy, the rest by plain loads ----
    const int32_t* gtile = P.tile + (size_t)inst * tile_elems;
    const int32_t* tile = gtile;
    if constexpr (kSmem) {
      tile = (const int32_t*)(base + L.tile);
      if (T.tid == 0 && tile_bytes) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(mbar, tile_bytes);
        for (uint32_t off = 0; off < tile_bytes; off += 32768u)
          bulk_g2s((uint8_t*)(base + L.tile) + off, (const uint8_t*)gtile + off,
                   tile_bytes - off < 32768u ? tile_bytes - off : 32768u, mbar);
      }
    }
    const int64_t M = P.supply[inst];
    for (int k = T.tid; k < Sn; k += TPI) {
      g[k] = 0;
      capE[k] = P.alive[(size_t)inst * Sn + k] ? P.cap[(size_t)inst * Sn + k] : 0;
    }
    for (int i = T.tid; i < n; i += TPI) {
      src[i] = P.src[(size_t)inst * n + i];
      snk[i] = P.snk[(size_t)inst * n + i];
      srcf[i] = 0;
      snkf[i] = 0;
    }
    for (int k = T.tid; k < S; k += TPI) cnt[k] = 0;
    if (T.tid == 0) { *F_p = 0; *cost_p = 0; *A_p = 0; *status_p = 0; }
    if (kSmem && tile_bytes) { mbar_wait(mbar, phase); phase ^= 1u; }
    T.sync();

    // ---- successive shortest paths ----
    for (;;) {
      const int64_t F = *F_p;
      if (F >= M || *status_p) break;
      for (int k = T.tid; k < Sn + 4; k += TPI) { kin[k] = kKeyInf; kout[k] = kKeyInf; }
      uint64_t tkey = kKeyInf;
      T.sync();
      int more = 1;
      while (more) {  // Bellman-Ford sweeps to the fixed point
        int ch = 0;
        if (T.tid == 0) *tnew = kKeyInf;
        // s* -> in_0 (cost src, 1 hop), then in_0 -> out_0 where g < cap
        for (int vb = 0; vb < n; vb += NG) {
          const int v = vb + gi;
          if (li == 0 && v < n) {
            uint64_t kv = kin[v];
            if (src[v] != kAbsent) {
              const uint64_t c = ((uint64_t)(uint32_t)src[v] << kHopBits) | 1ull;
              if (c < kv) { kin[v] = c; kv = c; ch = 1; }
            }
            if (kv != kKeyInf && g[v] < capE[v] && kv + 1 < kout[v]) { kout[v] = kv + 1; ch = 1; }
          }
        }
        T.sync();
        // forward: dense min-plus relaxation of every stage boundary
        for (int s = 0; s + 1 < S; ++s) {
          const int32_t* Ts = tile + (size_t)s * n * ld;
          const uint64_t* ko = kout + (size_t)s * n;
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            uint64_t acc = kKeyInf;
            if (v < n) {
              const int4* row = (const int4*)(Ts + (size_t)v * ld);
              for (int c = li; c < chunks; c += G) {
                const int4 w = row[c];
                const int u = 4 * c;
                if (w.x != kAbsent) { const uint64_t k = ko[u + 0]; if (k != kKeyInf) acc = umin64(acc, key_fwd(k, w.x)); }
                if (w.y != kAbsent) { const uint64_t k = ko[u + 1]; if (k != kKeyInf) acc = umin64(acc, key_fwd(k, w.y)); }
                if (w.z != kAbsent) { const uint64_t k = ko[u + 2]; if (k != kKeyInf) acc = umin64(acc, key_fwd(k, w.z)); }
                if (w.w != kAbsent) { const uint64_t k = ko[u + 3]; if (k != kKeyInf) acc = umin64(acc, key_fwd(k, w.w)); }
              }
            }
            for (int off = G >> 1; off > 0; off >>= 1) acc = umin64(acc, shfl_xor_u64(acc, off, G));
            if (v < n && li == 0) {
              const int idx = (s + 1) * n + v;
              uint64_t kv = kin[idx];
              if (acc < kv) { kin[idx] = acc; kv = acc; ch = 1; }
              if (kv != kKeyInf && g[idx] < capE[idx] && kv + 1 < kout[idx]) { kout[idx] = kv + 1; ch = 1; }
            }
          }
          T.sync();
        }
        // out_{S-1} -> t*
        {
          uint64_t tc = kKeyInf;
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            if (li == 0 && v < n && snk[v] != kAbsent) {
              const uint64_t k = kout[(S - 1) * n + v];
              if (k != kKeyInf) tc = umin64(tc, key_fwd(k, snk[v]));
            }
          }
          for (int off = 16; off > 0; off >>= 1) tc = umin64(tc, shfl_xor_u64(tc, off, 32));
          if (lane == 0 && tc != kKeyInf) atomicMin((unsigned long long*)tnew, (unsigned long long)tc);
        }
        T.sync();
        {
          const uint64_t tn = *tnew;
          if (tn < tkey) { tkey = tn; if (T.tid == 0) ch = 1; }
        }
        // t* -> out_{S-1} (reverse sink arcs, snk_f > 0)
        if (tkey != kKeyInf) {
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            if (li == 0 && v < n && snkf[v] > 0) {
              const int idx = (S - 1) * n + v;
              const uint64_t c = tkey - ((uint64_t)(uint32_t)snk[v] << kHopBits) + 1ull;
              if (c < kout[idx]) { kout[idx] = c; ch = 1; }
            }
          }
        }
        T.sync();
        // backward: reverse node arcs out_s -> in_s (g > 0) and reverse inter-stage arcs
        // in_s -> out_{s-1} over the positive-flow list of boundary s-1
        for (int s = S - 1; s >= 0; --s) {
          for (int vb = 0; vb < n; vb += NG) {
            const int v = vb + gi;
            if (li == 0 && v < n) {
              const int idx = s * n + v;
              const uint64_t ko = kout[idx];
              if (g[idx] > 0 && ko != kKeyInf && ko + 1 < kin[idx]) { kin[idx] = ko + 1; ch = 1; }
            }
          }
          if (s == 0) break;
          const uint32_t* al = arcs + (size_t)(s - 1) * Lcap;
          const int c = cnt[s - 1];
          for (int e = T.tid; e < c; e += TPI) {
            const uint32_t ent = al[e];
            const int u = (int)(ent >> 20), v = (int)((ent >> 8) & 0xFFFu);
            const int idx = s * n + v;
            uint64_t ki = kin[idx];
            const uint64_t kov = kout[idx];
            if (g[idx] > 0 && kov != kKeyInf) ki = umin64(ki, kov + 1);
            if (ki == kKeyInf) continue;
            const int32_t C = tile[((size_t)(s - 1) * n + v) * ld + u];
            const uint64_t cand = ki - ((uint64_t)(uint32_t)C << kHopBits) + 1ull;
            const uint64_t old = atomicMin((unsigned long long*)&kout[(s - 1) * n + u], (unsigned long long)cand);
            if (cand < old) ch = 1;
          }
          T.sync();
        }
        more = T.sync_or(ch);
      }
      if (tkey == kKeyInf) break;  // t* unreachable: F is the maximum flow

      // ---- trace the canonical augmenting path and augment (warp 0) ----
      if (T.tid < 32) {
        auto key_of = [&](int id) -> uint64_t {
          const int l = id / n, p = id % n;
          if (l == 0) return 0ull;
          if (l == Lt) return tkey;
          if (l & 1) return kin[((l - 1) / 2) * n + p];
          return kout[(l / 2 - 1) * n + p];
        };
        const int maxlen = 2 * Sn + 2;
        int x = Lt * n, len = 1, err = 0;
        if (lane == 0) path[0] = (uint32_t)x;
        while (x != 0) {
          const int l = x / n, p = x % n;
          const uint64_t kx = key_of(x);
          int pred = -1;
          if (l == Lt) {
            for (int b = 0; b < n && pred < 0; b += 32) {
              const int i = b + lane;
              bool ok = false;
              if (i < n && snk[i] != kAbsent) {
                const uint64_t k = kout[(S - 1) * n + i];
                ok = k != kKeyInf && key_fwd(k, snk[i]) == kx;
              }
              const uint32_t m = __ballot_sync(0xffffffffu, ok);
              if (m) pred = (2 * S) * n + b + __ffs(m) - 1;
            }
          } else if (l & 1) {  // in_{s,i}: s* or out_{s-1,u} (layer 2s) first, then out_{s,i} (layer 2s+2)
            const int s = (l - 1) / 2, i = p;
            if (s == 0) {
              if (src[i] != kAbsent && ((((uint64_t)(uint32_t)src[i]) << kHopBits) | 1ull) == kx) pred = 0;
            } else {
              const int32_t* row = tile + ((size_t)(s - 1) * n + i) * ld;
              for (int b = 0; b < n && pred < 0; b += 32) {
                const int u = b + lane;
                bool ok = false;
                if (u < n && row[u] != kAbsent) {
                  const uint64_t k = kout[(s - 1) * n + u];
                  ok = k != kKeyInf && key_fwd(k, row[u]) == kx;
                }
                const uint32_t m = __ballot_sync(0xffffffffu, ok);
                if (m) pred = (2 * s) * n + b + __ffs(m) - 1;
              }
            }
            if (pred < 0) {
              const int idx = s * n + i;
              if (g[idx] > 0 && kout[idx] != kKeyInf && kout[idx] + 1 == kx) pred = (2 * s + 2) * n + i;
            }
          } else {  // out_{s,i}: in_{s,i} (2s+1), then in_{s+1,v} reverse (2s+3), then t* reverse
            const int s = l / 2 - 1, i = p, idx = s * n + i;
            if (g[idx] < capE[idx] && kin[idx] != kKeyInf && kin[idx] + 1 == kx) {
              pred = (2 * s + 1) * n + i;
            } else if (s < S - 1) {
              const uint32_t* al = arcs + (size_t)s * Lcap;
              const int c = cnt[s];
              uint32_t best = 0xFFFFFFFFu;
              for (int e = lane; e < c; e += 32) {
                const uint32_t ent = al[e];
                if ((int)(ent >> 20) != i) continue;
                const int v = (int)((ent >> 8) & 0xFFFu);
                const uint64_t k = kin[(s + 1) * n + v];
                const int32_t C = tile[((size_t)s * n + v) * ld + i];
                if (k != kKeyInf && k + 1 == kx + ((uint64_t)(uint32_t)C << kHopBits)) best = min(best, (uint32_t)v);
              }
              best = __reduce_min_sync(0xffffffffu, best);
              if (best != 0xFFFFFFFFu) pred = (2 * s + 3) * n + (int)best;
            } else if (snkf[i] > 0 && tkey + 1 == kx + ((uint64_t)(uint32_t)snk[i] << kHopBits)) {
              pred = Lt * n;
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
            const int lu = u / n, lv = v / n, pu = u % n, pv = v % n;
            long long r = LLONG_MAX;
            if (u == 0 || v == Lt * n) {
            } else if ((lu & 1) && lv == lu + 1) {
              const int idx = ((lu - 1) / 2) * n + pu;
              r = capE[idx] - g[idx];
            } else if (!(lu & 1) && lv == lu - 1) {
              r = g[(lu / 2 - 1) * n + pu];
            } else if ((lu & 1) && lv == lu - 1) {
              const int s = lv / 2 - 1;
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
              const int lu = u / n, lv = v / n, pu = u % n, pv = v % n;
              if (u == 0) {
                if (lane == 0) srcf[pv] += (int32_t)d;
              } else if (v == Lt * n) {
                if (lane == 0) snkf[pu] += (int32_t)d;
              } else if ((lu & 1) && lv == lu + 1) {
                if (lane == 0) g[((lu - 1) / 2) * n + pu] += (int32_t)d;
              } else if (!(lu & 1) && lv == lu - 1) {
                if (lane == 0) g[(lu / 2 - 1) * n + pu] -= (int32_t)d;
              } else {
                const bool fwd = !(lu & 1);
                const int s = fwd ? lu / 2 - 1 : lv / 2 - 1;
                const uint32_t uu = fwd ? pu : pv, vv = fwd ? pv : pu;
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
                    const int f = (int)(al[found] & 0xFFu) + (fwd ? (int)d : -(int)d);
                    if (f > 0) {
                      al[found] = (uu << 20) | (vv << 8) | (uint32_t)f;
                    } else {
                      al[found] = al[c - 1];
                      cnt[s] = c - 1;
                    }
                  } else if (fwd && c < Lcap) {
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
              *cost_p += (int64_t)d * (int64_t)(tkey >> kHopBits);
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
      o.F[inst] = *F_p;
      o.cost[inst] = *cost_p;
      if (o.A) o.A[inst] = *A_p;
      if (o.status) o.status[inst] = *status_p;
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

template <int TPI>
cudaError_t launch_tpi(const Problem& P, const SspOut& o, cudaStream_t st, int num_sms, bool smem_tier) {
  const size_t ws = ssp_layout(P, smem_tier).total;
  if (smem_tier) {
    const size_t limit = 227 * 1024;
    int teams = TPI >= 128 ? 1 : 128 / TPI;
    while (teams > 1 && teams * ws > limit) --teams;
    const size_t smem = teams * ws;
    auto k = ssp_kernel<TPI, true>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, teams * TPI, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    long long grid = (long long)per_sm * num_sms;
    const long long need = (P.B + teams - 1) / teams;
    if (grid > need) grid = need;
    k<<<(int)grid, teams * TPI, smem, st>>>(P, o, ws);
  } else {
    long long grid = P.ws_teams;
    if (grid > P.B) grid = P.B;
    ssp_kernel<TPI, false><<<(int)grid, TPI, 0, st>>>(P, o, ws);
  }
  return cudaGetLastError();
}

}  // namespace

size_t ssp_smem_bytes(const Problem& P) { return ssp_layout(P, true).total; }
size_t ssp_global_ws_bytes(const Problem& P) { return ssp_layout(P, false).total; }

cudaError_t launch_ssp(const Problem& P, const SspOut& o, cudaStream_t st, int num_sms, bool force_global) {
  cudaError_t e = cudaMemsetAsync(P.counters, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const bool smem_tier = !force_global && ssp_smem_bytes(P) <= 227 * 1024;
  if (!smem_tier) return launch_tpi<256>(P, o, st, num_sms, false);
  if (P.n <= 32) return launch_tpi<32>(P, o, st, num_sms, true);
  if (P.n <= 64) return launch_tpi<64>(P, o, st, num_sms, true);
  if (P.n <= 128) return launch_tpi<128>(P, o, st, num_sms, true);
  return launch_tpi<256>(P, o, st, num_sms, true);
}

}  // namespace gwtf
