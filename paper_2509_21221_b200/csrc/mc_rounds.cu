// Multi-data-node decentralized rounds, MC-SYNC.
// "each data node ... must receive its own flow back", "unpaired outflow" per data node,
// flow-test settings 5-6.  K data nodes D_0..D_{K-1} share the relays and links; each
// has its own supply, SRC_k / SNK_k slots and source / sink costs.  Every non-FREE relay slot
// carries the data node (tag) of its chain, so requests, grants, Change and self-pairing stay
// within one data node; with K = 1 every rule is the single-commodity one (rounds.cu).
//
// One CTA per instance (grid-stride over the batch), the whole instance state in shared memory
// (the flow-test shapes are small), relay-parallel phases separated by __syncthreads, every phase
// a pure function of the state the definition names (the oracle's McRounds, oracle.cpp):
//   R0a self-pairing (round-start costs) | R0 costs back to front, adv(v, k) | R1 one request per
//   node (D_0..D_{K-1}, then relays) | R2 + R3 grants per target and tag, in requester order |
//   R4 Change / Redirect / DENY proposals (counter RNG, integer annealing thresholds) | R5 64-bit
//   atomicMin reservations | R6 commits | R7 quiet counter, optional digest.
// Pointers: relay slot >= 0, kNone, data-node slot i of D_k = -2 - (k * Mmax + i).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace gwtf {

namespace {

constexpr int kT = 256;  // threads per instance
constexpr int64_t INF = INT64_MAX;
constexpr uint64_t RES_NONE = ~0ull;
enum { K_NONE = 0, K_CHANGE = 1, K_REDIRECT = 2, K_DENY = 3 };
enum { ST_FREE = 0, ST_OUT = 1, ST_IN = 2, ST_PAIRED = 3 };

__device__ __forceinline__ uint64_t mix(uint64_t z) {  // splitmix64 finalizer
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t pick(uint64_t x, uint32_t m) { return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32); }
__device__ __forceinline__ int64_t sadd(int64_t a, int64_t b) { return (a == INF || b == INF) ? INF : a + b; }
__device__ __forceinline__ int64_t cst(int32_t c) { return c == kAbsent ? INF : (int64_t)c; }
__device__ __forceinline__ uint64_t dig(uint64_t pos, uint64_t val) { return mix(mix(pos) ^ val); }

struct McArgs {
  int32_t B, S, n, MC, K, Mmax;
  const int32_t* cap;    // [B][S][n]
  const uint8_t* alive;  // [B][S][n] or null
  const int32_t* tile;   // [B][S-1][n][ld]
  int32_t ld;
  const int32_t* src;    // [K][B][n]
  const int32_t* snk;    // [K][B][n]
  const int64_t* supply; // [K][B]
  uint64_t seed;
  int64_t inst_base;
  int32_t objective, W, deny_after, max_rounds;
  const uint32_t* thr;
  int32_t thr_width, thr_K;
  int32_t* rounds_run;   // [B]
  int64_t* F_dec;        // [K][B]
  int64_t* cost_dec;     // [K][B]
  int32_t* dangling;     // [B]
  uint64_t* digests;     // [B][max_rounds] or null
  int32_t *up_out, *down_out, *tag_out;  // [B][S][n][MC] or null (final state)
  int32_t *sd_out, *su_out;              // [B][K][Mmax] or null
  int32_t resume;                        // start from the state in the five arrays above
  int64_t round0;                        // the RNG round counter at the start
};

struct McLayout { size_t up, down, tag, sd, su, kacc, deny, capv, scost, adv, rs, rt, rk, prop, ptouch, pkey, res, red, total; };
__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline McLayout mc_layout(int S, int n, int MC, int K, int Mmax) {
  McLayout L;
  const size_t Sn = (size_t)S * n, ns = Sn * MC, nd = (size_t)K * Mmax;
  size_t o = 0;
  L.up = o; o += al16(ns * 4);
  L.down = o; o += al16(ns * 4);
  L.tag = o; o += al16(ns * 4);
  L.sd = o; o += al16(nd * 4);
  L.su = o; o += al16(nd * 4);
  L.kacc = o; o += al16(Sn * 4);
  L.deny = o; o += al16(Sn * 4);
  L.capv = o; o += al16(Sn * 4);
  L.scost = o; o += al16(ns * 8);
  L.adv = o; o += al16(Sn * K * 8);
  L.rs = o; o += al16((Sn + K) * 4);   // requester slot (relays, then D_k)
  L.rt = o; o += al16((Sn + K) * 4);   // target: relay gid, -1-k = D_k-sink, INT_MIN = none
  L.rk = o; o += al16(Sn * 4);         // commodity of the request
  L.prop = o; o += al16(Sn * 4 * 4);
  L.ptouch = o; o += al16(Sn * 4 * 4);
  L.pkey = o; o += al16(Sn * 8);
  L.res = o; o += al16((ns + 2 * nd) * 8);
  L.red = o; o += 64;
  L.total = o;
  return L;
}

__global__ void __launch_bounds__(kT) mc_rounds_kernel(const McArgs A) {
  extern __shared__ __align__(16) uint8_t smb[];
  const int S = A.S, n = A.n, MC = A.MC, K = A.K, Mmax = A.Mmax, Sn = S * n, ns = Sn * MC, tid = threadIdx.x;
  const McLayout L = mc_layout(S, n, MC, K, Mmax);
  int32_t* up = (int32_t*)(smb + L.up);
  int32_t* down = (int32_t*)(smb + L.down);
  int32_t* tag = (int32_t*)(smb + L.tag);
  int32_t* sd = (int32_t*)(smb + L.sd);
  int32_t* su = (int32_t*)(smb + L.su);
  int32_t* kacc = (int32_t*)(smb + L.kacc);
  int32_t* deny = (int32_t*)(smb + L.deny);
  int32_t* capv = (int32_t*)(smb + L.capv);
  int64_t* scost = (int64_t*)(smb + L.scost);
  int64_t* adv = (int64_t*)(smb + L.adv);
  int32_t* rs = (int32_t*)(smb + L.rs);
  int32_t* rt = (int32_t*)(smb + L.rt);
  int32_t* rk = (int32_t*)(smb + L.rk);
  int32_t* prop = (int32_t*)(smb + L.prop);
  int32_t* ptouch = (int32_t*)(smb + L.ptouch);
  uint64_t* pkey = (uint64_t*)(smb + L.pkey);
  uint64_t* res = (uint64_t*)(smb + L.res);
  unsigned long long* red = (unsigned long long*)(smb + L.red);  // [0] changes, [1..] sums
  for (int b = blockIdx.x; b < A.B; b += gridDim.x) {
    const int32_t* tile = A.tile + (size_t)b * (S > 1 ? S - 1 : 0) * n * A.ld;
    auto srcc = [&](int k, int i) -> int64_t { return cst(A.src[((size_t)k * A.B + b) * n + i]); };
    auto snkc = [&](int k, int i) -> int64_t { return cst(A.snk[((size_t)k * A.B + b) * n + i]); };
    auto Mk = [&](int k) -> int { return (int)A.supply[(size_t)k * A.B + b]; };
    auto alive = [&](int g) -> bool { return A.alive == nullptr || A.alive[(size_t)b * Sn + g] != 0; };
    auto st = [&](int p) -> int { return (up[p] != kNone ? 2 : 0) | (down[p] != kNone ? 1 : 0); };
    auto dk = [&](int32_t p) -> int { return (-2 - p) / Mmax; };
    auto di = [&](int32_t p) -> int { return (-2 - p) % Mmax; };
    // d(a, c): node -1-k = data node k (SRC side for a, SNK side for c); absent / impossible = INF
    auto d = [&](int a, int c) -> int64_t {
      if (a < 0) return (c >= 0 && c < n) ? srcc(-1 - a, c) : INF;
      const int sa = a / n;
      if (c < 0) return sa == S - 1 ? snkc(-1 - c, a - sa * n) : INF;
      if (c / n != sa + 1) return INF;
      return cst(tile[((size_t)sa * n + (c - (sa + 1) * n)) * A.ld + (a - sa * n)]);
    };
    auto node_of = [&](int32_t p) -> int { return p >= 0 ? p / MC : -1 - dk(p); };
    auto set_up_of = [&](int32_t p, int32_t v) { if (p >= 0) up[p] = v; else su[dk(p) * Mmax + di(p)] = v; };
    auto set_down_of = [&](int32_t p, int32_t v) { if (p >= 0) down[p] = v; else sd[dk(p) * Mmax + di(p)] = v; };
    auto res_up = [&](int32_t p) -> int { return p >= 0 ? p : ns + (-2 - p); };
    auto res_dn = [&](int32_t p) -> int { return p >= 0 ? p : ns + K * Mmax + (-2 - p); };
    if (A.resume) {  // a given state (the export layouts; tag -1 on FREE slots)
      for (int p = tid; p < ns; p += kT) {
        up[p] = A.up_out[(size_t)b * ns + p];
        down[p] = A.down_out[(size_t)b * ns + p];
        tag[p] = max(A.tag_out[(size_t)b * ns + p], 0);
      }
      for (int k = tid; k < K * Mmax; k += kT) { sd[k] = A.sd_out[(size_t)b * K * Mmax + k]; su[k] = A.su_out[(size_t)b * K * Mmax + k]; }
    } else {
      for (int p = tid; p < ns; p += kT) { up[p] = kNone; down[p] = kNone; tag[p] = 0; }
      for (int k = tid; k < K * Mmax; k += kT) { sd[k] = kNone; su[k] = kNone; }
    }
    for (int v = tid; v < Sn; v += kT) { kacc[v] = 0; deny[v] = 0; capv[v] = alive(v) ? A.cap[(size_t)b * Sn + v] : 0; }
    for (int k = tid; k < ns + 2 * K * Mmax; k += kT) res[k] = RES_NONE;
    __syncthreads();
    // R0: cost to sink back to front (stage-synchronous)
    auto costs = [&]() {
      for (int s = S - 1; s >= 0; --s) {
        for (int t = tid; t < n * MC; t += kT) {
          const int i = t / MC, j = t - i * MC, v = s * n + i, p = v * MC + j;
          int64_t c = INF;
          if (j < capv[v] && down[p] != kNone) c = down[p] <= -2 ? d(v, -1 - dk(down[p])) : sadd(d(v, down[p] / MC), scost[down[p]]);
          scost[p] = c;
        }
        __syncthreads();
      }
    };
    int quiet = 0, r = 0;
    uint64_t round = (uint64_t)A.round0;
    const uint64_t hinst = mix(mix(A.seed) ^ (uint64_t)(A.inst_base + b));  // fixed per instance
    while (r < A.max_rounds) {
      const uint64_t hpre = mix(hinst ^ round);
      auto h = [&](int gid, int stream) -> uint64_t { return mix(hpre ^ ((uint64_t)gid * 4 + stream)); };
      if (tid == 0) red[0] = 0;
      // ---- R0a self-pairing on round-start costs ----
      costs();
      int changed = 0;
      for (int v = tid; v < Sn; v += kT) {
        if (!alive(v)) continue;
        int x = -1, o = -1;
        for (int j = 0; j < capv[v] && x < 0; ++j) {
          const int p = v * MC + j;
          if (st(p) != ST_IN) continue;
          int ob = -1;
          for (int jj = 0; jj < capv[v]; ++jj) {
            const int q = v * MC + jj;
            if (st(q) == ST_OUT && tag[q] == tag[p] && (ob < 0 || scost[q] < scost[ob])) ob = q;
          }
          if (ob >= 0) { x = p; o = ob; }
        }
        if (x < 0) continue;
        const int32_t cdn = down[o];
        down[x] = cdn;
        set_up_of(cdn, x);
        down[o] = kNone;
        changed = 1;
      }
      __syncthreads();
      // ---- R0 costs on the post-R0a state, advertisements per tag ----
      costs();
      for (int t = tid; t < Sn * K; t += kT) {
        const int v = t / K, k = t - v * K;
        int64_t best = INF;
        if (alive(v))
          for (int j = 0; j < capv[v]; ++j) {
            const int p = v * MC + j;
            if (st(p) == ST_OUT && tag[p] == k && scost[p] < best) best = scost[p];
          }
        adv[t] = best;
      }
      __syncthreads();
      // ---- R1 requests ----
      for (int rr = tid; rr < Sn; rr += kT) {
        int32_t x = kNone, tg = INT32_MIN, kk = -1;
        if (alive(rr)) {
          int xin = -1, xfree = -1;
          bool has_out = false;
          for (int j = 0; j < capv[rr]; ++j) {
            const int p = rr * MC + j, t = st(p);
            if (t == ST_IN && xin < 0) xin = p;
            if (t == ST_FREE && xfree < 0) xfree = p;
            if (t == ST_OUT) has_out = true;
          }
          int32_t cand = kNone;
          if (xin >= 0) cand = xin;
          else if (!has_out && xfree >= 0) cand = xfree;
          if (cand != kNone) {
            const int s = rr / n, i = rr - s * n;
            const int klo = xin >= 0 ? tag[xin] : 0, khi = xin >= 0 ? tag[xin] : K - 1;
            int64_t bc = INF;
            if (s == S - 1) {
              for (int k = klo; k <= khi; ++k) {
                bool fr = false;
                for (int q = 0; q < Mk(k) && !fr; ++q) fr = su[k * Mmax + q] == kNone;
                const int64_t c = snkc(k, i);
                if (fr && c != INF && c < bc) { bc = c; tg = -1 - k; kk = k; }
              }
            } else {
              for (int jj = 0; jj < n; ++jj) {
                const int j = (s + 1) * n + jj;
                const int64_t dj = d(rr, j);
                if (!alive(j) || dj == INF) continue;
                for (int k = klo; k <= khi; ++k) {
                  const int64_t a = adv[(size_t)j * K + k];
                  if (a != INF && dj + a < bc) { bc = dj + a; tg = j; kk = k; }
                }
              }
            }
            if (kk >= 0) x = cand;
          }
        }
        rs[rr] = x;
        rt[rr] = kk >= 0 ? tg : INT32_MIN;
        rk[rr] = kk;
      }
      for (int k = tid; k < K; k += kT) {  // D_k: lowest unpaired SRC_k slot -> stage-0 advertisers of tag k
        int slot = -1, tg = INT32_MIN;
        for (int q = 0; q < Mk(k); ++q) if (sd[k * Mmax + q] == kNone) { slot = q; break; }
        if (slot >= 0) {
          int64_t bc = INF;
          for (int j = 0; j < n; ++j) {
            const int64_t a = adv[(size_t)j * K + k], c = srcc(k, j);
            if (alive(j) && c != INF && a != INF && c + a < bc) { bc = c + a; tg = j; }
          }
        }
        rs[Sn + k] = tg != INT32_MIN ? -2 - (k * Mmax + slot) : kNone;
        rt[Sn + k] = tg;
      }
      __syncthreads();
      // ---- R2 + R3: per target relay and tag, requesters in order (D_k first, then relays by gid) ----
      for (int t = tid; t < Sn * K; t += kT) {
        const int j = t / K, k = t - j * K;
        const int64_t ac = adv[t];
        if (ac == INF) continue;
        const int s = j / n;
        int cur = 0;
        auto next_slot = [&]() -> int {
          while (cur < capv[j]) {
            const int p = j * MC + cur++;
            if (st(p) == ST_OUT && tag[p] == k && scost[p] == ac) return p;
          }
          return -1;
        };
        if (s == 0) {
          if (rt[Sn + k] == j) {
            const int p = next_slot();
            if (p >= 0) { sd[dk(rs[Sn + k]) * Mmax + di(rs[Sn + k])] = p; up[p] = rs[Sn + k]; changed = 1; }
          }
          continue;
        }
        for (int q = (s - 1) * n; q < s * n; ++q) {
          if (rt[q] != j || rk[q] != k) continue;
          const int p = next_slot();
          if (p < 0) break;
          down[rs[q]] = p;
          tag[rs[q]] = k;
          up[p] = rs[q];
          deny[q] = 0;
          changed = 1;
        }
      }
      for (int k = tid; k < K; k += kT) {  // D_k-sink: free SNK_k slots in index order, gid order
        int q = 0;
        for (int g = (S - 1) * n; g < Sn; ++g) {
          if (rt[g] != -1 - k) continue;
          while (q < Mk(k) && su[k * Mmax + q] != kNone) ++q;
          if (q >= Mk(k)) break;
          down[rs[g]] = -2 - (k * Mmax + q);
          tag[rs[g]] = k;
          su[k * Mmax + q] = rs[g];
          deny[g] = 0;
          changed = 1;
          ++q;
        }
      }
      __syncthreads();
      // ---- R4 proposals by idle relays (post-R3 state) + R5 reservations ----
      for (int p = tid; p < Sn; p += kT) {
        int kind = K_NONE;
        int32_t x = kNone, y = kNone, z = kNone, t0 = -1, t1 = -1, t2 = -1, t3 = -1;
        uint64_t key = RES_NONE;
        if (alive(p) && rt[p] == INT32_MIN) {
          const int s = p / n, i = p - s * n;
          int xin = -1, zfree = -1, np = 0;
          bool has_out = false;
          for (int j = 0; j < capv[p]; ++j) {
            const int q = p * MC + j, t = st(q);
            if (t == ST_IN && xin < 0) xin = q;
            if (t == ST_FREE && zfree < 0) zfree = q;
            if (t == ST_OUT) has_out = true;
            np += t == ST_PAIRED;
          }
          if (xin >= 0) {  // DENY after deny_after idle rounds holding unpaired inflow
            deny[p] += 1;
            if (deny[p] >= A.deny_after) { kind = K_DENY; x = xin; t0 = xin; t1 = res_up(up[xin]); key = (uint64_t)p; }
          } else if (n >= 2) {
            uint32_t qi = pick(h(p, 0), (uint32_t)(n - 1));
            if ((int)qi >= i) qi += 1;
            const int q = s * n + (int)qi;
            int nq = 0;
            if (alive(q)) for (int j = 0; j < capv[q]; ++j) nq += st(q * MC + j) == ST_PAIRED;
            auto nth = [&](int v, int want) -> int {
              for (int j = 0; j < capv[v]; ++j)
                if (st(v * MC + j) == ST_PAIRED) { if (want == 0) return v * MC + j; --want; }
              return -1;
            };
            if (nq > 0) {
              int64_t delta = 0;
              bool ok = false;
              if (zfree >= 0 && !has_out) {  // Redirect: z takes y's (up, down, tag)
                y = nth(q, (int)pick(h(p, 2), (uint32_t)nq));
                const int a = node_of(up[y]), c = node_of(down[y]);
                const int64_t dax = d(a, p), dxc = d(p, c), dab = d(a, q), dbc = d(q, c);
                if (dax != INF && dxc != INF && dab != INF && dbc != INF) {
                  delta = A.objective == 0 ? (dax + dxc) - (dab + dbc) : max(dax, dxc) - max(dab, dbc);
                  kind = K_REDIRECT; z = zfree;
                  t0 = y; t1 = res_up(up[y]); t2 = res_dn(down[y]); t3 = z;
                  ok = true;
                }
              } else if (np > 0) {  // Change: both chains of the same data node
                x = nth(p, (int)pick(h(p, 1), (uint32_t)np));
                y = nth(q, (int)pick(h(p, 2), (uint32_t)nq));
                const int j1 = node_of(down[x]), j2 = node_of(down[y]);
                if (tag[x] == tag[y] && j1 != j2) {
                  const int64_t a1 = d(p, j2), a2 = d(q, j1), b1 = d(p, j1), b2 = d(q, j2);
                  if (a1 != INF && a2 != INF && b1 != INF && b2 != INF) {
                    delta = A.objective == 0 ? (a1 + a2) - (b1 + b2) : max(a1, a2) - max(b1, b2);
                    kind = K_CHANGE;
                    t0 = x; t1 = y; t2 = res_dn(down[x]); t3 = res_dn(down[y]);
                    ok = true;
                  }
                }
              }
              if (ok) {
                bool accept = delta < 0;
                if (delta > 0 && delta < A.thr_width) {
                  const int kk = min(kacc[p], A.thr_K);
                  accept = (h(p, 3) >> 32) < (uint64_t)A.thr[(size_t)kk * A.thr_width + delta];
                }
                if (accept) key = ((uint64_t)(delta + (1ll << 40)) << 22) | (uint64_t)p;
                else kind = K_NONE;
              }
            }
          }
        }
        if (key == RES_NONE) kind = K_NONE;
        prop[p * 4] = kind;
        if (kind != K_NONE) {
          prop[p * 4 + 1] = x; prop[p * 4 + 2] = y; prop[p * 4 + 3] = z;
          pkey[p] = key;
          ptouch[p * 4] = t0; ptouch[p * 4 + 1] = t1; ptouch[p * 4 + 2] = t2; ptouch[p * 4 + 3] = t3;
          atomicMin((unsigned long long*)&res[t0], (unsigned long long)key);
          atomicMin((unsigned long long*)&res[t1], (unsigned long long)key);
          if (t2 >= 0) atomicMin((unsigned long long*)&res[t2], (unsigned long long)key);
          if (t3 >= 0) atomicMin((unsigned long long*)&res[t3], (unsigned long long)key);
        }
      }
      __syncthreads();
      // ---- R6 commits ----
      for (int p = tid; p < Sn; p += kT) {
        const int kind = prop[p * 4];
        if (kind == K_NONE) continue;
        bool win = true;
        for (int q = 0; q < 4; ++q) { const int32_t t = ptouch[p * 4 + q]; if (t >= 0) win = win && res[t] == pkey[p]; }
        if (!win) continue;
        const int32_t x = prop[p * 4 + 1], y = prop[p * 4 + 2], z = prop[p * 4 + 3];
        if (kind == K_CHANGE) {
          const int32_t dx = down[x], dy = down[y];
          down[x] = dy; down[y] = dx;
          set_up_of(dy, x); set_up_of(dx, y);
          kacc[p] += 1;
        } else if (kind == K_REDIRECT) {
          const int32_t a = up[y], c = down[y];
          up[z] = a; down[z] = c; tag[z] = tag[y];
          set_down_of(a, z); set_up_of(c, z);
          up[y] = kNone; down[y] = kNone;
          kacc[p] += 1;
        } else {
          const int32_t a = up[x];
          up[x] = kNone;
          set_down_of(a, kNone);
          deny[p] = 0;
        }
        changed = 1;
      }
      __syncthreads();
      for (int p = tid; p < Sn; p += kT) {  // release the reservations
        if (prop[p * 4] == K_NONE) continue;
        for (int q = 0; q < 4; ++q) { const int32_t t = ptouch[p * 4 + q]; if (t >= 0) res[t] = RES_NONE; }
      }
      // ---- R7 ----
      const int any = __syncthreads_or(changed);
      quiet = any ? 0 : quiet + 1;
      round += 1;
      if (A.digests) {  // the oracle's McRounds::digest
        if (tid == 0) red[1] = 0;
        __syncthreads();
        uint64_t acc = 0;
        auto enc = [&](int32_t p, uint64_t side) -> uint64_t {
          return p == kNone ? 0 : p >= 0 ? 1 + (uint64_t)p : side + ((uint64_t)dk(p) << 20) + (uint64_t)di(p);
        };
        for (int p = tid; p < ns; p += kT) {
          const int s = st(p);
          acc += dig(4ull * p, (uint64_t)s) + dig(4ull * p + 1, enc(up[p], 1ull << 40)) +
                 dig(4ull * p + 2, enc(down[p], 1ull << 41)) + dig(4ull * p + 3, s == ST_FREE ? 0 : (uint64_t)tag[p] + 1);
        }
        const uint64_t b1 = 4ull * ns, b2 = b1 + (uint64_t)K * Mmax, b3 = b2 + (uint64_t)K * Mmax, b4 = b3 + 2ull * Sn;
        for (int q = tid; q < K * Mmax; q += kT) {
          acc += dig(b1 + q, sd[q] == kNone ? 0 : 1 + (uint64_t)sd[q]);
          acc += dig(b2 + q, su[q] == kNone ? 0 : 1 + (uint64_t)su[q]);
        }
        for (int v = tid; v < Sn; v += kT) acc += dig(b3 + 2ull * v, (uint64_t)(uint32_t)kacc[v]) + dig(b3 + 2ull * v + 1, (uint64_t)(uint32_t)deny[v]);
        if (tid == 0) acc += dig(b4, (uint64_t)(uint32_t)quiet);
        atomicAdd(&red[1], (unsigned long long)acc);
        __syncthreads();
        if (tid == 0) A.digests[(size_t)b * A.max_rounds + r] = red[1];
        __syncthreads();
      }
      ++r;
      if (quiet >= A.W) break;
    }
    if (A.digests) for (int k = r + tid; k < A.max_rounds; k += kT) A.digests[(size_t)b * A.max_rounds + k] = 0;
    // ---- results: complete SRC_k -> SNK_k chains per data node, dangling outflows ----
    for (int k = 0; k < K; ++k) {
      if (tid == 0) { red[2] = 0; red[3] = 0; }
      __syncthreads();
      unsigned long long f = 0, c = 0;
      for (int q = tid; q < Mk(k); q += kT) {
        int32_t p = sd[k * Mmax + q];
        if (p == kNone) continue;
        int64_t cc = d(-1 - k, p / MC);
        int guard = 0;
        bool ok = true;
        while (p >= 0 && ++guard <= S + 1) {
          const int32_t nx = down[p];
          if (nx == kNone) { ok = false; break; }
          cc = sadd(cc, d(p / MC, nx <= -2 ? -1 - dk(nx) : nx / MC));
          p = nx;
        }
        if (ok && p <= -2 && dk(p) == k && cc != INF) { f += 1; c += (unsigned long long)cc; }
      }
      atomicAdd(&red[2], f);
      atomicAdd(&red[3], c);
      __syncthreads();
      if (tid == 0) { A.F_dec[(size_t)k * A.B + b] = (int64_t)red[2]; A.cost_dec[(size_t)k * A.B + b] = (int64_t)red[3]; }
      __syncthreads();
    }
    if (tid == 0) red[4] = 0;
    __syncthreads();
    int dg = 0;
    for (int p = tid; p < ns; p += kT) dg += st(p) == ST_OUT;
    atomicAdd(&red[4], (unsigned long long)dg);
    if (A.up_out) for (int p = tid; p < ns; p += kT) {
      A.up_out[(size_t)b * ns + p] = up[p];
      A.down_out[(size_t)b * ns + p] = down[p];
      A.tag_out[(size_t)b * ns + p] = st(p) == ST_FREE ? -1 : tag[p];
    }
    if (A.sd_out) for (int k = tid; k < K * Mmax; k += kT) {
      A.sd_out[(size_t)b * K * Mmax + k] = sd[k];
      A.su_out[(size_t)b * K * Mmax + k] = su[k];
    }
    __syncthreads();
    if (tid == 0) { A.rounds_run[b] = r; A.dangling[b] = (int32_t)red[4]; }
    __syncthreads();
  }
}

}  // namespace

size_t mc_rounds_smem(int S, int n, int MC, int K, int Mmax) { return mc_layout(S, n, MC, K, Mmax).total; }

cudaError_t launch_mc_rounds(const McRoundsCall& c, cudaStream_t st, int num_sms) {
  McArgs A{};
  A.B = c.B; A.S = c.S; A.n = c.n; A.MC = c.MC; A.K = c.K; A.Mmax = c.Mmax;
  A.cap = c.cap; A.alive = c.alive; A.tile = c.tile; A.ld = c.ld; A.src = c.src; A.snk = c.snk; A.supply = c.supply;
  A.seed = c.seed; A.inst_base = c.inst_base; A.objective = c.objective; A.W = c.W; A.deny_after = c.deny_after;
  A.max_rounds = c.max_rounds; A.thr = c.thr; A.thr_width = c.thr_width; A.thr_K = c.thr_K;
  A.rounds_run = c.rounds_run; A.F_dec = c.F_dec; A.cost_dec = c.cost_dec; A.dangling = c.dangling;
  A.digests = c.digests; A.up_out = c.up_out; A.down_out = c.down_out; A.tag_out = c.tag_out;
  A.sd_out = c.sd_out; A.su_out = c.su_out; A.resume = c.resume; A.round0 = c.round0;
  const size_t smem = mc_layout(c.S, c.n, c.MC, c.K, c.Mmax).total;
  cudaError_t e = cudaFuncSetAttribute(mc_rounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mc_rounds_kernel, kT, smem);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<long long>(c.B, (long long)std::max(per_sm, 1) * num_sms);
  mc_rounds_kernel<<<std::max(grid, 1), kT, smem, st>>>(A);
  return cudaGetLastError();
}

}  // namespace gwtf
