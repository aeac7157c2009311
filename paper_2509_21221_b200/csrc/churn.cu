// Churn masking in place, Eq. 1 cost tiles, tile padding,
// validation scans and the dense export of the canonical assignment.
#include "common.cuh"

namespace gwtf {

namespace {

__device__ __forceinline__ size_t gtid() { return blockIdx.x * (size_t)blockDim.x + threadIdx.x; }
__device__ __forceinline__ size_t gstride() { return (size_t)gridDim.x * blockDim.x; }

int grid_for(size_t work) {
  size_t g = (work + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

// dense [B][S-1][n][n] -> padded [B][S-1][n][ld] (pad = absent)
__global__ void pad_tiles_kernel(const Problem P, const int32_t* __restrict__ link) {
  const size_t rows = (size_t)P.B * (P.S - 1) * P.n;
  const size_t total = rows * P.ld;
  for (size_t t = gtid(); t < total; t += gstride()) {
    const size_t row = t / P.ld;
    const int c = (int)(t % P.ld);
    P.tile[t] = c < P.n ? link[row * P.n + c] : kAbsent;
  }
}

// 16-bit copy of the padded tiles for the cluster tier's streamed relaxation (half the HBM bytes);
// absent arcs and padding carry the clamp value t16code, so the kernel needs no per-weight clamp
__global__ void pack_tile16_kernel(const Problem P) {
  const size_t rows = (size_t)P.B * (P.S - 1) * P.n;
  const size_t total = rows * P.ld16;
  for (size_t t = gtid(); t < total; t += gstride()) {
    const size_t row = t / P.ld16;
    const int c = (int)(t % P.ld16);
    const int32_t v = c < P.n ? P.tile[row * P.ld + c] : kAbsent;
    P.tile16[t] = v == kAbsent || v >= P.t16code ? (uint16_t)P.t16code : (uint16_t)v;
  }
}

// 16-bit copy of the padded tiles for the shared-memory tier (half the shared memory per instance:
// more instances resident per SM): absent links 0xFFFF, padding columns 0 (their keys are INF); valid
// only when every finite cost is < 65535 (bit 0 of bad otherwise)
__global__ void pack_tile16s_kernel(const Problem P, int32_t* bad) {
  const size_t per = (size_t)(P.S - 1) * P.n * P.ld;
  const size_t total = (size_t)P.B * per;
  int fail = 0;
  for (size_t t = gtid(); t < total; t += gstride()) {
    const size_t b = t / per, r = t - b * per;
    const int c = (int)(r % P.ld);
    const int32_t v = P.tile[t];
    uint16_t o = 0;
    if (c < P.n) {
      if (v == kAbsent) o = 0xFFFFu;
      else if (v >= 65535) fail = 1;
      else o = (uint16_t)v;
    }
    P.tile16s[b * (size_t)P.tile16s_stride + r] = o;
  }
  if (fail) atomicOr(bad, 1);
}

// the shared-memory tier's 8-bit copy (a quarter of the shared memory of the int32 tiles): absent
// links 0xFF, padding 0; valid only when every finite cost is < 255 (bit 0 of bad otherwise)
__global__ void pack_tile8s_kernel(const Problem P, int32_t* bad) {
  const size_t per = (size_t)(P.S - 1) * P.n * P.ld;
  const size_t total = (size_t)P.B * per;
  int fail = 0;
  for (size_t t = gtid(); t < total; t += gstride()) {
    const size_t b = t / per, r = t - b * per;
    const int c = (int)(r % P.ld);
    const int32_t v = P.tile[t];
    uint8_t o = 0;
    if (c < P.n) {
      if (v == kAbsent) o = 0xFFu;
      else if (v >= 255) fail = 1;
      else o = (uint8_t)v;
    }
    P.tile8s[b * (size_t)P.tile8s_stride + r] = o;
  }
  if (fail) atomicOr(bad, 1);
}

// 8-bit copy of the padded tiles (the cluster tier streams a quarter of the int32 bytes): valid
// only when every arc within n is present with a cost < 255 (bit 0 of bad otherwise); padding = 255
__global__ void pack_tile8_kernel(const Problem P, int32_t* bad) {
  const size_t rows = (size_t)P.B * (P.S - 1) * P.n;
  const size_t total = rows * P.ld8;
  int fail = 0;
  for (size_t t = gtid(); t < total; t += gstride()) {
    const size_t row = t / P.ld8;
    const int c = (int)(t % P.ld8);
    const int32_t v = c < P.n ? P.tile[row * P.ld + c] : 255;
    if (c < P.n && (v == kAbsent || v >= 255)) fail = 1;
    const uint8_t b8 = (uint8_t)(v == kAbsent || v >= 255 ? 255 : v);
    P.tile8[t] = b8;
    if (c < P.n) {  // source-major copy: row u = column u of the dest-major tile
      const size_t bs = row / P.n, dst = row % P.n;
      P.tile8t[(bs * P.n + c) * P.ld8 + dst] = b8;
    }
  }
  if (fail) atomicOr(bad, 1);
}

// max finite value and min value of an int32 array (validation of costs / capacities)
__global__ void scan_kernel(const int32_t* __restrict__ v, int64_t count, int32_t* out_max, int32_t* out_min) {
  int mx = INT_MIN, mn = INT_MAX;
  for (size_t t = gtid(); t < (size_t)count; t += gstride()) {
    const int x = v[t];
    if (x != kAbsent && x > mx) mx = x;
    if (x < mn) mn = x;
  }
  for (int off = 16; off > 0; off >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  }
  if ((threadIdx.x & 31) == 0) { atomicMax(out_max, mx); atomicMin(out_min, mn); }
}

__global__ void edge_update_kernel(const Problem P, const int32_t* __restrict__ upd, int64_t k, int32_t* bad) {
  for (size_t e = gtid(); e < (size_t)k; e += gstride()) {
    const int32_t* u = upd + 5 * e;
    const int b = u[0], s = u[1], v = u[2], w = u[3], c = u[4];
    const bool cost_ok = c == kAbsent || (c >= 0 && c < (1 << 30));
    if (b < 0 || b >= P.B || !cost_ok) { atomicOr(bad, 1); continue; }
    if (c != kAbsent) {
      // the bounds gwtf_flow_create enforces: a simple residual path's cost must
      // fit the 64-bit key's 42-bit cost field, and M of them an int64 total; such an update is
      // rejected (not applied), bit 4
      const uint64_t path = (uint64_t)(2 * P.S * P.n + 2) * (uint64_t)c;  // < 2^61
      if (path >= (1ull << 42) || (P.Mmax > 0 && path > ((1ull << 62) - 1) / (uint64_t)P.Mmax)) {
        atomicOr(bad, 4);
        continue;
      }
    }
    if (c != kAbsent) atomicMax(&P.counters[6], c);  // weight bound of the cluster tier's 32-bit keys
    if (s == -1) {
      if (v < 0 || v >= P.n) { atomicOr(bad, 1); continue; }
      P.src[(size_t)b * P.n + v] = c;
    } else if (s == P.S - 1) {
      if (w < 0 || w >= P.n) { atomicOr(bad, 1); continue; }
      P.snk[(size_t)b * P.n + w] = c;
    } else if (s >= 0 && s < P.S - 1 && v >= 0 && v < P.n && w >= 0 && w < P.n) {
      P.tile[(((size_t)b * (P.S - 1) + s) * P.n + v) * P.ld + w] = c;
      if (P.tile8) {  // the 8-bit copy: an absent link or a cost >= 255 retires it (bit 8)
        if (c == kAbsent || c >= 255) atomicOr(bad, 8);
        P.tile8[(((size_t)b * (P.S - 1) + s) * P.n + v) * P.ld8 + w] = (uint8_t)(c == kAbsent || c >= 255 ? 255 : c);
        P.tile8t[(((size_t)b * (P.S - 1) + s) * P.n + w) * P.ld8 + v] = (uint8_t)(c == kAbsent || c >= 255 ? 255 : c);
      }
      if (P.tile8s) {  // the shared-memory tier's 8-bit copy (absent: 0xFF); a cost >= 255 retires it (bit 32)
        if (c != kAbsent && c >= 255) atomicOr(bad, 32);
        else P.tile8s[(size_t)b * P.tile8s_stride + ((size_t)s * P.n + v) * P.ld + w] = c == kAbsent ? (uint8_t)0xFFu : (uint8_t)c;
      }
      if (P.tile16s) {  // the shared-memory tier's 16-bit copy (absent: 0xFFFF); a cost >= 65535 retires it (bit 16)
        if (c != kAbsent && c >= 65535) atomicOr(bad, 16);
        else P.tile16s[(size_t)b * P.tile16s_stride + ((size_t)s * P.n + v) * P.ld + w] = c == kAbsent ? (uint16_t)0xFFFFu : (uint16_t)c;
      }
      if (P.tile16) {  // the cluster tier's 16-bit copy; a finite cost >= t16code retires it (bit 2)
        if (c != kAbsent && c >= P.t16code) atomicOr(bad, 2);
        P.tile16[(((size_t)b * (P.S - 1) + s) * P.n + v) * P.ld16 + w] =
            c == kAbsent || c >= P.t16code ? (uint16_t)P.t16code : (uint16_t)c;
      }
    } else {
      atomicOr(bad, 1);
    }
  }
}

__device__ __forceinline__ int32_t cost_between(const Problem& P, int b, int a, int c) {
  // a = -1 data node (SRC side) / relay gid; c = -1 data node (SNK side) / relay gid
  const int n = P.n;
  if (a < 0) return (c >= 0 && c < n) ? P.src[(size_t)b * n + c] : kAbsent;
  if (c < 0) return (a / n == P.S - 1) ? P.snk[(size_t)b * n + a % n] : kAbsent;
  const int sa = a / n;
  if (c / n != sa + 1) return kAbsent;
  return P.tile[(((size_t)b * (P.S - 1) + sa) * n + c % n) * P.ld + a % n];
}

__device__ __forceinline__ bool slot_gone(const Problem& P, int b, int32_t p) {
  // a relay-slot pointer whose relay is dead (or slot beyond its effective capacity)
  if (p < 0) return false;
  const int v = p / P.MC, j = p % P.MC;
  const size_t o = (size_t)b * P.S * P.n + v;
  return !P.alive[o] || j >= P.cap[o];
}

// Clear every round-state pointer into a crashed relay or across an absent link; reset the
// per-relay counters.  Order-independent: each slot only clears its own fields.
__global__ void churn_state_kernel(const Problem P) {
  const int Sn = P.S * P.n, MC = P.MC;
  const size_t nslot = (size_t)P.B * Sn * MC;
  for (size_t t = gtid(); t < nslot; t += gstride()) {
    const int b = (int)(t / ((size_t)Sn * MC));
    const int p = (int)(t % ((size_t)Sn * MC));
    const int v = p / MC, j = p % MC;
    const size_t o = (size_t)b * Sn + v;
    const bool usable = P.alive[o] && j < P.cap[o];
    int32_t u = P.up[t], d = P.down[t];
    if (!usable) {
      u = kNone;
      d = kNone;
    } else {
      if (u != kNone) {
        const int a = u >= 0 ? u / MC : -1;
        if (slot_gone(P, b, u) || cost_between(P, b, a, v) == kAbsent) u = kNone;
      }
      if (d != kNone) {
        const int c = d >= 0 ? d / MC : -1;
        if (slot_gone(P, b, d) || cost_between(P, b, v, c) == kAbsent) d = kNone;
      }
    }
    P.up[t] = u;
    P.down[t] = d;
  }
  const size_t nm = (size_t)P.B * P.Mmax;
  for (size_t t = gtid(); t < nm; t += gstride()) {
    const int b = (int)(t / P.Mmax);
    const int32_t sd = P.src_down[t];
    if (sd != kNone && (slot_gone(P, b, sd) || cost_between(P, b, -1, sd / MC) == kAbsent)) P.src_down[t] = kNone;
    const int32_t su = P.snk_up[t];
    if (su != kNone && (slot_gone(P, b, su) || cost_between(P, b, su / MC, -1) == kAbsent)) P.snk_up[t] = kNone;
  }
  for (size_t t = gtid(); t < (size_t)P.B * Sn; t += gstride()) { P.kacc[t] = 0; P.deny[t] = 0; }
  for (size_t t = gtid(); t < (size_t)P.B; t += gstride()) P.quiet[t] = 0;
}

// Validation of an imported round state (gwtf_flow_import_round_state): every
// pointer of a usable slot is answered by its target (pairing bijectivity), crosses
// exactly one stage boundary or reaches the data node at the ends, data-node slots stay below
// the instance's supply, unusable slots (dead relay, j >= cap) hold nothing.
__global__ void import_check_kernel(const Problem P, int32_t* bad) {
  const int Sn = P.S * P.n, MC = P.MC;
  const int32_t ns = Sn * MC;
  const size_t nslot = (size_t)P.B * ns;
  int fail = 0;
  for (size_t t = gtid(); t < nslot; t += gstride()) {
    const int b = (int)(t / ns);
    const int p = (int)(t % ns);
    const int v = p / MC, j = p % MC, s = v / P.n;
    const size_t o = (size_t)b * Sn + v;
    const int32_t* up = P.up + (size_t)b * ns;
    const int32_t* dn = P.down + (size_t)b * ns;
    const int64_t M = P.supply[b];
    const int32_t u = up[p], d = dn[p];
    if (!(P.alive[o] && j < P.cap[o])) { fail |= u != kNone || d != kNone; continue; }
    if (u >= 0) fail |= u >= ns || u / MC / P.n != s - 1 || dn[u] != p;
    else if (u != kNone) fail |= s != 0 || -2 - u >= M || P.src_down[(size_t)b * P.Mmax - 2 - u] != p;
    if (d >= 0) fail |= d >= ns || d / MC / P.n != s + 1 || up[d] != p;
    else if (d != kNone) fail |= s != P.S - 1 || -2 - d >= M || P.snk_up[(size_t)b * P.Mmax - 2 - d] != p;
  }
  for (size_t t = gtid(); t < (size_t)P.B * P.Mmax; t += gstride()) {
    const int b = (int)(t / P.Mmax);
    const int k = (int)(t % P.Mmax);
    const int32_t sd = P.src_down[t], su = P.snk_up[t];
    if (k >= P.supply[b]) { fail |= sd != kNone || su != kNone; continue; }
    if (sd != kNone) fail |= sd < 0 || sd >= ns || P.up[(size_t)b * ns + sd] != -2 - k;
    if (su != kNone) fail |= su < 0 || su >= ns || P.down[(size_t)b * ns + su] != -2 - k;
  }
  for (size_t t = gtid(); t < (size_t)P.B * Sn; t += gstride()) fail |= P.kacc[t] < 0 || P.deny[t] < 0;
  if (fail) atomicOr(bad, 1);
}

__global__ void dense_arcs_kernel(const Problem P, int32_t* dense) {
  const size_t nb = (size_t)(P.S - 1);
  const size_t total = (size_t)P.B * nb * P.Lcap;
  for (size_t t = gtid(); t < total; t += gstride()) {
    const size_t bs = t / P.Lcap;
    const int e = (int)(t % P.Lcap);
    if (e >= P.arc_cnt[bs]) continue;
    const uint32_t ent = P.arcs[t];
    const int u = (int)(ent >> 20), v = (int)((ent >> 8) & 0xFFFu);
    dense[(bs * P.n + v) * P.n + u] = (int32_t)(ent & 0xFFu);
  }
}

// Eq. 1 in integer half-units:
//   D2(i,j) = c_i + c_j + lam_ij + lam_ji + floor(4 size / (beta_ij + beta_ji)), c_D = 0
__device__ __forceinline__ int32_t eq1_d2(int32_t ci, int32_t cj, int32_t lij, int32_t lji, int32_t bij,
                                          int32_t bji, int64_t size) {
  return (int32_t)((int64_t)ci + cj + lij + lji + (4 * size) / ((int64_t)bij + bji));
}

__global__ void eq1_kernel(int32_t B, int32_t S, int32_t n, int32_t L, const int32_t* __restrict__ comp,
                           const int32_t* __restrict__ loc, const int32_t* __restrict__ dloc,
                           const int32_t* __restrict__ lat, const int32_t* __restrict__ bw, int64_t size,
                           int32_t* src, int32_t* snk, int32_t* link) {
  const size_t per = (size_t)(S - 1) * n * n + 2 * (size_t)n;
  const size_t total = (size_t)B * per;
  for (size_t t = gtid(); t < total; t += gstride()) {
    const size_t b = t / per;
    size_t k = t % per;
    const int32_t* lt = lat + b * L * L;
    const int32_t* bt = bw + b * L * L;
    const int32_t* cp = comp + b * S * n;
    const int32_t* lc = loc + b * S * n;
    const int dl = dloc[b];
    if (k < (size_t)n) {  // D -> (0, i)
      const int i = (int)k, li = lc[i];
      src[b * n + i] = eq1_d2(0, cp[i], lt[dl * L + li], lt[li * L + dl], bt[dl * L + li], bt[li * L + dl], size);
    } else if (k < 2 * (size_t)n) {  // (S-1, i) -> D
      const int i = (int)(k - n), a = (S - 1) * n + i, la = lc[a];
      snk[b * n + i] = eq1_d2(cp[a], 0, lt[la * L + dl], lt[dl * L + la], bt[la * L + dl], bt[dl * L + la], size);
    } else {
      k -= 2 * (size_t)n;
      const int s = (int)(k / ((size_t)n * n)), v = (int)((k / n) % n), u = (int)(k % n);
      const int a = s * n + u, c = (s + 1) * n + v, la = lc[a], lb = lc[c];
      link[b * (size_t)(S - 1) * n * n + k] =
          eq1_d2(cp[a], cp[c], lt[la * L + lb], lt[lb * L + la], bt[la * L + lb], bt[lb * L + la], size);
    }
  }
}

}  // namespace

cudaError_t launch_pad_tiles(const Problem& P, const int32_t* link, cudaStream_t st) {
  const size_t total = (size_t)P.B * (P.S - 1) * P.n * P.ld;
  if (total) pad_tiles_kernel<<<grid_for(total), 256, 0, st>>>(P, link);
  return cudaGetLastError();
}

cudaError_t launch_pack_tile8s(const Problem& P, int32_t* bad, cudaStream_t st) {
  const size_t total = (size_t)P.B * (P.S - 1) * P.n * P.ld;
  if (total && P.tile8s) pack_tile8s_kernel<<<grid_for(total), 256, 0, st>>>(P, bad);
  return cudaGetLastError();
}

cudaError_t launch_pack_tile16s(const Problem& P, int32_t* bad, cudaStream_t st) {
  const size_t total = (size_t)P.B * (P.S - 1) * P.n * P.ld;
  if (total && P.tile16s) pack_tile16s_kernel<<<grid_for(total), 256, 0, st>>>(P, bad);
  return cudaGetLastError();
}

cudaError_t launch_pack_tile16(const Problem& P, cudaStream_t st) {
  const size_t total = (size_t)P.B * (P.S - 1) * P.n * P.ld16;
  if (total && P.tile16) pack_tile16_kernel<<<grid_for(total), 256, 0, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_pack_tile8(const Problem& P, int32_t* bad, cudaStream_t st) {
  const size_t total = (size_t)P.B * (P.S - 1) * P.n * P.ld8;
  if (total && P.tile8) pack_tile8_kernel<<<grid_for(total), 256, 0, st>>>(P, bad);
  return cudaGetLastError();
}

cudaError_t launch_scan_costs(const int32_t* v, int64_t count, int32_t* out_max, int32_t* out_min, cudaStream_t st) {
  if (count > 0) scan_kernel<<<grid_for((size_t)count), 256, 0, st>>>(v, count, out_max, out_min);
  return cudaGetLastError();
}

cudaError_t launch_churn(const Problem& P, const uint8_t* alive_new, const int32_t* upd, int64_t k, int32_t* bad,
                         cudaStream_t st) {
  if (upd && k > 0) edge_update_kernel<<<grid_for((size_t)k), 256, 0, st>>>(P, upd, k, bad);
  {  // the mask before this churn (warm reroute tells rejoined relays from unused ones)
    cudaError_t e = cudaMemcpyAsync(P.alive_prev, P.alive, (size_t)P.B * P.S * P.n, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  if (alive_new) {
    cudaError_t e = cudaMemcpyAsync(P.alive, alive_new, (size_t)P.B * P.S * P.n, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  churn_state_kernel<<<grid_for((size_t)P.B * P.S * P.n * P.MC + P.B * P.Mmax), 256, 0, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_import_check(const Problem& P, int32_t* bad, cudaStream_t st) {
  import_check_kernel<<<grid_for((size_t)P.B * P.S * P.n * P.MC + (size_t)P.B * P.Mmax), 256, 0, st>>>(P, bad);
  return cudaGetLastError();
}

// residual node capacities after the last exact solve: (alive ? cap : 0) - node flow
__global__ void residual_caps_kernel(const Problem P, int32_t* __restrict__ out) {
  const size_t total = (size_t)P.B * P.S * P.n;
  for (size_t t = gtid(); t < total; t += gstride()) out[t] = (P.alive[t] ? P.cap[t] : 0) - P.g[t];
}

cudaError_t launch_residual_caps(const Problem& P, int32_t* out, cudaStream_t st) {
  const size_t total = (size_t)P.B * P.S * P.n;
  if (total) residual_caps_kernel<<<grid_for(total), 256, 0, st>>>(P, out);
  return cudaGetLastError();
}

cudaError_t launch_dense_arcs(const Problem& P, int32_t* dense, cudaStream_t st) {
  const size_t total = (size_t)P.B * (P.S - 1) * P.Lcap;
  if (total) dense_arcs_kernel<<<grid_for(total), 256, 0, st>>>(P, dense);
  return cudaGetLastError();
}

cudaError_t launch_eq1(int32_t B, int32_t S, int32_t n, int32_t L, const int32_t* comp, const int32_t* loc,
                       const int32_t* dloc, const int32_t* lat, const int32_t* bw, int64_t size_kbit, int32_t* src,
                       int32_t* snk, int32_t* link, cudaStream_t st) {
  const size_t total = (size_t)B * ((size_t)(S - 1) * n * n + 2 * (size_t)n);
  if (total) eq1_kernel<<<grid_for(total), 256, 0, st>>>(B, S, n, L, comp, loc, dloc, lat, bw, size_kbit, src, snk, link);
  return cudaGetLastError();
}

}  // namespace gwtf
