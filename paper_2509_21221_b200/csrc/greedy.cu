// SWARM-style greedy routing baseline.  PAPER.md:111-113: SWARM "nodes employ
// a greedy procedure to select their next stage successor"; SPEC.md:199-207 greedy_route: "the
// alive next-stage node with minimum edge_cost(from, .), ties -> lowest NodeId".
//
// Reading: microbatches are routed one at a time from the data node D through
// stages 0..S-1 and back to D, each hop to the alive successor with spare capacity and a link,
// minimum cost first, lowest index on ties; a microbatch that finds no successor (or no sink
// arc) is not routed and releases what it reserved -- every later one would retrace it, so
// routing stops there.  One warp per instance: a hop is a warp-wide arg-min over the n
// candidates ((cost << 32 | index) keys, shuffle reduction).
#include <cuda_runtime.h>
#include <stdint.h>

#include "gwtf_internal.h"

namespace gwtf {

namespace {

constexpr int kWarps = 4;  // instances per CTA

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t x) {
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, x, off);
    x = y < x ? y : x;
  }
  return x;
}

__global__ void __launch_bounds__(32 * kWarps) greedy_kernel(const Problem P, int32_t* __restrict__ rem_all,
                                                              int64_t* __restrict__ F_out, int64_t* __restrict__ cost_out) {
  __shared__ int32_t path_sm[kWarps][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int S = P.S, n = P.n, ld = P.ld;
  int32_t* path = path_sm[w];
  for (int b = blockIdx.x * kWarps + w; b < P.B; b += gridDim.x * kWarps) {
    int32_t* rem = rem_all + (size_t)b * S * n;
    const int32_t* tile = P.tile + (size_t)b * (S - 1) * n * ld;
    const int32_t* src = P.src + (size_t)b * n;
    const int32_t* snk = P.snk + (size_t)b * n;
    for (int k = lane; k < S * n; k += 32)
      rem[k] = P.alive[(size_t)b * S * n + k] ? P.cap[(size_t)b * S * n + k] : 0;
    __syncwarp();
    const int64_t M = P.supply[b];
    int64_t F = 0, cost = 0;
    for (; F < M; ++F) {
      int64_t c = 0;
      int u = -1, s = 0;
      bool ok = true;
      for (; s < S; ++s) {
        uint64_t best = ~0ull;
        for (int v = lane; v < n; v += 32) {
          const int32_t d = s == 0 ? src[v] : tile[((size_t)(s - 1) * n + v) * ld + u];
          if (d != kAbsent && rem[s * n + v] > 0) {
            const uint64_t key = ((uint64_t)(uint32_t)d << 32) | (uint32_t)v;
            best = key < best ? key : best;
          }
        }
        best = warp_min_u64(best);
        if (best == ~0ull) { ok = false; break; }
        u = (int)(best & 0xFFFFFFFFu);
        c += (int64_t)(best >> 32);
        if (lane == 0) { rem[s * n + u] -= 1; path[s] = u; }
        __syncwarp();
      }
      if (ok && snk[u] == kAbsent) ok = false;
      if (!ok) {  // release the reservations of this microbatch and stop
        for (int t = lane; t < s; t += 32) rem[t * n + path[t]] += 1;
        __syncwarp();
        break;
      }
      cost += c + snk[u];
    }
    if (lane == 0) { F_out[b] = F; cost_out[b] = cost; }
  }
}

}  // namespace

cudaError_t launch_greedy(const Problem& P, int32_t* rem, int64_t* F, int64_t* cost, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((P.B + kWarps - 1) / kWarps, 148 * 16);
  greedy_kernel<<<grid, 32 * kWarps, 0, st>>>(P, rem, F, cost);
  return cudaGetLastError();
}

}  // namespace gwtf
