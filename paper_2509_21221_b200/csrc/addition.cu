// Batched node-addition optimizer: the S! placements of S joining
// candidates, one per stage, each solved by the exact min-cost max-flow ("the
// optimal choice of node addition is determined by running the minimum cost flow algorithm for
// each combination of S candidate nodes added to each of the S stages").
//
//   addition_build_kernel: one block per placement p = first + b (grid-stride); the
//     permutation is decoded from p in the factorial number system (lexicographic order), the
//     candidate perm[s] joins stage s as client n of an (n+1)-client instance.
//   addition_select_kernel: block-wide arg-best over the placements: max F, then min cost, then
//     lowest index (lexicographically first assignment).
#include <cuda_runtime.h>
#include <stdint.h>

#include "gwtf_internal.h"

namespace gwtf {

namespace {

// permutation p (lexicographic rank) of {0..S-1}: perm[s] = candidate placed in stage s
__device__ __forceinline__ void decode_perm(int64_t p, int S, int8_t* perm) {
  int64_t fact[21];
  fact[0] = 1;
  for (int i = 1; i <= S; ++i) fact[i] = fact[i - 1] * i;
  uint32_t used = 0;
  for (int s = 0; s < S; ++s) {
    const int64_t f = fact[S - 1 - s];
    int d = (int)(p / f);
    p -= (int64_t)d * f;
    int c = 0;
    for (;; ++c) {  // the d-th unused candidate
      if (used & (1u << c)) continue;
      if (d == 0) break;
      --d;
    }
    used |= 1u << c;
    perm[s] = (int8_t)c;
  }
}

__global__ void addition_build_kernel(int32_t S, int32_t n, const int32_t* __restrict__ cap,
                                      const int32_t* __restrict__ src, const int32_t* __restrict__ snk,
                                      const int32_t* __restrict__ link, const int32_t* __restrict__ ccap,
                                      const int32_t* __restrict__ cin, const int32_t* __restrict__ cout,
                                      const int32_t* __restrict__ ccc, int64_t first, int64_t count,
                                      int32_t* __restrict__ cap_o, int32_t* __restrict__ src_o,
                                      int32_t* __restrict__ snk_o, int32_t* __restrict__ link_o) {
  __shared__ int8_t perm[20];
  const int n1 = n + 1;
  const int per_link = (S - 1) * n1 * n1;
  for (int64_t b = blockIdx.x; b < count; b += gridDim.x) {  // one block per placement
    __syncthreads();
    if (threadIdx.x == 0) decode_perm(first + b, S, perm);
    __syncthreads();
    for (int e = threadIdx.x; e < S * n1; e += blockDim.x) {  // capacities
      const int s = e / n1, i = e - s * n1;
      cap_o[b * S * n1 + e] = i < n ? cap[s * n + i] : ccap[perm[s]];
    }
    for (int e = threadIdx.x; e < n1; e += blockDim.x) {  // D -> stage 0, stage S-1 -> D
      src_o[b * n1 + e] = e < n ? src[e] : cin[((size_t)perm[0] * S + 0) * n];
      snk_o[b * n1 + e] = e < n ? snk[e] : cout[((size_t)perm[S - 1] * S + (S - 1)) * n];
    }
    for (int e = threadIdx.x; e < per_link; e += blockDim.x) {  // link[s][v][u] = d((s,u) -> (s+1,v))
      const int s = e / (n1 * n1), rem = e - s * n1 * n1, v = rem / n1, u = rem - v * n1;
      int32_t c;
      if (u < n && v < n) c = link[((size_t)s * n + v) * n + u];
      else if (u == n && v < n) c = cout[((size_t)perm[s] * S + s) * n + v];        // candidate@s -> (s+1,v)
      else if (u < n && v == n) c = cin[((size_t)perm[s + 1] * S + (s + 1)) * n + u];  // (s,u) -> candidate@s+1
      else c = ccc[perm[s] * S + perm[s + 1]];                                          // candidate -> candidate
      link_o[(size_t)b * per_link + e] = c;
    }
  }
}

__global__ void addition_select_kernel(int64_t count, const int64_t* __restrict__ F, const int64_t* __restrict__ cost,
                                       int64_t* __restrict__ best) {
  __shared__ int64_t sF[1024], sC[1024], sI[1024];
  int64_t bF = -1, bC = 0, bI = -1;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    const int64_t f = F[i], c = cost[i];
    if (f > bF || (f == bF && c < bC)) { bF = f; bC = c; bI = i; }  // i ascending: ties keep the lowest
  }
  sF[threadIdx.x] = bF; sC[threadIdx.x] = bC; sI[threadIdx.x] = bI;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const int o = threadIdx.x + w;
      const bool better = sF[o] > sF[threadIdx.x] ||
                          (sF[o] == sF[threadIdx.x] && (sC[o] < sC[threadIdx.x] ||
                                                        (sC[o] == sC[threadIdx.x] && sI[o] >= 0 && sI[o] < sI[threadIdx.x])));
      if (sI[o] >= 0 && (sI[threadIdx.x] < 0 || better)) { sF[threadIdx.x] = sF[o]; sC[threadIdx.x] = sC[o]; sI[threadIdx.x] = sI[o]; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) best[0] = sI[0];
}

}  // namespace

cudaError_t launch_addition_build(int32_t S, int32_t n, const int32_t* cap, const int32_t* src, const int32_t* snk,
                                  const int32_t* link, const int32_t* ccap, const int32_t* cin, const int32_t* cout,
                                  const int32_t* ccc, int64_t first, int64_t count, int32_t* cap_o, int32_t* src_o,
                                  int32_t* snk_o, int32_t* link_o, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>(count, 148 * 16);
  if (count > 0)
    addition_build_kernel<<<grid, 256, 0, st>>>(S, n, cap, src, snk, link, ccap, cin, cout, ccc, first, count, cap_o,
                                                 src_o, snk_o, link_o);
  return cudaGetLastError();
}

cudaError_t launch_addition_select(int64_t count, const int64_t* F, const int64_t* cost, int64_t* best, cudaStream_t st) {
  addition_select_kernel<<<1, 1024, 0, st>>>(count, F, cost, best);
  return cudaGetLastError();
}

}  // namespace gwtf
