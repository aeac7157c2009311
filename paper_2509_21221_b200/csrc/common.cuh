// Device helpers shared by the sm_100a kernels: team synchronisation, TMA bulk copies
// through an mbarrier, packed (cost, hops) keys.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gwtf_internal.h"

namespace gwtf {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// A team = TPI consecutive threads of a CTA working on one instance.  TPI == 32 uses warp
// primitives; larger teams use named barrier (team index + 1; barrier 0 is __syncthreads).
template <int TPI>
struct Team {
  int tid;   // thread index inside the team
  int id;    // team index inside the CTA
  __device__ __forceinline__ void sync() const {
    if constexpr (TPI == 32) {
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(TPI) : "memory");
    }
  }
  // barrier + OR of a predicate over the team
  __device__ __forceinline__ int sync_or(int p) const {
    if constexpr (TPI == 32) {
      __syncwarp();
      return __any_sync(0xffffffffu, p);
    } else {
      uint32_t r;
      asm volatile(
          "{\n\t.reg .pred q, o;\n\t"
          "setp.ne.u32 q, %1, 0;\n\t"
          "bar.red.or.pred o, %2, %3, q;\n\t"
          "selp.u32 %0, 1, 0, o;\n\t}"
          : "=r"(r)
          : "r"(p), "r"(id + 1), "r"(TPI)
          : "memory");
      return (int)r;
    }
  }
};

// ---- TMA (bulk async copy engine) global -> shared through an mbarrier -------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- distributed shared memory (thread-block clusters) ----------------------------------
// shared::cluster address of `local_ptr`'s counterpart in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t dsmem_addr(const void* local_ptr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local_ptr)), "r"(rank));
  return r;
}
__device__ __forceinline__ uint64_t dsmem_ld_u64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}
// 64-bit unsigned atomic min on another CTA's shared memory.  A plain atomicMin on a
// map_shared_rank() pointer (and atom.shared::cluster.min.u64) compiles to a generic 64-bit
// ATOM with a CAS-loop fallback that loses updates across SMs on sm_100a (measured: a
// 16-CTA min returned 998 instead of 985); the CAS itself is a native remote operation.
__device__ __forceinline__ uint64_t dsmem_atomic_min_u64(uint32_t addr, uint64_t v) {
  uint64_t cur = dsmem_ld_u64(addr);
  while (v < cur) {
    uint64_t prev;
    asm volatile("atom.shared::cluster.cas.b64 %0, [%1], %2, %3;" : "=l"(prev) : "r"(addr), "l"(cur), "l"(v) : "memory");
    if (prev == cur) return cur;
    cur = prev;
  }
  return cur;
}

// ---- packed lexicographic keys: key = cost << 20 | hops -------------
__device__ __forceinline__ uint64_t key_fwd(uint64_t k, int32_t c) {  // k + (c, 1)
  return k + ((uint64_t)(uint32_t)c << kHopBits) + 1ull;
}
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int off, int width) {
  return __shfl_xor_sync(0xffffffffu, v, off, width);
}

}  // namespace gwtf
