// gwtf_api.cpp -- host side of the C-ABI declared in include/gwtf.h: validation, the handle's
// device workspace, the annealing threshold table and kernel orchestration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gwtf.h"
#include "gwtf_internal.h"

namespace gwtf {
size_t ssp_global_ws_bytes(const Problem& P);
}

using namespace gwtf;

namespace {

thread_local std::string g_err;

gwtf_status fail(gwtf_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

struct Timer {
  std::string name;
  cudaEvent_t a, b;
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct gwtf_flow_s {
  Problem P{};
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t flags = 0;
  int num_sms = 148;
  bool poisoned = false;
  bool has_assignment = false;
  std::vector<void*> allocs;
  // snapshot of the mutable state
  std::vector<std::pair<void*, size_t>> mutable_bufs;
  std::vector<void*> snap;
  bool has_snapshot = false;
  // host-pointer mode scratch (device copies of outputs)
  std::vector<DevBuf> scratch;
  // profiling
  bool profiling = false;
  std::vector<Timer> pending;
  std::vector<std::string> names;
  std::vector<float> ms;
  std::vector<int32_t> launches;
  int32_t* bad_flag = nullptr;
  // second stream of gwtf_flow_solve_and_rounds (created on first use)
  cudaStream_t stream2 = nullptr;
  int64_t kernel_launches = 0;  // kernels this handle has launched (gwtf_flow_stats[15])
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace {

bool host_mode(const gwtf_flow_s* h) { return (h->flags & GWTF_HOST_PTRS) != 0; }

gwtf_status cuda_fail(gwtf_flow_s* h, cudaError_t e, const char* where) {
  if (h) h->poisoned = true;
  return fail(GWTF_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(h, expr)                                           \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return cuda_fail((h), _e, #expr);  \
  } while (0)

// Device memory of a handle comes from the library's own stream-ordered pool (one per device,
// cudaMallocFromPoolAsync on the handle's stream): creating and destroying handles back to back (the
// e2e pipeline, node-addition batches, multi-source turns) reuses pool memory instead of paying
// cudaMalloc / cudaFree, whose unmap synchronises the device.  A private pool leaves the device's
// default pool (and other libraries' settings) alone.  It keeps up to kPoolKeep bytes after a
// synchronisation (GWTF_POOL_KEEP_MB overrides): 8 GB, 4% of a B200's HBM, holds one stress handle
// (4.6 GB of tiles, copies and state), so re-creating it maps no new memory (measured: a create +
// destroy pair cost 0.1-0.7 s more with a 1 GB threshold); anything above goes back to the device.
constexpr uint64_t kPoolKeep = 8ull << 30;
void* dev_alloc(gwtf_flow_s* h, size_t bytes) {
  static cudaMemPool_t pools[64] = {};
  static bool tried[64] = {};
  cudaMemPool_t pool = nullptr;
  if (h->device >= 0 && h->device < 64) {
    if (!tried[h->device]) {
      tried[h->device] = true;
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = h->device;
      if (cudaMemPoolCreate(&pools[h->device], &props) == cudaSuccess) {
        uint64_t keep = kPoolKeep;
        if (const char* f = getenv("GWTF_POOL_KEEP_MB")) keep = (uint64_t)strtoull(f, nullptr, 10) << 20;
        cudaMemPoolSetAttribute(pools[h->device], cudaMemPoolAttrReleaseThreshold, &keep);
      } else {
        pools[h->device] = nullptr;
      }
      cudaGetLastError();
    }
    pool = pools[h->device];
  }
  void* q = nullptr;
  const cudaError_t e = pool ? cudaMallocFromPoolAsync(&q, bytes, pool, h->stream) : cudaMallocAsync(&q, bytes, h->stream);
  if (e != cudaSuccess) { cudaGetLastError(); return nullptr; }
  return q;
}
void dev_free(gwtf_flow_s* h, void* p) {
  if (p) cudaFreeAsync(p, h->stream);
}

template <class T>
gwtf_status alloc(gwtf_flow_s* h, T** p, size_t count, bool is_mutable = false) {
  if (count == 0) count = 1;
  void* q = dev_alloc(h, count * sizeof(T));
  if (!q) {
    cudaGetLastError();
    return fail(GWTF_E_NOMEM, "device allocation failed (" + std::to_string(count * sizeof(T)) + " bytes)");
  }
  h->allocs.push_back(q);
  if (is_mutable) h->mutable_bufs.push_back({q, count * sizeof(T)});
  *p = static_cast<T*>(q);
  return GWTF_OK;
}

// device scratch slot i of at least `bytes` (host-pointer mode)
void* scratch(gwtf_flow_s* h, size_t i, size_t bytes) {
  if (h->scratch.size() <= i) h->scratch.resize(i + 1);
  DevBuf& b = h->scratch[i];
  if (b.bytes < bytes) {
    dev_free(h, b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (!(b.p = dev_alloc(h, bytes))) return nullptr;
    b.bytes = bytes;
  }
  return b.p;
}

void prof_begin(gwtf_flow_s* h, const char* name, Timer* t, cudaStream_t st = nullptr) {
  if (!h->profiling) return;
  t->name = name;
  cudaEventCreate(&t->a);
  cudaEventCreate(&t->b);
  cudaEventRecord(t->a, st ? st : h->stream);
}
void prof_end(gwtf_flow_s* h, Timer* t, cudaStream_t st = nullptr) {
  if (!h->profiling) return;
  cudaEventRecord(t->b, st ? st : h->stream);
  h->pending.push_back(*t);
}

// Annealing thresholds thr[k][delta] = min(2^32-1, floor(exp(-delta/(T0 alpha^k)) 2^32))
// ("T reduced after each accepted change by a factor alpha"),
// IEEE double with the host libm, no fast-math.
uint32_t thr_value(double T0, double alpha, int k, int delta) {
  const double T = T0 * std::pow(alpha, (double)k);
  const double v = std::floor(std::exp(-(double)delta / T) * 4294967296.0);
  if (v >= 4294967295.0) return 4294967295u;
  if (v <= 0.0) return 0u;
  return (uint32_t)v;
}

gwtf_status anneal_table(double T0, double alpha, std::vector<uint32_t>& t, int32_t& width, int32_t& K) {
  if (!(T0 > 0.0)) {
    width = 1;
    K = 0;
    t.assign(1, 0);
    return GWTF_OK;
  }
  if (!(alpha > 0.0 && alpha < 1.0)) return fail(GWTF_E_INVALID, "alpha must be in (0,1) when T0 > 0");
  width = 1;
  while (thr_value(T0, alpha, 0, width) != 0)
    if (++width > (1 << 20)) return fail(GWTF_E_INVALID, "T0 too large: annealing table wider than 2^20");
  K = 0;
  while (thr_value(T0, alpha, K, 1) != 0)
    if (++K > (1 << 16)) return fail(GWTF_E_INVALID, "alpha too close to 1: more than 2^16 temperature levels");
  if ((int64_t)(K + 1) * width > (1 << 24)) return fail(GWTF_E_INVALID, "annealing table too large");
  t.assign((size_t)(K + 1) * width, 0);
  for (int k = 0; k <= K; ++k)
    for (int d = 1; d < width; ++d) t[(size_t)k * width + d] = thr_value(T0, alpha, k, d);
  return GWTF_OK;
}

// copy an input array (host or device) to a device buffer on the stream
gwtf_status copy_in(gwtf_flow_s* h, void* dst, const void* src, size_t bytes) {
  CK(h, cudaMemcpyAsync(dst, src, bytes, host_mode(h) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                        h->stream));
  return GWTF_OK;
}

// outputs: in host mode write to device scratch, then copy out after the launch
struct OutMap {
  void* user;
  void* dev;
  size_t bytes;
};

template <class T>
gwtf_status map_out(gwtf_flow_s* h, T* user, size_t count, size_t slot, T** dev, std::vector<OutMap>& maps) {
  if (!user) { *dev = nullptr; return GWTF_OK; }
  if (!host_mode(h)) { *dev = user; return GWTF_OK; }
  void* d = scratch(h, slot, std::max<size_t>(count * sizeof(T), 16));
  if (!d) return fail(GWTF_E_NOMEM, "output scratch allocation failed");
  *dev = static_cast<T*>(d);
  maps.push_back({user, d, count * sizeof(T)});
  return GWTF_OK;
}

gwtf_status finish_out(gwtf_flow_s* h, const std::vector<OutMap>& maps) {
  for (const OutMap& m : maps) CK(h, cudaMemcpyAsync(m.user, m.dev, m.bytes, cudaMemcpyDeviceToHost, h->stream));
  if (host_mode(h)) CK(h, cudaStreamSynchronize(h->stream));
  return GWTF_OK;
}

gwtf_status enter(gwtf_flow_s* h) {
  if (!h) return fail(GWTF_E_INVALID, "NULL handle");
  if (h->poisoned) return fail(GWTF_E_CUDA, "handle poisoned by an earlier CUDA error");
  CK(h, cudaSetDevice(h->device));
  return GWTF_OK;
}

}  // namespace

extern "C" {

const char* gwtf_last_error(void) { return g_err.c_str(); }
int32_t gwtf_abi_version(void) { return GWTF_ABI_VERSION; }

gwtf_status gwtf_eq1_cost_tiles(int32_t B, int32_t S, int32_t n, int32_t L, const int32_t* comp, const int32_t* loc,
                                const int32_t* dloc, const int32_t* lat, const int32_t* bw, int64_t size_kbit,
                                int32_t* src_out, int32_t* snk_out, int32_t* link_out, void* stream) {
  if (B < 1 || S < 1 || n < 1 || L < 1 || size_kbit < 0)
    return fail(GWTF_E_INVALID, "eq1: B, S, n, L must be >= 1 and size >= 0");
  if (!comp || !loc || !dloc || !lat || !bw || !src_out || !snk_out || (S > 1 && !link_out))
    return fail(GWTF_E_INVALID, "eq1: NULL array");
  cudaError_t e = launch_eq1(B, S, n, L, comp, loc, dloc, lat, bw, size_kbit, src_out, snk_out, link_out,
                             (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(GWTF_E_CUDA, std::string("eq1: ") + cudaGetErrorString(e));
  return GWTF_OK;
}

gwtf_status gwtf_addition_build(int32_t S, int32_t n, const int32_t* cap, const int32_t* src_cost,
                                const int32_t* snk_cost, const int32_t* link_cost, const int32_t* cand_cap,
                                const int32_t* cand_in, const int32_t* cand_out, const int32_t* cand_cc,
                                int64_t first, int64_t count, int32_t* cap_out, int32_t* src_out, int32_t* snk_out,
                                int32_t* link_out, void* stream) {
  if (S < 1 || S > 20 || n < 1) return fail(GWTF_E_INVALID, "addition: S must be in 1..20 and n >= 1");
  int64_t fact = 1;
  for (int i = 2; i <= S; ++i) fact *= i;
  if (first < 0 || count < 0 || first + count > fact) return fail(GWTF_E_INVALID, "addition: placements outside [0, S!)");
  if (!cap || !src_cost || !snk_cost || (S > 1 && !link_cost) || !cand_cap || !cand_in || !cand_out || !cand_cc ||
      !cap_out || !src_out || !snk_out || (S > 1 && !link_out))
    return fail(GWTF_E_INVALID, "addition: NULL array");
  cudaError_t e = launch_addition_build(S, n, cap, src_cost, snk_cost, link_cost, cand_cap, cand_in, cand_out, cand_cc,
                                        first, count, cap_out, src_out, snk_out, link_out, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(GWTF_E_CUDA, std::string("addition build: ") + cudaGetErrorString(e));
  return GWTF_OK;
}

gwtf_status gwtf_addition_select(int64_t count, const int64_t* flow_value, const int64_t* total_cost,
                                 int64_t* best_index, void* stream) {
  if (count < 1 || !flow_value || !total_cost || !best_index) return fail(GWTF_E_INVALID, "addition select: count/NULL");
  cudaError_t e = launch_addition_select(count, flow_value, total_cost, best_index, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(GWTF_E_CUDA, std::string("addition select: ") + cudaGetErrorString(e));
  return GWTF_OK;
}

gwtf_status gwtf_flow_create(const gwtf_problem_desc* d, gwtf_flow_t* out) {
  if (!d || !out) return fail(GWTF_E_INVALID, "NULL desc/out");
  *out = nullptr;
  if (d->abi_version != GWTF_ABI_VERSION) return fail(GWTF_E_INVALID, "abi_version mismatch");
  const int64_t B = d->num_instances, S = d->num_stages, n = d->clients_per_stage, MC = d->max_cap;
  if (B < 1 || S < 1 || n < 1) return fail(GWTF_E_INVALID, "num_instances, num_stages, clients_per_stage must be >= 1");
  if (MC < 0 || MC > 32) return fail(GWTF_E_INVALID, "max_cap must be in [0, 32]");
  if (n > 4096) return fail(GWTF_E_UNSUPPORTED, "clients_per_stage > 4096");
  if (S > 64) return fail(GWTF_E_UNSUPPORTED, "num_stages > 64");
  if (S * n >= (1 << 21)) return fail(GWTF_E_UNSUPPORTED, "S*n >= 2^21");
  if (!d->cap || !d->src_cost || !d->snk_cost || !d->supply || (S > 1 && !d->link_cost))
    return fail(GWTF_E_INVALID, "NULL input array");
  if (d->steady_window < 1 || d->deny_after < 1) return fail(GWTF_E_INVALID, "steady_window, deny_after must be >= 1");
  if (d->objective != GWTF_OBJ_SUM && d->objective != GWTF_OBJ_MINIMAX) return fail(GWTF_E_INVALID, "objective");
  std::vector<uint32_t> thr;
  int32_t width = 1, K = 0;
  gwtf_status st = anneal_table(d->T0, d->alpha, thr, width, K);
  if (st != GWTF_OK) return st;

  gwtf_flow_s* h = new gwtf_flow_s();
  h->device = d->device;
  h->stream = (cudaStream_t)d->stream;
  h->flags = d->flags;
  auto bail = [&](gwtf_status s) {
    gwtf_flow_destroy(h);
    return s;
  };
  if (cudaSetDevice(h->device) != cudaSuccess) { cudaGetLastError(); delete h; return fail(GWTF_E_CUDA, "cudaSetDevice"); }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  Problem& P = h->P;
  P.B = (int32_t)B; P.S = (int32_t)S; P.n = (int32_t)n; P.MC = (int32_t)MC;
  P.ld = (int32_t)((n + 3) / 4 * 4);
  const size_t Sn = (size_t)S * n, nb = (size_t)(S - 1);

  // supply -> host for validation and Mmax
  std::vector<int64_t> sup(B);
  if (host_mode(h)) std::memcpy(sup.data(), d->supply, B * sizeof(int64_t));
  else if (cudaMemcpy(sup.data(), d->supply, B * sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return bail(fail(GWTF_E_INVALID, "supply is not a readable device pointer"));
  }
  int64_t Mmax = 0;
  for (int64_t v : sup) {
    if (v < 0) return bail(fail(GWTF_E_INVALID, "negative supply"));
    Mmax = std::max(Mmax, v);
  }
  if (Mmax >= (1 << 24)) return bail(fail(GWTF_E_UNSUPPORTED, "supply >= 2^24"));
  P.Mmax = std::max<int64_t>(Mmax, 1);
  P.Lcap = (int32_t)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(Mmax, n * std::max<int64_t>(MC, 1)), n * n));

  gwtf_status s;
#define AL(ptr, cnt, mut) if ((s = alloc(h, &(ptr), (cnt), (mut))) != GWTF_OK) return bail(s)
  AL(P.tile, B * nb * n * P.ld, true);
  AL(P.src, B * n, true);
  AL(P.snk, B * n, true);
  AL(P.cap, B * Sn, false);
  AL(P.alive, B * Sn, true);
  AL(P.alive_prev, B * Sn, true);
  AL(P.supply, B, false);
  AL(P.g, B * Sn, false);
  AL(P.src_f, B * n, false);
  AL(P.snk_f, B * n, false);
  AL(P.arcs, B * nb * P.Lcap, false);
  AL(P.arc_cnt, B * std::max<size_t>(nb, 1), false);
  const size_t nslot = B * Sn * std::max<int64_t>(MC, 1);
  AL(P.up, nslot, true);
  AL(P.down, nslot, true);
  AL(P.src_down, B * P.Mmax, true);
  AL(P.snk_up, B * P.Mmax, true);
  AL(P.kacc, B * Sn, true);
  AL(P.deny, B * Sn, true);
  AL(P.quiet, B, true);
  AL(P.round, B, true);
  AL(P.counters, 8, false);
  AL(P.redo, B, false);
  AL(P.stats, 2048, false);
  AL(h->bad_flag, 4, false);
  uint32_t* thr_d = nullptr;
  AL(thr_d, thr.size(), false);
  int32_t* link_tmp = nullptr;
  if (nb) AL(link_tmp, B * nb * n * n, false);
#undef AL
  P.thr = thr_d;
  P.thr_width = width;
  P.thr_K = K;
  P.seed = d->seed;
  P.inst_base = d->inst_base;
  P.objective = d->objective;
  P.W = d->steady_window;
  P.deny_after = d->deny_after;
#ifdef GWTF_DEV_FLAGS
  // development builds only (make DEV=1): testing switches, some of which (e.g. bit 64, no tile
  // stream) deliberately give wrong results; a product build never reads them
  if (const char* dbg = getenv("GWTF_DEBUG_FLAGS")) P.debug = atoi(dbg);
#endif

  // exact-solve tiers for instances that do not fit in shared memory: the cluster tier (one
  // thread-block cluster per instance, tiles streamed from HBM) when the device can host it,
  // else the global-memory team tier
  const bool big = ssp_smem_bytes(P) > 227 * 1024;
  if (big || (h->flags & GWTF_FORCE_CLUSTER_TIER)) {
    P.cluster_size = ssp_cluster_size(P);
    if (P.cluster_size > 0) {
      P.ws_cluster_slots = (int32_t)std::min<int64_t>(h->num_sms / P.cluster_size, B);
      uint8_t* wc = nullptr;
      if ((s = alloc(h, &wc, (size_t)P.ws_cluster_slots * 2 * (2 * Sn + 4) * 4)) != GWTF_OK) return bail(s);
      P.ws_cluster = wc;
      if ((s = alloc(h, &P.arcw, B * std::max<size_t>(nb, 1) * P.Lcap)) != GWTF_OK) return bail(s);
    } else if (h->flags & GWTF_FORCE_CLUSTER_TIER) {
      return bail(fail(GWTF_E_UNSUPPORTED, "cluster tier unavailable for this shape"));
    }
  }
  if ((big && P.cluster_size == 0) || (h->flags & GWTF_FORCE_GLOBAL_TIER)) {
    P.ws_teams = (int32_t)std::min<int64_t>(h->num_sms, B);
    P.ws_per_team = ssp_global_ws_bytes(P);
    uint8_t* ws = nullptr;
    if ((s = alloc(h, &ws, (size_t)P.ws_teams * P.ws_per_team)) != GWTF_OK) return bail(s);
    P.ws = ws;
  }

  // global scratch of the rounds kernel when an instance does not fit in shared memory
  if (!rounds_use_smem(P)) {
    const int tpi = rounds_tpi(P);
    P.ws_rounds_teams = (int32_t)std::min<int64_t>((int64_t)h->num_sms * std::max(1, 2048 / tpi), B);
    uint8_t* wr = nullptr;
    if ((s = alloc(h, &wr, (size_t)P.ws_rounds_teams * rounds_ws_bytes(P, false))) != GWTF_OK) return bail(s);
    P.ws_rounds = wr;
  }

  // inputs
  if ((s = copy_in(h, P.cap, d->cap, B * Sn * 4)) != GWTF_OK) return bail(s);
  if (d->alive) {
    if ((s = copy_in(h, P.alive, d->alive, B * Sn)) != GWTF_OK) return bail(s);
  } else if (cudaMemsetAsync(P.alive, 1, B * Sn, h->stream) != cudaSuccess) {
    return bail(cuda_fail(h, cudaGetLastError(), "memset alive"));
  }
  if ((s = copy_in(h, P.src, d->src_cost, B * n * 4)) != GWTF_OK) return bail(s);
  if ((s = copy_in(h, P.snk, d->snk_cost, B * n * 4)) != GWTF_OK) return bail(s);
  if ((s = copy_in(h, P.supply, d->supply, B * 8)) != GWTF_OK) return bail(s);
  if (nb) {
    if ((s = copy_in(h, link_tmp, d->link_cost, B * nb * n * n * 4)) != GWTF_OK) return bail(s);
    if (launch_pad_tiles(P, link_tmp, h->stream) != cudaSuccess) return bail(cuda_fail(h, cudaGetLastError(), "pad"));
  }
  if (cudaMemcpyAsync(thr_d, thr.data(), thr.size() * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
    return bail(cuda_fail(h, cudaGetLastError(), "thr upload"));

  // validation scans: costs in [0, 2^30) or absent, caps in [0, max_cap]
  int32_t* mm = h->bad_flag;  // [0] max cost, [1] min cost, [2] max cap, [3] min cap
  const int32_t init[4] = {INT32_MIN, INT32_MAX, INT32_MIN, INT32_MAX};
  CK(h, cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, h->stream));
  CK(h, launch_scan_costs(P.src, B * n, mm + 0, mm + 1, h->stream));
  CK(h, launch_scan_costs(P.snk, B * n, mm + 0, mm + 1, h->stream));
  if (nb) CK(h, launch_scan_costs(link_tmp, B * nb * n * n, mm + 0, mm + 1, h->stream));
  CK(h, launch_scan_costs(P.cap, B * Sn, mm + 2, mm + 3, h->stream));
  int32_t got[4];
  CK(h, cudaMemcpyAsync(got, mm, sizeof(got), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  if (got[1] < 0) return bail(fail(GWTF_E_INVALID, "negative cost"));
  const int64_t maxc = std::max<int32_t>(got[0], 0);
  if (maxc >= (1 << 30)) return bail(fail(GWTF_E_INVALID, "cost >= 2^30 (other than GWTF_ABSENT)"));
  if (got[3] < 0 || got[2] > MC) return bail(fail(GWTF_E_INVALID, "cap outside [0, max_cap]"));
  const long double bound = (long double)(2 * S * n + 2) * (long double)maxc;
  if (bound >= (long double)(1ull << 42)) return bail(fail(GWTF_E_OVERFLOW, "(2Sn+2)*maxcost >= 2^42"));
  if (bound * (long double)Mmax >= (long double)(1ull << 62)) return bail(fail(GWTF_E_OVERFLOW, "(2Sn+2)*maxcost*M >= 2^62"));
  // 32-bit packed keys (cost << H | hops) when the largest arc weight leaves the guard band
  // free: (maxcost << H) + 1 < 2^29 with 2^H > 2Sn+1; else 64-bit keys
  {
    int H = 0;
    while ((1ll << H) <= 2 * S * n + 1) ++H;
    P.hbits = (H < 29 && ((maxc << H) + 1) < (1ll << 29)) ? H : 0;
  }
  if (link_tmp) {
    dev_free(h, link_tmp);
    h->allocs.erase(std::find(h->allocs.begin(), h->allocs.end(), (void*)link_tmp));
  }
  {  // absent code of the 16-bit tiles = the cluster tier's 32-bit key clamp T32 (ssp_cluster.cu)
    int H = 0;
    while ((1ll << H) <= 2 * S * n + 2) ++H;
    const int CB = 32 - H;
    P.t16code = CB >= 4 ? (int32_t)std::min<int64_t>((1ll << (CB - 1)) - 1, 0xFFFF) : 0;
  }
  if (P.cluster_size > 0 && nb && maxc < P.t16code && !getenv("GWTF_NO_TILE16")) {  // 16-bit tile copy streamed by the cluster tier
    P.ld16 = (int32_t)((n + 7) / 8 * 8);
    if ((s = alloc(h, &P.tile16, B * nb * n * P.ld16, true)) != GWTF_OK) return bail(s);
    CK(h, launch_pack_tile16(P, h->stream));
    if (maxc < 255 && !getenv("GWTF_NO_TILE8")) {  // and the 8-bit copy when every arc is present
      P.ld8 = (int32_t)((n + 15) / 16 * 16);
      if ((s = alloc(h, &P.tile8, B * nb * n * P.ld8, true)) != GWTF_OK) return bail(s);
      // + 16 bytes: the frontier step's 32-bit loads may run up to 3 bytes past the last column
      if ((s = alloc(h, &P.tile8t, B * nb * n * P.ld8 + 16, true)) != GWTF_OK) return bail(s);
      CK(h, cudaMemsetAsync(P.tile8t, 255, B * nb * n * P.ld8 + 16, h->stream));  // padding columns
      int32_t bad8 = 0;
      CK(h, cudaMemsetAsync(h->bad_flag, 0, 4, h->stream));
      CK(h, launch_pack_tile8(P, h->bad_flag, h->stream));
      CK(h, cudaMemcpyAsync(&bad8, h->bad_flag, 4, cudaMemcpyDeviceToHost, h->stream));
      CK(h, cudaStreamSynchronize(h->stream));
      if (bad8) P.tile8 = nullptr;  // an absent link: stream the 16-bit copy
    }
  }
  // the shared-memory tier's 16-bit tile copy (half the shared memory per instance) when every
  // finite cost is < 65535
  if (nb && maxc < 65535 && ssp_smem_bytes(P) <= 227 * 1024 && !getenv("GWTF_NO_TILE16S")) {
    P.tile16s_stride = (int64_t)(((size_t)nb * n * P.ld * 2 + 15) / 16 * 16 / 2);
    if ((s = alloc(h, &P.tile16s, B * (size_t)P.tile16s_stride, true)) != GWTF_OK) return bail(s);
    int32_t bad16 = 0;
    CK(h, cudaMemsetAsync(h->bad_flag, 0, 4, h->stream));
    CK(h, launch_pack_tile16s(P, h->bad_flag, h->stream));
    CK(h, cudaMemcpyAsync(&bad16, h->bad_flag, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (bad16) P.tile16s = nullptr;  // a cost >= 65535: the int32 tiles
  }
  // and the 8-bit copy (a quarter of the shared memory) when every finite cost is < 255
  if (P.tile16s && maxc < 255 && !getenv("GWTF_NO_TILE8S")) {
    P.tile8s_stride = (int64_t)(((size_t)nb * n * P.ld + 15) / 16 * 16);
    if ((s = alloc(h, &P.tile8s, B * (size_t)P.tile8s_stride, true)) != GWTF_OK) return bail(s);
    int32_t bad8s = 0;
    CK(h, cudaMemsetAsync(h->bad_flag, 0, 4, h->stream));
    CK(h, launch_pack_tile8s(P, h->bad_flag, h->stream));
    CK(h, cudaMemcpyAsync(&bad8s, h->bad_flag, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (bad8s) P.tile8s = nullptr;
  }
  {  // counters[6]: bound on the largest finite arc weight (raised by apply_churn's edge updates)
    const int32_t mw = (int32_t)maxc;
    CK(h, cudaMemcpyAsync(P.counters + 6, &mw, 4, cudaMemcpyHostToDevice, h->stream));
  }
  CK(h, launch_init_round_state(P, h->stream));
  CK(h, cudaMemcpyAsync(P.alive_prev, P.alive, B * Sn, cudaMemcpyDeviceToDevice, h->stream));
  CK(h, cudaMemsetAsync(P.stats, 0, 2048 * sizeof(unsigned long long), h->stream));
  CK(h, cudaMemsetAsync(P.arc_cnt, 0, B * std::max<size_t>(nb, 1) * 4, h->stream));
  *out = h;
  return GWTF_OK;
}

gwtf_status gwtf_flow_solve_batch(gwtf_flow_t h, int64_t* flow_value, int64_t* total_cost, int32_t* augmentations,
                                  int32_t* inst_status) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!flow_value || !total_cost) return fail(GWTF_E_INVALID, "flow_value/total_cost must not be NULL");
  const size_t B = h->P.B;
  std::vector<OutMap> maps;
  SspOut o{};
  if ((s = map_out(h, flow_value, B, 0, &o.F, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, total_cost, B, 1, &o.cost, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, augmentations, B, 2, &o.A, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, inst_status, B, 3, &o.status, maps)) != GWTF_OK) return s;
  Timer t;
  const int tier = (h->flags & GWTF_FORCE_GLOBAL_TIER) ? 1 : (h->flags & GWTF_FORCE_CLUSTER_TIER) ? 2 : 0;
  const bool cluster = tier != 1 && h->P.cluster_size > 0 && (tier == 2 || ssp_smem_bytes(h->P) > 227 * 1024);
  prof_begin(h, cluster ? "ssp_cluster_kernel" : "ssp_kernel", &t);
  CK(h, launch_ssp(h->P, o, h->stream, h->num_sms, tier));
  h->kernel_launches += ssp_launch_count(h->P, tier);
  prof_end(h, &t);
  h->has_assignment = true;
  return finish_out(h, maps);
}

gwtf_status gwtf_flow_decentralized_rounds(gwtf_flow_t h, int32_t max_rounds, int32_t* rounds_run, int64_t* dec_flow,
                                           int64_t* dec_cost, int32_t* dangling, uint64_t* round_digests) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (max_rounds < 0) return fail(GWTF_E_INVALID, "max_rounds < 0");
  const size_t B = h->P.B;
  std::vector<OutMap> maps;
  RoundsOut o{};
  o.max_rounds = max_rounds;
  if ((s = map_out(h, rounds_run, B, 4, &o.rounds_run, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, dec_flow, B, 5, &o.F_dec, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, dec_cost, B, 6, &o.cost_dec, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, dangling, B, 7, &o.dangling, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, round_digests, B * std::max(max_rounds, 1), 8, &o.digests, maps)) != GWTF_OK) return s;
  Timer t;
  prof_begin(h, "rounds_kernel", &t);
  CK(h, launch_rounds(h->P, o, h->stream, h->num_sms));
  h->kernel_launches += 1;
  prof_end(h, &t);
  return finish_out(h, maps);
}

gwtf_status gwtf_flow_solve_and_rounds(gwtf_flow_t h, int32_t max_rounds, int64_t* flow_value, int64_t* total_cost,
                                       int32_t* augmentations, int32_t* inst_status, int32_t* rounds_run,
                                       int64_t* dec_flow, int64_t* dec_cost, int32_t* dangling) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!flow_value || !total_cost) return fail(GWTF_E_INVALID, "flow_value/total_cost must not be NULL");
  if (max_rounds < 0) return fail(GWTF_E_INVALID, "max_rounds < 0");
  if (!h->stream2) {
    CK(h, cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
    CK(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  }
  const size_t B = h->P.B;
  std::vector<OutMap> maps;
  SspOut so{};
  if ((s = map_out(h, flow_value, B, 0, &so.F, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, total_cost, B, 1, &so.cost, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, augmentations, B, 2, &so.A, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, inst_status, B, 3, &so.status, maps)) != GWTF_OK) return s;
  RoundsOut ro{};
  ro.max_rounds = max_rounds;
  if ((s = map_out(h, rounds_run, B, 4, &ro.rounds_run, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, dec_flow, B, 5, &ro.F_dec, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, dec_cost, B, 6, &ro.cost_dec, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, dangling, B, 7, &ro.dangling, maps)) != GWTF_OK) return s;
  // fork: the rounds (second stream) and the exact solve (handle stream) read the same masked graph
  // and write disjoint state and counters; join before anything else runs on the handle's stream
  CK(h, cudaEventRecord(h->ev_fork, h->stream));
  CK(h, cudaStreamWaitEvent(h->stream2, h->ev_fork, 0));
  Timer tr, ts;
  const int tier = (h->flags & GWTF_FORCE_GLOBAL_TIER) ? 1 : (h->flags & GWTF_FORCE_CLUSTER_TIER) ? 2 : 0;
  const bool cluster = tier != 1 && h->P.cluster_size > 0 && (tier == 2 || ssp_smem_bytes(h->P) > 227 * 1024);
  // beside the cluster tier of the solve (one cluster of ~10 SMs per instance) the rounds' clusters
  // shrink to 2 CTAs: measured on the stress step, clusters of 8 or 4 keep some of the solve's
  // clusters from being co-resident (10.2 / 10.9 s step), clusters of 2 do not (6.9 s; the solve
  // alone takes 6.8 s).  The rounds are launched first (launching the solve first measured 12.4 s).
  Problem PR = h->P;
  if (cluster) PR.rounds_cluster_pref = 2;
  prof_begin(h, "rounds_kernel", &tr, h->stream2);
  CK(h, launch_rounds(PR, ro, h->stream2, h->num_sms));
  h->kernel_launches += 1;
  prof_end(h, &tr, h->stream2);
  prof_begin(h, cluster ? "ssp_cluster_kernel" : "ssp_kernel", &ts);
  CK(h, launch_ssp(h->P, so, h->stream, h->num_sms, tier));
  h->kernel_launches += ssp_launch_count(h->P, tier);
  prof_end(h, &ts);
  CK(h, cudaEventRecord(h->ev_join, h->stream2));
  CK(h, cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  h->has_assignment = true;
  return finish_out(h, maps);
}

gwtf_status gwtf_flow_apply_churn(gwtf_flow_t h, const uint8_t* alive_new, const int32_t* edge_updates, int64_t k) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (k < 0 || (k > 0 && !edge_updates)) return fail(GWTF_E_INVALID, "edge_updates/k");
  const Problem& P = h->P;
  const uint8_t* a = alive_new;
  const int32_t* u = k > 0 ? edge_updates : nullptr;
  if (host_mode(h)) {
    if (alive_new) {
      void* d = scratch(h, 9, (size_t)P.B * P.S * P.n);
      if (!d) return fail(GWTF_E_NOMEM, "scratch");
      CK(h, cudaMemcpyAsync(d, alive_new, (size_t)P.B * P.S * P.n, cudaMemcpyHostToDevice, h->stream));
      a = (const uint8_t*)d;
    }
    if (u) {
      void* d = scratch(h, 10, (size_t)k * 20);
      if (!d) return fail(GWTF_E_NOMEM, "scratch");
      CK(h, cudaMemcpyAsync(d, edge_updates, (size_t)k * 20, cudaMemcpyHostToDevice, h->stream));
      u = (const int32_t*)d;
    }
  }
  CK(h, cudaMemsetAsync(h->bad_flag, 0, 4, h->stream));
  Timer t;
  prof_begin(h, "churn", &t);
  CK(h, launch_churn(P, a, u, k, h->bad_flag, h->stream));
  h->kernel_launches += 1 + (u && k > 0 ? 1 : 0);
  prof_end(h, &t);
  h->has_assignment = false;
  if (u) {
    int32_t bad = 0;
    CK(h, cudaMemcpyAsync(&bad, h->bad_flag, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (bad & 2) h->P.tile16 = nullptr;  // a cost no longer fits 16 bits: stream the int32 tiles
    if (bad & 16) h->P.tile16s = nullptr;  // a cost >= 65535: int32 tiles in shared memory
    if (bad & (16 | 32)) h->P.tile8s = nullptr;  // a cost >= 255: no 8-bit tiles in shared memory
    if (bad & (2 | 8)) h->P.tile8 = nullptr;  // an absent link or a cost >= 255: no 8-bit stream
    if (bad & 1) return fail(GWTF_E_INVALID, "edge update out of range (valid updates were applied)");
    if (bad & 4) return fail(GWTF_E_OVERFLOW, "edge update cost breaks the key bounds (rejected; valid updates were applied)");
  }
  return GWTF_OK;
}

gwtf_status gwtf_flow_get_assignment(gwtf_flow_t h, int32_t* node_flow, int32_t* src_flow, int32_t* snk_flow,
                                     int32_t* arc_flow_dense) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!h->has_assignment) return fail(GWTF_E_STATE, "no solve_batch since create/churn");
  const Problem& P = h->P;
  const size_t Sn = (size_t)P.S * P.n, nb = (size_t)(P.S - 1);
  const cudaMemcpyKind kind = host_mode(h) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (node_flow) CK(h, cudaMemcpyAsync(node_flow, P.g, P.B * Sn * 4, kind, h->stream));
  if (src_flow) CK(h, cudaMemcpyAsync(src_flow, P.src_f, (size_t)P.B * P.n * 4, kind, h->stream));
  if (snk_flow) CK(h, cudaMemcpyAsync(snk_flow, P.snk_f, (size_t)P.B * P.n * 4, kind, h->stream));
  if (arc_flow_dense && nb) {
    const size_t bytes = (size_t)P.B * nb * P.n * P.n * 4;
    int32_t* dst = arc_flow_dense;
    if (host_mode(h)) {
      dst = (int32_t*)scratch(h, 11, bytes);
      if (!dst) return fail(GWTF_E_NOMEM, "scratch");
    }
    CK(h, cudaMemsetAsync(dst, 0, bytes, h->stream));
    CK(h, launch_dense_arcs(P, dst, h->stream));
    if (host_mode(h)) CK(h, cudaMemcpyAsync(arc_flow_dense, dst, bytes, cudaMemcpyDeviceToHost, h->stream));
  }
  if (host_mode(h)) CK(h, cudaStreamSynchronize(h->stream));
  return GWTF_OK;
}

gwtf_status gwtf_flow_residual_caps(gwtf_flow_t h, int32_t* cap_out) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!cap_out) return fail(GWTF_E_INVALID, "residual_caps: NULL output");
  if (!h->has_assignment) return fail(GWTF_E_STATE, "no solve_batch since create/churn");
  const Problem& P = h->P;
  const size_t bytes = (size_t)P.B * P.S * P.n * 4;
  int32_t* dst = cap_out;
  if (host_mode(h)) {
    dst = (int32_t*)scratch(h, 17, bytes);
    if (!dst) return fail(GWTF_E_NOMEM, "scratch");
  }
  CK(h, launch_residual_caps(P, dst, h->stream));
  h->kernel_launches += 1;
  if (host_mode(h)) {
    CK(h, cudaMemcpyAsync(cap_out, dst, bytes, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
  }
  return GWTF_OK;
}

gwtf_status gwtf_flow_export_round_state(gwtf_flow_t h, int32_t* up, int32_t* down, int32_t* src_down,
                                         int32_t* snk_up, int32_t* kacc, int32_t* deny, int32_t* quiet,
                                         int64_t* round) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  const Problem& P = h->P;
  const size_t Sn = (size_t)P.S * P.n;
  const size_t nslot = (size_t)P.B * Sn * P.MC;
  const cudaMemcpyKind kind = host_mode(h) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (up && nslot) CK(h, cudaMemcpyAsync(up, P.up, nslot * 4, kind, h->stream));
  if (down && nslot) CK(h, cudaMemcpyAsync(down, P.down, nslot * 4, kind, h->stream));
  if (src_down) CK(h, cudaMemcpyAsync(src_down, P.src_down, (size_t)P.B * P.Mmax * 4, kind, h->stream));
  if (snk_up) CK(h, cudaMemcpyAsync(snk_up, P.snk_up, (size_t)P.B * P.Mmax * 4, kind, h->stream));
  if (kacc) CK(h, cudaMemcpyAsync(kacc, P.kacc, P.B * Sn * 4, kind, h->stream));
  if (deny) CK(h, cudaMemcpyAsync(deny, P.deny, P.B * Sn * 4, kind, h->stream));
  if (quiet) CK(h, cudaMemcpyAsync(quiet, P.quiet, (size_t)P.B * 4, kind, h->stream));
  if (round) CK(h, cudaMemcpyAsync(round, P.round, (size_t)P.B * 8, kind, h->stream));
  if (host_mode(h)) CK(h, cudaStreamSynchronize(h->stream));
  return GWTF_OK;
}

gwtf_status gwtf_mc_rounds(int32_t B, int32_t S, int32_t n, int32_t max_cap, int32_t K, const int32_t* cap,
                           const uint8_t* alive, const int32_t* link_cost, const int32_t* src_cost,
                           const int32_t* snk_cost, const int64_t* supply, uint64_t seed, int64_t inst_base, double T0,
                           double alpha, int32_t objective, int32_t steady_window, int32_t deny_after,
                           int32_t max_rounds, int32_t* rounds_run, int64_t* dec_flow, int64_t* dec_cost,
                           int32_t* dangling, uint64_t* round_digests, int32_t* up, int32_t* down, int32_t* tag,
                           int32_t* src_down, int32_t* snk_up, int32_t resume, int64_t round0, void* stream) {
  if (B < 1 || S < 1 || n < 1 || K < 1 || max_cap < 0 || max_cap > 32 || max_rounds < 0 || steady_window < 1 ||
      deny_after < 1 || (objective != GWTF_OBJ_SUM && objective != GWTF_OBJ_MINIMAX))
    return fail(GWTF_E_INVALID, "mc_rounds: shape / parameter out of range");
  if (!cap || !src_cost || !snk_cost || !supply || (S > 1 && !link_cost) || !rounds_run || !dec_flow || !dec_cost ||
      !dangling)
    return fail(GWTF_E_INVALID, "mc_rounds: NULL required array");
  if ((up || down || tag || src_down || snk_up) && !(up && down && tag && src_down && snk_up))
    return fail(GWTF_E_INVALID, "mc_rounds: up/down/tag/src_down/snk_up all or none");
  if (resume && !up) return fail(GWTF_E_INVALID, "mc_rounds: resume needs the state arrays");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int64_t> sup((size_t)K * B);
  if (cudaMemcpyAsync(sup.data(), supply, sup.size() * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return fail(GWTF_E_CUDA, "mc_rounds: supply readback");
  int64_t mmax = 1;
  for (int64_t m : sup) {
    if (m < 0 || m > (1 << 20)) return fail(GWTF_E_INVALID, "mc_rounds: supply outside [0, 2^20]");
    mmax = std::max(mmax, m);
  }
  const size_t smem = mc_rounds_smem(S, n, max_cap, K, (int)mmax);
  if (smem > 227 * 1024) return fail(GWTF_E_UNSUPPORTED, "mc_rounds: instance state exceeds shared memory");
  std::vector<uint32_t> thr;
  int32_t width = 1, Kt = 0;
  if (gwtf_status s = anneal_table(T0, alpha, thr, width, Kt); s != GWTF_OK) return s;
  uint32_t* thr_d = nullptr;
  if (cudaMallocAsync(&thr_d, thr.size() * 4, st) != cudaSuccess) return fail(GWTF_E_NOMEM, "mc_rounds: thr");
  cudaMemcpyAsync(thr_d, thr.data(), thr.size() * 4, cudaMemcpyHostToDevice, st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  McRoundsCall c{};
  c.B = B; c.S = S; c.n = n; c.MC = max_cap; c.K = K; c.Mmax = (int32_t)mmax;
  c.cap = cap; c.alive = alive; c.tile = link_cost; c.ld = n; c.src = src_cost; c.snk = snk_cost; c.supply = supply;
  c.seed = seed; c.inst_base = inst_base; c.objective = objective; c.W = steady_window; c.deny_after = deny_after;
  c.max_rounds = max_rounds; c.thr = thr_d; c.thr_width = width; c.thr_K = Kt;
  c.rounds_run = rounds_run; c.F_dec = dec_flow; c.cost_dec = dec_cost; c.dangling = dangling;
  c.digests = round_digests; c.up_out = up; c.down_out = down; c.tag_out = tag;
  c.sd_out = src_down; c.su_out = snk_up; c.resume = resume; c.round0 = round0;
  const cudaError_t e = launch_mc_rounds(c, st, sms);
  cudaFreeAsync(thr_d, st);
  if (e != cudaSuccess) return fail(GWTF_E_CUDA, cudaGetErrorString(e));
  return GWTF_OK;
}

gwtf_status gwtf_flow_import_round_state(gwtf_flow_t h, const int32_t* up, const int32_t* down,
                                         const int32_t* src_down, const int32_t* snk_up, const int32_t* kacc,
                                         const int32_t* deny, const int32_t* quiet, const int64_t* round) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!up || !down || !src_down || !snk_up) return fail(GWTF_E_INVALID, "up/down/src_down/snk_up are required");
  const Problem& P = h->P;
  const size_t Sn = (size_t)P.S * P.n;
  const size_t nslot = (size_t)P.B * Sn * P.MC;
  const cudaMemcpyKind kind = host_mode(h) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  if (nslot) CK(h, cudaMemcpyAsync(P.up, up, nslot * 4, kind, h->stream));
  if (nslot) CK(h, cudaMemcpyAsync(P.down, down, nslot * 4, kind, h->stream));
  if (P.Mmax) CK(h, cudaMemcpyAsync(P.src_down, src_down, (size_t)P.B * P.Mmax * 4, kind, h->stream));
  if (P.Mmax) CK(h, cudaMemcpyAsync(P.snk_up, snk_up, (size_t)P.B * P.Mmax * 4, kind, h->stream));
  if (kacc) CK(h, cudaMemcpyAsync(P.kacc, kacc, P.B * Sn * 4, kind, h->stream));
  else CK(h, cudaMemsetAsync(P.kacc, 0, P.B * Sn * 4, h->stream));
  if (deny) CK(h, cudaMemcpyAsync(P.deny, deny, P.B * Sn * 4, kind, h->stream));
  else CK(h, cudaMemsetAsync(P.deny, 0, P.B * Sn * 4, h->stream));
  if (quiet) CK(h, cudaMemcpyAsync(P.quiet, quiet, (size_t)P.B * 4, kind, h->stream));
  else CK(h, cudaMemsetAsync(P.quiet, 0, (size_t)P.B * 4, h->stream));
  if (round) CK(h, cudaMemcpyAsync(P.round, round, (size_t)P.B * 8, kind, h->stream));
  else CK(h, cudaMemsetAsync(P.round, 0, (size_t)P.B * 8, h->stream));
  CK(h, cudaMemsetAsync(h->bad_flag, 0, 4, h->stream));
  CK(h, launch_import_check(P, h->bad_flag, h->stream));
  h->kernel_launches += 1;
  int32_t bad = 0;
  CK(h, cudaMemcpyAsync(&bad, h->bad_flag, 4, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  if (bad) {
    CK(h, launch_init_round_state(P, h->stream));  // never leave an inconsistent pairing behind
    return fail(GWTF_E_INVALID, "imported round state is not a valid pairing (state reset to empty)");
  }
  return GWTF_OK;
}

gwtf_status gwtf_flow_snapshot(gwtf_flow_t h) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!h->has_snapshot) {
    for (auto& mb : h->mutable_bufs) {
      void* q = nullptr;
      if (!(q = dev_alloc(h, mb.second))) return fail(GWTF_E_NOMEM, "snapshot");
      h->snap.push_back(q);
    }
    h->has_snapshot = true;
  }
  for (size_t i = 0; i < h->mutable_bufs.size(); ++i)
    CK(h, cudaMemcpyAsync(h->snap[i], h->mutable_bufs[i].first, h->mutable_bufs[i].second, cudaMemcpyDeviceToDevice,
                          h->stream));
  return GWTF_OK;
}

gwtf_status gwtf_flow_restore(gwtf_flow_t h) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!h->has_snapshot) return fail(GWTF_E_STATE, "no snapshot");
  for (size_t i = 0; i < h->mutable_bufs.size(); ++i)
    CK(h, cudaMemcpyAsync(h->mutable_bufs[i].first, h->snap[i], h->mutable_bufs[i].second, cudaMemcpyDeviceToDevice,
                          h->stream));
  h->has_assignment = false;
  return GWTF_OK;
}

gwtf_status gwtf_flow_set_profiling(gwtf_flow_t h, int32_t on) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  h->profiling = on != 0;
  for (Timer& t : h->pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  h->pending.clear();
  h->names.clear();
  h->ms.clear();
  h->launches.clear();
  return GWTF_OK;
}

gwtf_status gwtf_flow_kernel_times(gwtf_flow_t h, const char** names, float* ms, int32_t* launches, int32_t cap,
                                   int32_t* count) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  for (Timer& t : h->pending) {
    CK(h, cudaEventSynchronize(t.b));
    float v = 0.f;
    CK(h, cudaEventElapsedTime(&v, t.a, t.b));
    size_t i = std::find(h->names.begin(), h->names.end(), t.name) - h->names.begin();
    if (i == h->names.size()) { h->names.push_back(t.name); h->ms.push_back(0.f); h->launches.push_back(0); }
    h->ms[i] += v;
    h->launches[i] += 1;
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  h->pending.clear();
  const int32_t c = (int32_t)h->names.size();
  if (count) *count = c;
  for (int32_t i = 0; i < std::min(c, cap); ++i) {
    if (names) names[i] = h->names[i].c_str();
    if (ms) ms[i] = h->ms[i];
    if (launches) launches[i] = h->launches[i];
  }
  return GWTF_OK;
}

gwtf_status gwtf_flow_greedy_baseline(gwtf_flow_t h, int64_t* flow_value, int64_t* total_cost) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!flow_value || !total_cost) return fail(GWTF_E_INVALID, "greedy: NULL output");
  const size_t B = h->P.B;
  std::vector<OutMap> maps;
  int64_t *F = nullptr, *C = nullptr;
  if ((s = map_out(h, flow_value, B, 14, &F, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, total_cost, B, 15, &C, maps)) != GWTF_OK) return s;
  int32_t* rem = (int32_t*)scratch(h, 16, B * (size_t)h->P.S * h->P.n * 4);
  if (!rem) return fail(GWTF_E_NOMEM, "greedy scratch");
  Timer t;
  prof_begin(h, "greedy_kernel", &t);
  CK(h, launch_greedy(h->P, rem, F, C, h->stream));
  h->kernel_launches += 1;
  prof_end(h, &t);
  return finish_out(h, maps);
}

gwtf_status gwtf_flow_warm_reroute(gwtf_flow_t h, int32_t* node_flow, int32_t* src_flow, int32_t* snk_flow,
                                   int32_t* arc_flow_dense, int64_t* flow_value, int64_t* total_cost, int64_t* stats,
                                   int32_t* inst_status) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!node_flow || !src_flow || !snk_flow || !flow_value || !total_cost)
    return fail(GWTF_E_INVALID, "warm_reroute: NULL required array");
  const Problem& P = h->P;
  if (P.S > 1 && !arc_flow_dense) return fail(GWTF_E_INVALID, "warm_reroute: NULL arc_flow_dense");
  const size_t B = P.B, Sn = (size_t)P.S * P.n, A = (size_t)std::max(P.S - 1, 0) * P.n * P.n;
  if (2 * (2 * (int64_t)P.n + (int64_t)Sn + (int64_t)A) >= (1ll << 24) - 1)
    return fail(GWTF_E_UNSUPPORTED, "warm_reroute: residual arc ids need more than 24 bits");
  // in/out flow arrays: device mode works in place; host mode copies in and back out
  std::vector<OutMap> maps;
  int32_t* io[4] = {src_flow, node_flow, arc_flow_dense, snk_flow};
  const size_t cnt[4] = {B * P.n, B * Sn, B * A, B * P.n};
  int32_t* dev[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int k = 0; k < 4; ++k) {
    if (!io[k] || cnt[k] == 0) { dev[k] = io[k]; continue; }
    if ((s = map_out(h, io[k], cnt[k], 18 + k, &dev[k], maps)) != GWTF_OK) return s;
    if (host_mode(h) && (s = copy_in(h, dev[k], io[k], cnt[k] * 4)) != GWTF_OK) return s;
  }
  int64_t *F = nullptr, *C = nullptr, *St = nullptr;
  int32_t* Q = nullptr;
  if ((s = map_out(h, flow_value, B, 22, &F, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, total_cost, B, 23, &C, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, stats, 3 * B, 24, &St, maps)) != GWTF_OK) return s;
  if ((s = map_out(h, inst_status, B, 25, &Q, maps)) != GWTF_OK) return s;
  int32_t* Qd = Q;  // the kernels always write a status (the fallback pass reads it)
  if (!Qd && !(Qd = (int32_t*)scratch(h, 27, B * 4))) return fail(GWTF_E_NOMEM, "warm_reroute status");
  void* ws = scratch(h, 26, warm_ws_bytes(P, warm_grid(P)));
  if (!ws) return fail(GWTF_E_NOMEM, "warm_reroute workspace");
  Timer t;
  prof_begin(h, "warm_kernel", &t);
  CK(h, launch_warm(P, dev[0], dev[1], dev[2], dev[3], ws, F, C, St, Qd, (h->flags & GWTF_WARM_REPAIR_ALL) != 0, h->stream));
  h->kernel_launches += (P.debug & 4096) ? 3 : 2;
  // the instances the repair leaves (triage: too much of the flow to re-route; or a stopped
  // repair): the exact solve of that subset, written straight into the caller's arrays (the
  // handle's own solver state stays untouched)
  int32_t* sel = (int32_t*)scratch(h, 28, (B + 1) * 4);
  const size_t nbl = (size_t)std::max(P.S - 1, 1) * P.Lcap;
  Problem P2 = P;
  P2.arcs = (uint32_t*)scratch(h, 29, B * nbl * 4);
  P2.arc_cnt = (int32_t*)scratch(h, 30, B * std::max(P.S - 1, 1) * 4);
  P2.arcw = P.arcw ? (int32_t*)scratch(h, 31, B * nbl * 4) : nullptr;
  int32_t* aug = (int32_t*)scratch(h, 32, B * 4);
  if (!sel || !P2.arcs || !P2.arc_cnt || (P.arcw && !P2.arcw) || !aug) return fail(GWTF_E_NOMEM, "warm_reroute cold subset");
  P2.sel = sel;
  P2.sel_count = sel + B;
  P2.src_f = dev[0];
  P2.g = dev[1];
  P2.snk_f = dev[3];
  CK(h, launch_warm_collect((int32_t)B, Qd, sel, sel + B, P.stats + 12, h->stream));
  const int tier = (h->flags & GWTF_FORCE_GLOBAL_TIER) ? 1 : (h->flags & GWTF_FORCE_CLUSTER_TIER) ? 2 : 0;
  CK(h, launch_ssp(P2, SspOut{F, C, aug, Qd}, h->stream, h->num_sms, tier));
  CK(h, launch_warm_dense(P2, sel, sel + B, dev[2], aug, St, h->stream));
  h->kernel_launches += 1 + ssp_launch_count(P, tier) + (P.S > 1 ? 2 : 1);
  prof_end(h, &t);
  if (!inst_status) {  // no status array from the caller: a failed instance fails the call
    std::vector<int32_t> q(B);
    CK(h, cudaMemcpyAsync(q.data(), Qd, B * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    for (size_t b = 0; b < B; ++b)
      if (q[b] != 0) return fail(GWTF_E_STATE, "warm_reroute: an instance did not reach the optimum (status != 0)");
  }
  return finish_out(h, maps);
}

gwtf_status gwtf_flow_stats(gwtf_flow_t h, int64_t* out, int32_t cap) {
  gwtf_status s = enter(h);
  if (s != GWTF_OK) return s;
  if (!out || cap < 0) return fail(GWTF_E_INVALID, "stats: NULL out");
  std::vector<unsigned long long> v(2048);
  CK(h, cudaMemcpyAsync(v.data(), h->P.stats, 2048 * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  v[15] = (unsigned long long)h->kernel_launches;  // host-side: kernels launched by this handle
  for (int i = 0; i < std::min(cap, 2048); ++i) out[i] = (int64_t)v[i];
  return GWTF_OK;
}

gwtf_status gwtf_flow_destroy(gwtf_flow_t h) {
  if (!h) return GWTF_OK;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  if (h->stream2) {
    cudaStreamSynchronize(h->stream2);
    cudaStreamDestroy(h->stream2);
    cudaEventDestroy(h->ev_fork);
    cudaEventDestroy(h->ev_join);
  }
  for (Timer& t : h->pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  for (void* p : h->allocs) dev_free(h, p);
  for (void* p : h->snap) dev_free(h, p);
  for (DevBuf& b : h->scratch) dev_free(h, b.p);
  cudaGetLastError();
  delete h;
  return GWTF_OK;
}

}  // extern "C"
