// gen/gen.cu -- host and device drivers of the seeded generator (gen/gwtf_gen.h).
// Input plumbing only: raw random fields, no method arithmetic (see header).
#include "gwtf_gen.h"
#include <cuda_runtime.h>
#include <limits.h>

#define GEN_ABSENT INT32_MAX

// One element of each field, shared by the host loop and the device kernel so
// both produce the same bytes.
GEN_HD void gen_node_elem(const gen_config& c, uint64_t is, int64_t b, int32_t k,
                          int32_t* cap, uint8_t* alive, int32_t* comp, int32_t* loc) {
  const int64_t o = b * (int64_t)c.S * c.n + k;
  if (cap) cap[o] = gen_uniform(is, GEN_F_CAP, (uint64_t)k, c.cap_lo, c.cap_hi);
  if (alive) alive[o] = (uint8_t)gen_bernoulli(is, GEN_F_ALIVE, (uint64_t)k, c.alive_thr);
  if (comp) comp[o] = gen_uniform(is, GEN_F_COMP, (uint64_t)k, c.comp_lo, c.comp_hi);
  if (loc) loc[o] = gen_uniform(is, GEN_F_LOC, (uint64_t)k, 0, c.L - 1);
}

GEN_HD int32_t gen_link_elem(const gen_config& c, uint64_t is, int64_t k) {
  if (c.absent_thr && gen_bernoulli(is, GEN_F_ABSENT, (uint64_t)k, c.absent_thr)) return GEN_ABSENT;
  return gen_uniform(is, GEN_F_LINK, (uint64_t)k, c.cost_lo, c.cost_hi);
}

GEN_HD void gen_loc_elem(const gen_config& c, uint64_t is, int64_t b, int32_t k,
                         int32_t* lat, int32_t* bw) {
  const int32_t a = k / c.L, d = k % c.L;
  const int64_t o = b * (int64_t)c.L * c.L + k;
  if (lat) lat[o] = (a == d) ? gen_uniform(is, GEN_F_LAT, (uint64_t)k, c.lat_intra_lo, c.lat_intra_hi)
                             : gen_uniform(is, GEN_F_LAT, (uint64_t)k, c.lat_inter_lo, c.lat_inter_hi);
  if (bw) bw[o] = (a == d) ? c.bw_intra : gen_uniform(is, GEN_F_BW, (uint64_t)k, c.bw_inter_lo, c.bw_inter_hi);
}

GEN_HD void gen_churn_elem(const gen_config& c, uint64_t is, int64_t b, int32_t k,
                           const uint8_t* alive_base, uint8_t* alive_new) {
  const int64_t o = b * (int64_t)c.S * c.n + k;
  const int was = alive_base[o];
  alive_new[o] = (uint8_t)(was ? !gen_bernoulli(is, GEN_F_CRASH, (uint64_t)k, c.crash_thr)
                               : gen_bernoulli(is, GEN_F_REJOIN, (uint64_t)k, c.rejoin_thr));
}

extern "C" int gen_instances_host(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                                  int32_t* cap, uint8_t* alive, int64_t* supply,
                                  int32_t* src, int32_t* snk, int32_t* link,
                                  int32_t* comp, int32_t* loc, int32_t* dloc, int32_t* lat, int32_t* bw) {
  if (!c || c->S < 1 || c->n < 1 || B < 0) return 1;
  const int32_t Sn = c->S * c->n;
  const int64_t tile = (int64_t)(c->S - 1) * c->n * c->n;
  for (int64_t b = 0; b < B; ++b) {
    const uint64_t is = gen_instance_seed(base_seed, c->cfg_id, (uint64_t)(inst0 + b));
    for (int32_t k = 0; k < Sn; ++k) gen_node_elem(*c, is, b, k, cap, alive, comp, loc);
    if (supply) supply[b] = c->M;
    if (c->cost_kind == GEN_COST_DIRECT) {
      for (int32_t i = 0; i < c->n; ++i) {
        if (src) src[b * c->n + i] = gen_uniform(is, GEN_F_SRC, (uint64_t)i, c->cost_lo, c->cost_hi);
        if (snk) snk[b * c->n + i] = gen_uniform(is, GEN_F_SNK, (uint64_t)i, c->cost_lo, c->cost_hi);
      }
      if (link) for (int64_t k = 0; k < tile; ++k) link[b * tile + k] = gen_link_elem(*c, is, k);
    } else {
      if (dloc) dloc[b] = gen_uniform(is, GEN_F_DLOC, 0, 0, c->L - 1);
      for (int32_t k = 0; k < c->L * c->L; ++k) gen_loc_elem(*c, is, b, k, lat, bw);
    }
  }
  return 0;
}

extern "C" int gen_churn_host(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                              const uint8_t* alive_base, uint8_t* alive_new, uint8_t* linkdrop) {
  if (!c || !alive_base || !alive_new) return 1;
  const int32_t Sn = c->S * c->n;
  const int64_t tile = (int64_t)(c->S - 1) * c->n * c->n;
  for (int64_t b = 0; b < B; ++b) {
    const uint64_t is = gen_instance_seed(base_seed, c->cfg_id, (uint64_t)(inst0 + b));
    for (int32_t k = 0; k < Sn; ++k) gen_churn_elem(*c, is, b, k, alive_base, alive_new);
    if (linkdrop)
      for (int64_t k = 0; k < tile; ++k)
        linkdrop[b * tile + k] = (uint8_t)gen_bernoulli(is, GEN_F_LINKDROP, (uint64_t)k, c->linkdrop_thr);
  }
  return 0;
}

// ---- device twins: one thread per element, grid-stride ---------------------
__global__ void k_gen_nodes(gen_config c, uint64_t base_seed, int64_t inst0, int64_t B,
                            int32_t* cap, uint8_t* alive, int64_t* supply,
                            int32_t* src, int32_t* snk, int32_t* comp, int32_t* loc,
                            int32_t* dloc, int32_t* lat, int32_t* bw) {
  const int32_t Sn = c.S * c.n, LL = c.L * c.L;
  const int32_t per = Sn + 2 * c.n + LL + 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    const int32_t k = (int32_t)(t % per);
    const uint64_t is = gen_instance_seed(base_seed, c.cfg_id, (uint64_t)(inst0 + b));
    if (k < Sn) {
      gen_node_elem(c, is, b, k, cap, alive, comp, loc);
    } else if (k < Sn + 2 * c.n) {
      if (c.cost_kind != GEN_COST_DIRECT) continue;
      const int32_t i = (k - Sn) % c.n;
      if (k - Sn < c.n) { if (src) src[b * c.n + i] = gen_uniform(is, GEN_F_SRC, (uint64_t)i, c.cost_lo, c.cost_hi); }
      else { if (snk) snk[b * c.n + i] = gen_uniform(is, GEN_F_SNK, (uint64_t)i, c.cost_lo, c.cost_hi); }
    } else if (k < Sn + 2 * c.n + LL) {
      if (c.cost_kind == GEN_COST_EQ1) gen_loc_elem(c, is, b, k - Sn - 2 * c.n, lat, bw);
    } else if (k == Sn + 2 * c.n + LL) {
      if (supply) supply[b] = c.M;
    } else {
      if (c.cost_kind == GEN_COST_EQ1 && dloc) dloc[b] = gen_uniform(is, GEN_F_DLOC, 0, 0, c.L - 1);
    }
  }
}

__global__ void k_gen_links(gen_config c, uint64_t base_seed, int64_t inst0, int64_t B, int32_t* link,
                            const uint8_t* unused, uint8_t* linkdrop) {
  const int64_t tile = (int64_t)(c.S - 1) * c.n * c.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B * tile;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / tile, k = t % tile;
    const uint64_t is = gen_instance_seed(base_seed, c.cfg_id, (uint64_t)(inst0 + b));
    if (link) link[t] = gen_link_elem(c, is, k);
    if (linkdrop) linkdrop[t] = (uint8_t)gen_bernoulli(is, GEN_F_LINKDROP, (uint64_t)k, c.linkdrop_thr);
  }
}

__global__ void k_gen_churn_nodes(gen_config c, uint64_t base_seed, int64_t inst0, int64_t B,
                                  const uint8_t* alive_base, uint8_t* alive_new) {
  const int32_t Sn = c.S * c.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B * Sn;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / Sn;
    const uint64_t is = gen_instance_seed(base_seed, c.cfg_id, (uint64_t)(inst0 + b));
    gen_churn_elem(c, is, b, (int32_t)(t % Sn), alive_base, alive_new);
  }
}

static int grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

extern "C" int gen_instances_device(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                                    int32_t* cap, uint8_t* alive, int64_t* supply,
                                    int32_t* src, int32_t* snk, int32_t* link,
                                    int32_t* comp, int32_t* loc, int32_t* dloc, int32_t* lat, int32_t* bw,
                                    void* stream) {
  if (!c || c->S < 1 || c->n < 1 || B < 0) return 1;
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t per = (int64_t)c->S * c->n + 2 * c->n + (int64_t)c->L * c->L + 2;
  k_gen_nodes<<<grid_for(B * per), 256, 0, st>>>(*c, base_seed, inst0, B, cap, alive, supply, src, snk,
                                                  comp, loc, dloc, lat, bw);
  const int64_t tile = (int64_t)(c->S - 1) * c->n * c->n;
  if (link && c->cost_kind == GEN_COST_DIRECT && tile > 0)
    k_gen_links<<<grid_for(B * tile), 256, 0, st>>>(*c, base_seed, inst0, B, link, nullptr, nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int gen_churn_device(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                                const uint8_t* alive_base, uint8_t* alive_new, uint8_t* linkdrop,
                                void* stream) {
  if (!c || !alive_base || !alive_new) return 1;
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  k_gen_churn_nodes<<<grid_for(B * c->S * c->n), 256, 0, st>>>(*c, base_seed, inst0, B, alive_base, alive_new);
  const int64_t tile = (int64_t)(c->S - 1) * c->n * c->n;
  if (linkdrop && tile > 0)
    k_gen_links<<<grid_for(B * tile), 256, 0, st>>>(*c, base_seed, inst0, B, nullptr, nullptr, linkdrop);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
