/* gen/gwtf_gen.h -- seeded, counter-based synthetic instance generator.
 *
 * This module is SHARED INPUT PLUMBING: it is the only code both the CPU
 * oracle (oracle/) and the CUDA product path (paper_2509_21221_b200/) see,
 * and it holds none of the method's arithmetic.  It draws raw random fields
 * (capacities, alive flags, raw per-link costs, Eq. 1 raw parameters, churn
 * draws); it never evaluates Eq. 1, never builds a residual graph, never
 * solves anything.  Eq. 1 is evaluated separately by the product
 * (gwtf_eq1_cost_tiles, a CUDA kernel) and by the oracle (oracle_eq1).
 *
 * Every field value is a pure function of (base_seed, cfg_id, instance id,
 * field id, element index), so any rank or thread regenerates any instance
 * independently (SURVEY.md 8(d) "Configs as concrete synthetic inputs").
 * The recipe is documented in DESIGN.md section 4.
 */
#ifndef GWTF_GEN_H
#define GWTF_GEN_H
#include <stdint.h>

#ifdef __CUDACC__
#define GEN_HD __host__ __device__ __forceinline__
#else
#define GEN_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* field ids of the counter-based draws */
enum {
  GEN_F_CAP = 1, GEN_F_ALIVE = 2, GEN_F_SRC = 3, GEN_F_SNK = 4, GEN_F_LINK = 5,
  GEN_F_COMP = 6, GEN_F_LOC = 7, GEN_F_LAT = 8, GEN_F_BW = 9, GEN_F_DLOC = 10,
  GEN_F_CRASH = 11, GEN_F_REJOIN = 12, GEN_F_LINKDROP = 13, GEN_F_ABSENT = 14
};

/* cost_kind */
enum { GEN_COST_DIRECT = 0, GEN_COST_EQ1 = 1 };

typedef struct gen_config {
  uint32_t cfg_id;
  int32_t S, n, max_cap;
  int64_t M;                 /* supply of the data node (microbatches) */
  int32_t cap_lo, cap_hi;    /* capacities: inclusive uniform integers */
  uint64_t alive_thr;        /* base alive iff (draw>>32) < alive_thr; 1<<32 = always */
  uint64_t absent_thr;       /* base link absent iff (draw>>32) < absent_thr; 0 = never */
  int32_t cost_kind;         /* GEN_COST_DIRECT or GEN_COST_EQ1 */
  int32_t cost_lo, cost_hi;  /* DIRECT: every arc cost (src, snk, inter-stage) */
  /* EQ1 raw parameters (PAPER.md:166-169 symbols c, lambda, beta, size) */
  int32_t L;                 /* number of geographic locations */
  int32_t comp_lo, comp_hi;  /* c_i, ms */
  int32_t lat_inter_lo, lat_inter_hi, lat_intra_lo, lat_intra_hi; /* lambda, ms */
  int32_t bw_inter_lo, bw_inter_hi, bw_intra;                     /* beta, Mbit/s */
  int64_t size_kbit;         /* activation size, kbit (kbit / (Mbit/s) = ms) */
  /* churn draws (between the pre-churn and the timed solve) */
  uint64_t crash_thr, rejoin_thr, linkdrop_thr;
} gen_config;

GEN_HD uint64_t gen_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
GEN_HD uint64_t gen_instance_seed(uint64_t base_seed, uint32_t cfg_id, uint64_t inst) {
  return gen_mix(base_seed ^ ((uint64_t)cfg_id << 48) ^ inst);
}
GEN_HD uint64_t gen_draw(uint64_t iseed, uint32_t field, uint64_t idx) {
  return gen_mix(gen_mix(iseed + (uint64_t)field * 0x9E3779B97F4A7C15ull) ^ idx);
}
GEN_HD uint32_t gen_pick(uint64_t x, uint32_t m) {
  return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32);
}
GEN_HD int32_t gen_uniform(uint64_t iseed, uint32_t field, uint64_t idx, int32_t lo, int32_t hi) {
  return lo + (int32_t)gen_pick(gen_draw(iseed, field, idx), (uint32_t)(hi - lo + 1));
}
GEN_HD int gen_bernoulli(uint64_t iseed, uint32_t field, uint64_t idx, uint64_t thr) {
  return (gen_draw(iseed, field, idx) >> 32) < thr;
}

/* ---- host entry points (gen/gen.cu, libgwtfgen.so) ---------------------
 * All arrays are for instances [inst0, inst0+B) with local index b.
 * Layouts (row-major, C order):
 *   cap[B][S][n] i32, alive[B][S][n] u8, supply[B] i64
 *   DIRECT: src[B][n] i32, snk[B][n] i32, link[B][S-1][n_dst][n_src] i32
 *           (link[b][s][v][u] = raw cost of u in stage s -> v in stage s+1;
 *            INT32_MAX = absent link)
 *   EQ1:    comp[B][S][n] i32, loc[B][S][n] i32, dloc[B] i32,
 *           lat[B][L][L] i32, bw[B][L][L] i32
 *   churn:  alive_new[B][S][n] u8, linkdrop[B][S-1][n][n] u8
 * Unused outputs may be NULL.  Return 0 on success. */
int gen_instances_host(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                       int32_t* cap, uint8_t* alive, int64_t* supply,
                       int32_t* src, int32_t* snk, int32_t* link,
                       int32_t* comp, int32_t* loc, int32_t* dloc, int32_t* lat, int32_t* bw);
int gen_churn_host(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                   const uint8_t* alive_base, uint8_t* alive_new, uint8_t* linkdrop);
/* Same, device pointers, enqueued on `stream` (cudaStream_t). */
int gen_instances_device(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                         int32_t* cap, uint8_t* alive, int64_t* supply,
                         int32_t* src, int32_t* snk, int32_t* link,
                         int32_t* comp, int32_t* loc, int32_t* dloc, int32_t* lat, int32_t* bw,
                         void* stream);
int gen_churn_device(const gen_config* c, uint64_t base_seed, int64_t inst0, int64_t B,
                     const uint8_t* alive_base, uint8_t* alive_new, uint8_t* linkdrop, void* stream);

#ifdef __cplusplus
}
#endif
#endif
