/* oracle/oracle.h -- plain, slow, obviously-correct CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code with the CUDA product path (paper_2509_21221_b200/);
 * the only common module is the seeded input generator gen/.
 *
 * Every function cites the PAPER.md (P:line) / SPEC.md (S:line) passage or
 * the DESIGN.md reading it follows.  Parity status of each function is listed
 * in DESIGN.md section 3 ("what pins the oracle").
 *
 * Graph: data node D is source
 * and sink; relays (s,i), s in [0,S), i in [0,n); capacity cap_e = alive?cap:0;
 * arc costs are integers, INT32_MAX = absent link.
 *   link[s][v][u] = d(u in stage s -> v in stage s+1)        (dest-major)
 *   src[i] = d(D -> (0,i)),  snk[i] = d((S-1,i) -> D)
 */
#ifndef GWTF_ORACLE_H
#define GWTF_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t S, n, max_cap;
  int64_t M;               /* data-node supply (microbatches) */
  const int32_t* cap;      /* [S][n] */
  const uint8_t* alive;    /* [S][n], NULL = all alive */
  const int32_t* src;      /* [n] */
  const int32_t* snk;      /* [n] */
  const int32_t* link;     /* [S-1][n][n] dest-major */
} orc_instance;

/* Eq. 1 in integer half-units: D2 = 2*d =
 * c_i + c_j + lam_ij + lam_ji + floor(4*size/(beta_ij+beta_ji)), data node c_D = 0.
 * comp/loc [S][n], lat/bw [L][L]; outputs src[n], snk[n], link[S-1][n][n]. */
int orc_eq1(int32_t S, int32_t n, int32_t L, const int32_t* comp, const int32_t* loc, int32_t dloc,
            const int32_t* lat, const int32_t* bw, int64_t size_kbit,
            int32_t* src, int32_t* snk, int32_t* link);

/* Canonical successive shortest paths.  Outputs the
 * max-flow value F, its min cost, the augmentation count A and the canonical
 * assignment.  Arrays may be NULL.  Returns 0, or <0 on internal check failure. */
int orc_ssp(const orc_instance* I, int64_t* F, int64_t* cost, int32_t* A,
            int32_t* node_flow /*[S][n]*/, int32_t* src_flow /*[n]*/, int32_t* snk_flow /*[n]*/,
            int32_t* arc_flow /*[S-1][n][n] dest-major*/, int64_t* cost_curve /*[M+1] or NULL*/);

/* Batch SSP over B instances laid out as the C-ABI does, T threads. */
int orc_ssp_batch(int64_t B, int32_t S, int32_t n, int32_t max_cap, const int32_t* cap,
                  const uint8_t* alive, const int32_t* src, const int32_t* snk, const int32_t* link,
                  const int64_t* supply, int64_t* F, int64_t* cost, int32_t* A, int32_t threads);

/* Warm-start rerouting after churn:
 * keep the pre-churn assignment of Iold (node/src/snk/arc flows, layouts as orc_ssp), strip
 * the units the churned instance Inew cannot carry, cancel negative residual cycles, resume
 * SSP.  (F, cost) equal orc_ssp(Inew)'s; the assignment may differ (several optima).
 * stats[3] = {units stripped, cycles cancelled, augmentations}.  Outputs may be NULL. */
int orc_warm_reroute(const orc_instance* Iold, const int32_t* node_flow, const int32_t* src_flow,
                     const int32_t* snk_flow, const int32_t* arc_flow, const orc_instance* Inew, int64_t* F,
                     int64_t* cost, int64_t* stats, int32_t* node_flow_out, int32_t* src_flow_out,
                     int32_t* snk_flow_out, int32_t* arc_flow_out);

/* Independent cross-check: primal network simplex with strongly feasible
 * spanning trees (Cunningham) on the node-split graph plus a bypass arc. */
int orc_network_simplex(const orc_instance* I, int64_t* F, int64_t* cost);

/* Certificates (SURVEY C3 iv): returns 0 iff the assignment is conserved and
 * within capacity, has value F and cost `cost`, is a maximum flow (F == M or
 * no residual s*-t* path) and is optimal (no negative residual cycle;
 * Bellman-Ford potentials with non-negative reduced costs).  >0 = which check failed. */
int orc_certify(const orc_instance* I, int64_t F, int64_t cost, const int32_t* node_flow,
                const int32_t* src_flow, const int32_t* snk_flow, const int32_t* arc_flow);

/* Annealing threshold table thr[k][delta] = min(2^32-1, floor(exp(-delta/(T0*alpha^k))*2^32))
 * (DESIGN.md 2.4).  width = first delta with thr[0][delta] == 0, K = first k
 * with thr[k][1] == 0.  table may be NULL (sizes only); cap = table capacity in entries. */
int orc_anneal_table(double T0, double alpha, int32_t* width, int32_t* K, uint32_t* table, int64_t cap);

/* ---- decentralized rounds, GWTF-SYNC ---- */
typedef struct orc_rounds orc_rounds;
enum { ORC_OBJ_SUM = 0, ORC_OBJ_MINIMAX = 1 };
orc_rounds* orc_rounds_create(const orc_instance* I, uint64_t seed, int64_t inst_id, double T0,
                              double alpha, int32_t objective, int32_t steady_window, int32_t deny_after);
void orc_rounds_destroy(orc_rounds* R);
/* Run rounds until W quiet rounds or max_rounds.  digests[r] = state digest after round r. */
int orc_rounds_run(orc_rounds* R, int32_t max_rounds, int32_t* rounds_run, int64_t* F_dec,
                   int64_t* cost_dec, int32_t* dangling, uint64_t* digests);
/* Churn: new alive mask [S][n] (NULL = unchanged) and edge updates
 * [k][5] = {b (ignored), s, v_dst, u_src, new_cost}; s = -1 -> src[v_dst], s = S-1 -> snk[u_src]. */
int orc_rounds_apply_churn(orc_rounds* R, const uint8_t* alive_new, const int32_t* updates, int64_t k);
/* State export: up/down [S][n][max_cap] (encoded pointers), src_down/snk_up [M],
 * kacc/deny [S][n], quiet, round. */
int orc_rounds_export(const orc_rounds* R, int32_t* up, int32_t* down, int32_t* src_down, int32_t* snk_up,
                      int32_t* kacc, int32_t* deny, int32_t* quiet, int64_t* round);
uint64_t orc_rounds_digest(const orc_rounds* R);
/* Inverse of orc_rounds_export (checkpoint / resume): install a round state given in the
 * export layouts.  Returns -1 (state unchanged) unless the pointers are a valid pairing:
 * bijective, within capacity, across one stage boundary or to the data node. */
int orc_rounds_import(orc_rounds* R, const int32_t* up, const int32_t* down, const int32_t* src_down,
                      const int32_t* snk_up, const int32_t* kacc, const int32_t* deny, int32_t quiet, int64_t round);
/* The R4 draws: mix64 = splitmix64 finalizer, h(gid, stream) =
 * mix(mix(mix(mix(seed) ^ inst) ^ round) ^ (gid*4 + stream)), pick(x, m) = ((x >> 32) * m) >> 32. */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_rng_h(uint64_t seed, int64_t inst, int64_t round, int32_t gid, int32_t stream);
uint32_t orc_pick(uint64_t x, uint32_t m);
/* The instance as currently masked (after churn): cap_eff [S][n], src [n], snk [n], link [S-1][n][n]. */
int orc_rounds_instance(const orc_rounds* R, int32_t* cap_eff, uint8_t* alive, int32_t* src, int32_t* snk,
                        int32_t* link);
/* LLaMA "crash during backward" victim rule; returns victim gid or -1. */
int32_t orc_llama_victim(const orc_rounds* R, uint64_t draw_stage, uint64_t draw_pick);

/* ---- multi-data-node decentralized rounds, MC-SYNC ----
 * K data nodes with source / sink costs src_k / snk_k [K][n] and supplies M_k [K] on the shared
 * relays and links of I (I->src / I->snk / I->M are ignored).  Every non-FREE slot carries the
 * data node of its chain; requests, grants, Change and self-pairing stay within one data node.
 * Rounds from the empty state; F_dec / cost_dec [K]; digests per round (optional).  Pointers:
 * relay slot >= 0, -1 none, data-node slot i of D_k = -2 - (k * Mmax + i), Mmax = max_k M_k. */
typedef struct orc_mc_rounds orc_mc_rounds;
orc_mc_rounds* orc_mc_rounds_create(const orc_instance* I, int32_t K, const int32_t* src_k, const int32_t* snk_k,
                                    const int64_t* M_k, uint64_t seed, int64_t inst_id, double T0, double alpha,
                                    int32_t objective, int32_t W, int32_t deny_after);
void orc_mc_rounds_destroy(orc_mc_rounds* R);
int orc_mc_rounds_run(orc_mc_rounds* R, int32_t max_rounds, int32_t* rounds_run, int64_t* F_dec, int64_t* cost_dec,
                      int32_t* dangling, uint64_t* digests);
/* up/down/tag [S][n][max_cap] (tag -1 on FREE slots), src_down/snk_up [K][Mmax], kacc/deny [S][n] */
int orc_mc_rounds_export(const orc_mc_rounds* R, int32_t* up, int32_t* down, int32_t* tag, int32_t* src_down,
                         int32_t* snk_up, int32_t* kacc, int32_t* deny, int32_t* quiet, int64_t* round);
uint64_t orc_mc_rounds_digest(const orc_mc_rounds* R);
/* Inverse of orc_mc_rounds_export (-1 unless a valid tagged pairing; kacc / deny may be NULL). */
int orc_mc_rounds_import(orc_mc_rounds* R, const int32_t* up, const int32_t* down, const int32_t* tag,
                         const int32_t* src_down, const int32_t* snk_up, const int32_t* kacc, const int32_t* deny,
                         int32_t quiet, int64_t round);

/* Whole per-instance workload of one bench step, for the cpu_baseline and
 * the full-size parity samples: pre-churn rounds to quiescence, churn, cold SSP on
 * the masked graph, repair rounds.  churn_kind 0 none, 1 random (alive_new +
 * updates), 2 victim.  Per-instance outputs [B]. */
typedef struct {
  int64_t F, cost; int32_t A, rounds; int64_t F_dec, cost_dec; int32_t dangling, pre_rounds;
  uint64_t digest;
  int64_t step_ns;  /* wall time of the step's work (churn + SSP + repair rounds), this instance */
} orc_result;
int orc_pipeline_batch(int64_t B, int32_t S, int32_t n, int32_t max_cap, const int32_t* cap,
                       const uint8_t* alive, const int32_t* src, const int32_t* snk, const int32_t* link,
                       const int64_t* supply, int32_t churn_kind, const uint8_t* alive_new,
                       const int32_t* updates, int64_t k_updates, const uint64_t* victim_draws,
                       uint64_t seed, int64_t inst_base, double T0, double alpha, int32_t objective,
                       int32_t W, int32_t deny_after, int32_t max_rounds, int32_t threads,
                       orc_result* out);

#ifdef __cplusplus
}
#endif
#endif
