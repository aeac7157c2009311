/* include/gwtf.h -- C-ABI of the B200 GWTF routing min-cost-flow library (ABI v1).
 *
 * The library solves, for a batch of B independent instances, GWTF's microbatch-routing
 * problem: route the largest number of microbatches from the data node D through S
 * pipeline stages of relay clients and back to D at minimum total cost
 *   min sum_{i,j} f(i,j) d(i,j)                              (Eq. 2)
 * subject to node capacities cap_i ("maximum number cap_i of microbatches")
 * and the data node's supply M ("Data nodes start with unpaired flows
 * matching their capacity"), with d(i,j) the Eq. 1 cost.
 * Each instance gets (a) the exact solve by successive shortest augmenting paths and
 * (b) the paper's decentralized Request Flow / Change / Redirect rounds (PAPER.md:241-263,
 * DENY PAPER.md:269) as synchronous per-node updates.  Normative semantics: DESIGN.md
 * section 2; the CPU oracle in oracle/ implements the same definitions independently.
 *
 * Conventions for every entry point:
 *  - No exception crosses the ABI; every call returns gwtf_status; gwtf_last_error()
 *    gives a thread-local message for the last non-OK status.
 *  - Array arguments are DEVICE pointers on the handle's device unless the handle was
 *    created with GWTF_HOST_PTRS, in which case they are HOST pointers (pinned memory is
 *    fastest) and the library does the copies itself on the handle's stream.
 *  - All work is enqueued on the handle's stream; outputs are valid after that stream
 *    synchronizes (HOST_PTRS handles synchronize before returning outputs).
 *  - A handle is bound to one device and stream and is not thread-safe.
 *  - A CUDA error poisons the handle: every later call returns GWTF_E_CUDA.
 *  - Costs are integers; GWTF_ABSENT (INT32_MAX) marks a missing link.
 */
#ifndef GWTF_H
#define GWTF_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define GWTF_ABI_VERSION 1
#define GWTF_ABSENT INT32_MAX
#define GWTF_HOST_PTRS (1u << 0) /* array arguments of every call on this handle are host pointers */
#define GWTF_WARM_REPAIR_ALL (1u << 1) /* gwtf_flow_warm_reroute repairs every instance (no triage) */
#define GWTF_FORCE_GLOBAL_TIER (1u << 30) /* testing: run the exact solve through the global-memory tier */
#define GWTF_FORCE_CLUSTER_TIER (1u << 29) /* testing: run the exact solve through the cluster tier */

typedef struct gwtf_flow_s* gwtf_flow_t; /* opaque; owns all device workspace */

typedef enum {
  GWTF_OK = 0,
  GWTF_E_INVALID = 1,     /* bad sizes, NULL required pointer, out-of-range value */
  GWTF_E_NOMEM = 2,       /* device allocation failed */
  GWTF_E_CUDA = 3,        /* CUDA error (sticky: the handle is poisoned) */
  GWTF_E_OVERFLOW = 4,    /* an integer bound of DESIGN.md 2.2 could be exceeded */
  GWTF_E_STATE = 5,       /* call out of order (e.g. get_assignment before solve_batch) */
  GWTF_E_UNSUPPORTED = 6  /* shape outside the compiled kernels' limits */
} gwtf_status;

typedef enum { GWTF_OBJ_SUM = 0, GWTF_OBJ_MINIMAX = 1 } gwtf_objective;

typedef struct {
  uint32_t abi_version;        /* must be GWTF_ABI_VERSION */
  int32_t num_instances;       /* B >= 1 */
  int32_t num_stages;          /* S, 1..64 */
  int32_t clients_per_stage;   /* n, 1..4096 (absent clients: alive = 0) */
  int32_t max_cap;             /* 0..32: bound on cap, sizes the per-relay slot arrays */
  /* inputs, read during create and COPIED into the handle (caller may free afterwards): */
  const int32_t* cap;          /* [B][S][n], 0..max_cap */
  const uint8_t* alive;        /* [B][S][n], NULL = all alive; crashed relay: capacity 0 */
  const int32_t* src_cost;     /* [B][n]  d(D, relay (0,i)); 0..2^30-1 or GWTF_ABSENT */
  const int32_t* snk_cost;     /* [B][n]  d(relay (S-1,i), D) */
  const int32_t* link_cost;    /* [B][S-1][n_dst][n_src]: link_cost[b][s][v][u] = d((s,u),(s+1,v)) */
  const int64_t* supply;       /* [B] M >= 0: microbatches of the data node (source supply = sink slots) */
  /* decentralized-round parameters */
  uint64_t seed;               /* counter-based RNG seed of the rounds (DESIGN.md 2.3 R4) */
  int64_t inst_base;           /* global id of instance 0 (RNG stream; multi-GPU shards) */
  double T0;                   /* initial annealing temperature (paper: 1.7); <= 0 disables uphill moves */
  double alpha;                /* cooling factor per accepted move, 0 < alpha < 1 (paper: 0.95) */
  int32_t objective;           /* gwtf_objective for Change/Redirect moves */
  int32_t steady_window;       /* W >= 1 quiet rounds = steady state (default 5) */
  int32_t deny_after;          /* idle rounds holding unpaired inflow before DENY (default 3) */
  int32_t device;              /* CUDA device ordinal */
  void* stream;                /* cudaStream_t (NULL = legacy default stream) */
  uint32_t flags;              /* GWTF_HOST_PTRS | GWTF_WARM_REPAIR_ALL | GWTF_FORCE_GLOBAL_TIER | GWTF_FORCE_CLUSTER_TIER */
} gwtf_problem_desc;

/* Eq. 1 evaluated on the device in integer half-units:
 *   D2(i,j) = c_i + c_j + lam[l_i][l_j] + lam[l_j][l_i] + floor(4*size/(beta[l_i][l_j] + beta[l_j][l_i]))
 * = 2 d(i,j) up to the floor of the transfer term; the data node has c_D = 0.
 * comp/loc [B][S][n] (ms, location index), dloc [B], lat/bw [B][L][L] (ms, Mbit/s),
 * size in kbit.  Writes src_out/snk_out [B][n] and link_out [B][S-1][n][n] (the layout
 * gwtf_problem_desc expects).  Device pointers; enqueued on `stream`. */
gwtf_status gwtf_eq1_cost_tiles(int32_t B, int32_t S, int32_t n, int32_t L, const int32_t* comp,
                                const int32_t* loc, const int32_t* dloc, const int32_t* lat,
                                const int32_t* bw, int64_t size_kbit, int32_t* src_out,
                                int32_t* snk_out, int32_t* link_out, void* stream);

/* Node addition ("the optimal choice of node addition is
 * determined by running the minimum cost flow algorithm for each combination of S candidate
 * nodes added to each of the S stages").  Builds placements
 * p = first .. first+count-1 of S candidates, one per stage, into a base instance, as a batch of
 * (n+1)-client instances in the gwtf_problem_desc layout: placement p is the p-th permutation of
 * the candidates in lexicographic order (factorial number system; perm[s] = candidate placed in
 * stage s, as client n).  Inputs (device pointers, read only):
 *   cap [S][n], src_cost [n], snk_cost [n], link_cost [S-1][n][n] (dest-major) of the base;
 *   cand_cap [S]; cand_in [S][S][n]: cand_in[c][s][u] = d((s-1,u) -> c in stage s) for s >= 1,
 *   cand_in[c][0][0] = d(D -> c in stage 0); cand_out [S][S][n]: cand_out[c][s][v] =
 *   d(c in stage s -> (s+1,v)) for s <= S-2, cand_out[c][S-1][0] = d(c -> D);
 *   cand_cc [S][S]: d(c1 -> c2) when c1 is in stage s and c2 in stage s+1.
 * Outputs (device, caller-owned): cap_out [count][S][n+1], src_out/snk_out [count][n+1],
 * link_out [count][S-1][n+1][n+1].  Solve them with gwtf_flow_create + gwtf_flow_solve_batch.
 * INVALID on S outside 1..20, n < 1, first/count outside [0, S!], NULL arrays. */
gwtf_status gwtf_addition_build(int32_t S, int32_t n, const int32_t* cap, const int32_t* src_cost,
                                const int32_t* snk_cost, const int32_t* link_cost, const int32_t* cand_cap,
                                const int32_t* cand_in, const int32_t* cand_out, const int32_t* cand_cc,
                                int64_t first, int64_t count, int32_t* cap_out, int32_t* src_out,
                                int32_t* snk_out, int32_t* link_out, void* stream);

/* The optimal placement among `count` solved placements (device arrays F, cost [count]): the
 * largest max-flow value, then the lowest cost, then the lowest index (the lexicographically first
 * assignment).  Writes its index to best_index (device int64).  INVALID on
 * count < 1 or NULL arrays. */
gwtf_status gwtf_addition_select(int64_t count, const int64_t* flow_value, const int64_t* total_cost,
                                 int64_t* best_index, void* stream);

/* Validate the description (errors: INVALID, OVERFLOW when (2Sn+2)*maxcost >= 2^42 or
 * (2Sn+2)*maxcost*M >= 2^62, UNSUPPORTED), allocate the handle's workspace, copy the
 * inputs into the handle's padded tiles, build the annealing threshold table on the
 * host (IEEE double) and initialise the round state (all slots FREE). */
gwtf_status gwtf_flow_create(const gwtf_problem_desc* d, gwtf_flow_t* out);

/* Exact solve of every instance on its current (masked) graph from zero flow: canonical
 * successive shortest paths with lexicographic (cost, hops) keys.
 * Outputs [B] (caller-owned): max-flow value F, its minimum cost, the number of
 * augmentations (may be NULL) and a per-instance status (0 = ok; may be NULL).
 * The canonical assignment is kept in the handle (gwtf_flow_get_assignment). */
gwtf_status gwtf_flow_solve_batch(gwtf_flow_t h, int64_t* flow_value, int64_t* total_cost,
                                  int32_t* augmentations, int32_t* inst_status);

/* Run synchronous decentralized rounds (phases R0a..R7) on every
 * instance until W consecutive quiet rounds or max_rounds rounds in this call.
 * Outputs [B]: rounds run, F_dec (complete SRC->SNK chains), cost_dec (their Eq. 2 cost),
 * dangling (unpaired outflow slots).  round_digests [B][max_rounds] (NULL = skip) gets the
 * state digest after each round (0 past the last round run). */
gwtf_status gwtf_flow_decentralized_rounds(gwtf_flow_t h, int32_t max_rounds, int32_t* rounds_run,
                                           int64_t* dec_flow, int64_t* dec_cost, int32_t* dangling,
                                           uint64_t* round_digests);

/* gwtf_flow_solve_batch and gwtf_flow_decentralized_rounds of the same step issued together: the two
 * solvers read the same (masked) graph and write disjoint state, so the rounds run on a second
 * stream of the handle concurrently with the exact solve and are joined back into the handle's
 * stream before the call returns (device mode: before later work on the stream runs).  Outputs
 * as in the two calls (no digests).  Same errors. */
gwtf_status gwtf_flow_solve_and_rounds(gwtf_flow_t h, int32_t max_rounds, int64_t* flow_value, int64_t* total_cost,
                                       int32_t* augmentations, int32_t* inst_status, int32_t* rounds_run,
                                       int64_t* dec_flow, int64_t* dec_cost, int32_t* dangling);

/* Churn between solves/rounds: alive_new [B][S][n] (NULL = unchanged)
 * replaces the alive mask (crash / rejoin); edge_updates [k][5] = {b, s, v_dst, u_src, cost}
 * sets link_cost[b][s][v_dst][u_src] = cost for 0 <= s < S-1, src_cost[b][v_dst] for
 * s = -1, snk_cost[b][u_src] for s = S-1 (cost may be GWTF_ABSENT: a dropped link).
 * Round-state pointers into crashed relays or across dropped links are cleared in place;
 * accepted-move counters, deny counters and quiet counters reset.  The next solve_batch
 * is a cold solve on the masked graph.  INVALID on out-of-range updates; OVERFLOW (that update
 * rejected) when a finite cost c breaks create's key bounds, (2Sn+2)*c >= 2^42 or
 * (2Sn+2)*c*Mmax >= 2^62.  Other valid updates are applied in both cases. */
gwtf_status gwtf_flow_apply_churn(gwtf_flow_t h, const uint8_t* alive_new, const int32_t* edge_updates,
                                  int64_t k);

/* Residual node capacities after the last solve_batch, cap_out [B][S][n] = (alive ? cap : 0) - node flow:
 * the capacities the next data node's single-commodity problem sees in the multi-data-node
 * decomposition (one single-commodity problem per data node over
 * residual capacities, in round-robin order).  STATE if no solve has run since create/churn. */
gwtf_status gwtf_flow_residual_caps(gwtf_flow_t h, int32_t* cap_out);

/* Canonical assignment of the last solve_batch: node_flow [B][S][n], src_flow [B][n],
 * snk_flow [B][n], arc_flow_dense [B][S-1][n_dst][n_src] (any may be NULL).  STATE if no
 * solve has run since create/churn. */
gwtf_status gwtf_flow_get_assignment(gwtf_flow_t h, int32_t* node_flow, int32_t* src_flow,
                                     int32_t* snk_flow, int32_t* arc_flow_dense);

/* Round state (DESIGN.md 2.3 encoding): up/down [B][S][n][max_cap] (>= 0 relay slot
 * gid*max_cap + j, -1 none, -2-k data-node slot k), src_down/snk_up [B][Mmax], kacc/deny
 * [B][S][n], quiet [B], round [B] (cumulative round counter).  Any may be NULL. */
gwtf_status gwtf_flow_export_round_state(gwtf_flow_t h, int32_t* up, int32_t* down, int32_t* src_down,
                                         int32_t* snk_up, int32_t* kacc, int32_t* deny, int32_t* quiet,
                                         int64_t* round);

/* Inverse of gwtf_flow_export_round_state (checkpoint / resume of the decentralized rounds,
 * SURVEY.md 5): installs a round state given in the export layouts (device pointers, or host
 * pointers with GWTF_HOST_PTRS; copied, the caller keeps ownership).  up/down/src_down/snk_up are
 * required; kacc/deny/quiet/round may be NULL (= 0).  The state is checked on the device: every
 * pointer must be answered by its target (pairing bijectivity), cross one stage
 * boundary (or reach the data node from stage 0 / S-1, slot index below the instance's supply),
 * and unusable slots (dead relay, j >= cap) must be FREE.  On a violation the round
 * state is reset to empty and GWTF_E_INVALID is returned.  Synchronizes the stream. */
gwtf_status gwtf_flow_import_round_state(gwtf_flow_t h, const int32_t* up, const int32_t* down,
                                         const int32_t* src_down, const int32_t* snk_up, const int32_t* kacc,
                                         const int32_t* deny, const int32_t* quiet, const int64_t* round);

/* Multi-data-node decentralized rounds, MC-SYNC (PAPER.md:203
 * "each data node ... must receive its own flow back", :249 "unpaired outflow", settings 5-6 of
 * :501-502).  Stateless: B instances sharing the relays and links of the single-commodity layout
 * (cap / alive [B][S][n], link_cost [B][S-1][n_dst][n_src]) with K data nodes each: src_cost /
 * snk_cost [K][B][n], supply [K][B] (int64, <= 2^20).  Runs the rounds from the empty state until
 * steady_window quiet rounds or max_rounds; every non-FREE slot carries its chain's data node, so
 * requests, grants, Change and self-pairing stay within one data node (K = 1 is
 * gwtf_flow_decentralized_rounds from an empty state).  Outputs (device, caller-owned): rounds_run
 * [B], dec_flow / dec_cost [K][B] (complete SRC_k -> SNK_k chains and their Eq. 2 cost), dangling
 * [B], round_digests [B][max_rounds] or NULL; the state arrays up / down / tag [B][S][n][max_cap] and
 * src_down / snk_up [B][K][Mmax] (all or none; data-node slot i of D_k = -2 - (k Mmax + i), Mmax =
 * max supply; tag -1 on FREE slots) receive the final state, and with resume != 0 they also give the
 * starting state (a valid tagged pairing, caller-checked; accepted-move and deny counters start at 0)
 * and round0 the RNG round counter to start from (0 from the empty state).
 * All device pointers on `stream` (a cudaStream_t); reads the supplies back (synchronizes).
 * INVALID on bad shapes or parameters, UNSUPPORTED when one instance's state exceeds 227 KB. */
gwtf_status gwtf_mc_rounds(int32_t B, int32_t S, int32_t n, int32_t max_cap, int32_t K, const int32_t* cap,
                           const uint8_t* alive, const int32_t* link_cost, const int32_t* src_cost,
                           const int32_t* snk_cost, const int64_t* supply, uint64_t seed, int64_t inst_base, double T0,
                           double alpha, int32_t objective, int32_t steady_window, int32_t deny_after,
                           int32_t max_rounds, int32_t* rounds_run, int64_t* dec_flow, int64_t* dec_cost,
                           int32_t* dangling, uint64_t* round_digests, int32_t* up, int32_t* down, int32_t* tag,
                           int32_t* src_down, int32_t* snk_up, int32_t resume, int64_t round0, void* stream);

/* Save / restore the handle's mutable state (masks, costs, round state) on the device,
 * e.g. to replay the same churn step several times in a benchmark. */
gwtf_status gwtf_flow_snapshot(gwtf_flow_t h);
gwtf_status gwtf_flow_restore(gwtf_flow_t h);

/* Per-kernel device time of the last calls when profiling is on (CUDA events on the
 * handle's stream): names[i] / ms[i] for up to cap kernels, *count set.  Profiling adds
 * an event pair around each kernel launch; off by default. */
gwtf_status gwtf_flow_set_profiling(gwtf_flow_t h, int32_t on);
gwtf_status gwtf_flow_kernel_times(gwtf_flow_t h, const char** names, float* ms, int32_t* launches,
                                   int32_t cap, int32_t* count);

/* SWARM-style greedy routing baseline (SPEC.md:199-207 greedy_route) on the
 * current (masked) graph of every instance: microbatches routed one at a time from the data node,
 * each hop to the alive next-stage client with spare capacity and a link, cheapest first, lowest
 * index on ties; the first microbatch that finds no successor (or no sink arc) stops the routing
 * (DESIGN.md 8c).  Outputs [B] (caller-owned, device or host per GWTF_HOST_PTRS): routed
 * microbatches and their total cost.  Does not touch the solver or round state. */
gwtf_status gwtf_flow_greedy_baseline(gwtf_flow_t h, int64_t* flow_value, int64_t* total_cost);

/* Warm-start rerouting after churn ("reroute" after a failure,
 * PAPER.md:274-288 crash handling), on the handle's current (churned) graph,
 * starting from a pre-churn assignment instead of zero flow.  Per instance:
 *   0. triage: when 4 x (units the churned graph can no longer carry) > the assignment's flow,
 *      re-routing would cost about as many searches as a cold solve; instances with fewer than
 *      4,096 links are cheaper to solve cold than to repair, and instances whose repair state
 *      exceeds 100 KB of shared memory (the cluster-tier shapes) are better served by the cold
 *      cluster tier: those are solved cold (the create flag GWTF_WARM_REPAIR_ALL skips the triage);
 *   1. otherwise the potential-carrying repair: potentials of the kept flow (Bellman-Ford), cut
 *      the units over capacity (crashed relay, relay over capacity, link / src / snk now
 *      GWTF_ABSENT), saturate the rejoined relays' shortcuts, route the excesses to the
 *      deficits, then resume successive shortest paths until F = M or no augmenting path is left;
 *   2. an instance whose repair stops (lowered costs, ranges) is solved cold as well.
 * The cold solves run the exact-solve kernels on that subset only.
 * node_flow [B][S][n], src_flow [B][n], snk_flow [B][n], arc_flow_dense [B][S-1][n_dst][n_src]
 * (the gwtf_flow_get_assignment layouts, taken before gwtf_flow_apply_churn) are read and
 * OVERWRITTEN in place with the repaired optimum.  Outputs [B]: max-flow value, min cost (equal
 * to a cold gwtf_flow_solve_batch's: the optimum's (F, cost) is unique; the assignment may
 * differ), stats [B][3] = {units cut, arcs saturated, repair iterations} for repaired instances
 * and {units cut, 0, augmentations} for cold-solved ones (may be NULL), inst_status (0 ok, else
 * the exact solve's status codes; may be NULL: then any nonzero status fails the call with
 * GWTF_E_STATE).  Does not touch the handle's own solver or round state.  INVALID on NULL
 * required arrays; UNSUPPORTED when 2(2n + Sn + (S-1)n^2) >= 2^24. */
gwtf_status gwtf_flow_warm_reroute(gwtf_flow_t h, int32_t* node_flow, int32_t* src_flow, int32_t* snk_flow,
                                   int32_t* arc_flow_dense, int64_t* flow_value, int64_t* total_cost,
                                   int64_t* stats, int32_t* inst_status);

/* Work counters of the exact solve accumulated since create (host int64 out[cap], cap <= 2048):
 * [0] dense boundary relaxations, [1] backward (reverse-arc) phases, [2] augmentations,
 * [3] Bellman-Ford passes, [4] traced path nodes (cluster tier), [11] frontier relaxations (cluster
 * tier), [12] instances gwtf_flow_warm_reroute solved cold, [13] instances re-solved with 64-bit
 * keys, [15] kernels launched by this handle (host count).  Synchronizes the stream. */
gwtf_status gwtf_flow_stats(gwtf_flow_t h, int64_t* out, int32_t cap);

/* Synchronizes the stream, frees everything.  NULL is a no-op. */
gwtf_status gwtf_flow_destroy(gwtf_flow_t h);

const char* gwtf_last_error(void);
int32_t gwtf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif
