// Internal declarations shared by the host API (gwtf_api.cpp) and the kernels (*.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

namespace gwtf {

constexpr int32_t kAbsent = INT32_MAX;
constexpr int kHopBits = 20;                 // packed key = cost << 20 | hops
constexpr uint64_t kKeyInf = ~0ull;
constexpr int32_t kNone = -1;                // round-state pointer encoding

// Everything a kernel needs about a batch; all pointers are device pointers owned by the handle.
struct Problem {
  int32_t B, S, n, ld, MC;     // ld = row stride of the padded tiles (n rounded up to 4)
  int64_t Mmax;                // max supply over the batch (SRC/SNK slot arrays)
  int32_t Lcap;                // positive-arc list capacity per boundary
  int32_t* tile;               // [B][S-1][n][ld] dest-major, padding = kAbsent
  uint16_t* tile16;            // cluster tier: [B][S-1][n][ld16] copy of tile, t16code = absent/padding
                               // (nullptr when some cost >= t16code or the tier is unused)
  int32_t ld16;                // n rounded up to 8
  uint8_t* tile8;              // cluster tier: [B][S-1][n][ld8] 8-bit copy when every arc is present and
                               // every cost < 255 (255 = padding); nullptr otherwise (or once retired)
  int32_t ld8;                 // n rounded up to 16
  uint8_t* tile8t;             // the same 8-bit costs source-major, [B][S-1][n_src][ld8] (frontier columns)
  int32_t t16code;             // T32 of the cluster tier's 32-bit keys (ssp_cluster.cu), < 2^16
  uint16_t* tile16s;           // shared-memory tier: [B][stride] 16-bit copy of the padded tiles (padding 0) when
                               // every arc is present with a cost < 65535; nullptr otherwise (or once retired)
  int64_t tile16s_stride;      // elements per instance (bytes a multiple of 16: one TMA bulk copy)
  uint8_t* tile8s;             // shared-memory tier: [B][stride] 8-bit copy (absent 0xFF, padding 0) when every
                               // finite cost is < 255; nullptr otherwise (or once retired)
  int64_t tile8s_stride;       // bytes per instance (a multiple of 16)
  int32_t* src;                // [B][n]
  int32_t* snk;                // [B][n]
  int32_t* cap;                // [B][S][n]
  uint8_t* alive;              // [B][S][n]
  uint8_t* alive_prev;         // [B][S][n] the mask before the last apply_churn (warm reroute: rejoined relays)
  int64_t* supply;             // [B]
  // exact-solve state (persistent for get_assignment)
  int32_t* g;                  // [B][S][n]
  int32_t* src_f;              // [B][n]
  int32_t* snk_f;              // [B][n]
  uint32_t* arcs;              // [B][S-1][Lcap]  (u << 20 | v << 8 | f)
  int32_t* arc_cnt;            // [B][S-1]
  int32_t* arcw;               // cluster tier: [B][S-1][Lcap] weight of each list entry
  // round state
  int32_t* up;                 // [B][S*n*MC]
  int32_t* down;               // [B][S*n*MC]
  int32_t* src_down;           // [B][Mmax]
  int32_t* snk_up;             // [B][Mmax]
  int32_t* kacc;               // [B][S*n]
  int32_t* deny;               // [B][S*n]
  int32_t* quiet;              // [B]
  int64_t* round;              // [B]
  // per-team scratch of the rounds kernel when the instance does not fit in shared memory
  uint8_t* ws_rounds;
  int32_t ws_rounds_teams;
  int32_t rounds_cost_mode;    // R0 strategy: 0 stage-synchronous, 1 chain walk per slot, 2 per relay
  // parameters of the rounds
  uint64_t seed;
  int64_t inst_base;
  int32_t objective, W, deny_after;
  const uint32_t* thr;         // [(K+1)][width]
  int32_t thr_width, thr_K;
  // persistent work queue counters: [0] ssp queue, [1] rounds queue, [2] redo count, [3] redo queue
  int32_t* counters;           // [8]
  int32_t* redo;               // [B] instances re-solved with 64-bit keys (32-bit key overflow guard)
  // work counters of the exact solve (gwtf_flow_stats): relax steps, backward phases,
  // augmentations, Bellman-Ford passes, traced path nodes
  unsigned long long* stats;   // [8]
  int32_t hbits;               // hop bits of the 32-bit packed keys; 0 = 64-bit keys only
  // cluster tier (instances too large for shared memory): cluster size and per-cluster path scratch
  int32_t cluster_size;        // 0 = cluster tier unavailable
  int32_t rounds_cluster_pref; // rounds cluster size chosen by the caller (0: by the cost model)
  uint8_t* ws_cluster;
  int32_t ws_cluster_slots;
  int32_t debug;               // GWTF_DEBUG_FLAGS (testing)
  // exact solve of a subset: the queue hands out sel[0 .. *sel_count) instead of 0 .. B (nullptr: all)
  const int32_t* sel;
  const int32_t* sel_count;
  // global workspace for teams whose instance does not fit in shared memory
  uint8_t* ws;
  size_t ws_per_team;
  int32_t ws_teams;
};

struct SspOut {
  int64_t* F; int64_t* cost; int32_t* A; int32_t* status;
};

struct RoundsOut {
  int32_t max_rounds;
  int32_t* rounds_run; int64_t* F_dec; int64_t* cost_dec; int32_t* dangling; uint64_t* digests;
};

// launchers (return cudaGetLastError())
size_t ssp_smem_bytes(const Problem& P);
size_t ssp_global_ws_bytes(const Problem& P);
size_t rounds_ws_bytes(const Problem& P, bool smem);
int rounds_tpi(const Problem& P);
bool rounds_use_smem(const Problem& P);
// tier: 0 automatic (shared memory, else cluster, else global), 1 force global, 2 force cluster
cudaError_t launch_ssp(const Problem& P, const SspOut& o, cudaStream_t st, int num_sms, int force_tier);
int ssp_launch_count(const Problem& P, int force_tier);  // kernels launch_ssp issues
size_t ssp_cluster_smem_bytes(const Problem& P, int C);
int ssp_cluster_size(const Problem& P);
cudaError_t launch_ssp_cluster(const Problem& P, const SspOut& o, cudaStream_t st, int C);
cudaError_t launch_rounds(const Problem& P, const RoundsOut& o, cudaStream_t st, int num_sms);
cudaError_t launch_init_round_state(const Problem& P, cudaStream_t st);
cudaError_t launch_import_check(const Problem& P, int32_t* bad, cudaStream_t st);
cudaError_t launch_churn(const Problem& P, const uint8_t* alive_new, const int32_t* upd, int64_t k,
                         int32_t* bad_flag, cudaStream_t st);
cudaError_t launch_pad_tiles(const Problem& P, const int32_t* link, cudaStream_t st);
cudaError_t launch_pack_tile16(const Problem& P, cudaStream_t st);
cudaError_t launch_pack_tile16s(const Problem& P, int32_t* bad, cudaStream_t st);
cudaError_t launch_pack_tile8s(const Problem& P, int32_t* bad, cudaStream_t st);
cudaError_t launch_pack_tile8(const Problem& P, int32_t* bad, cudaStream_t st);
cudaError_t launch_dense_arcs(const Problem& P, int32_t* dense, cudaStream_t st);
cudaError_t launch_residual_caps(const Problem& P, int32_t* out, cudaStream_t st);
cudaError_t launch_eq1(int32_t B, int32_t S, int32_t n, int32_t L, const int32_t* comp, const int32_t* loc,
                       const int32_t* dloc, const int32_t* lat, const int32_t* bw, int64_t size_kbit,
                       int32_t* src, int32_t* snk, int32_t* link, cudaStream_t st);
cudaError_t launch_addition_build(int32_t S, int32_t n, const int32_t* cap, const int32_t* src, const int32_t* snk,
                                  const int32_t* link, const int32_t* ccap, const int32_t* cin, const int32_t* cout,
                                  const int32_t* ccc, int64_t first, int64_t count, int32_t* cap_o, int32_t* src_o,
                                  int32_t* snk_o, int32_t* link_o, cudaStream_t st);
cudaError_t launch_addition_select(int64_t count, const int64_t* F, const int64_t* cost, int64_t* best, cudaStream_t st);
cudaError_t launch_greedy(const Problem& P, int32_t* rem, int64_t* F, int64_t* cost, cudaStream_t st);
// multi-data-node rounds (mc_rounds.cu): one stateless call over a batch
struct McRoundsCall {
  int32_t B, S, n, MC, K, Mmax;
  const int32_t* cap; const uint8_t* alive; const int32_t* tile; int32_t ld;
  const int32_t* src; const int32_t* snk; const int64_t* supply;
  uint64_t seed; int64_t inst_base; int32_t objective, W, deny_after, max_rounds;
  const uint32_t* thr; int32_t thr_width, thr_K;
  int32_t* rounds_run; int64_t* F_dec; int64_t* cost_dec; int32_t* dangling; uint64_t* digests;
  int32_t *up_out, *down_out, *tag_out, *sd_out, *su_out;
  int32_t resume;
  int64_t round0;
};
size_t mc_rounds_smem(int S, int n, int MC, int K, int Mmax);
cudaError_t launch_mc_rounds(const McRoundsCall& c, cudaStream_t st, int num_sms);
size_t warm_ws_bytes(const Problem& P, int grid);
int warm_grid(const Problem& P);
cudaError_t launch_warm_collect(int32_t B, int32_t* status, int32_t* sel, int32_t* sel_count, unsigned long long* ctr,
                                cudaStream_t st);
cudaError_t launch_warm_dense(const Problem& P2, const int32_t* sel, const int32_t* sel_count, int32_t* dense,
                              const int32_t* aug, int64_t* stats, cudaStream_t st);
cudaError_t launch_warm(const Problem& P, int32_t* src_f, int32_t* g, int32_t* arc, int32_t* snk_f, void* ws,
                        int64_t* F, int64_t* cost, int64_t* stats, int32_t* status, bool repair_all, cudaStream_t st);
cudaError_t launch_scan_costs(const int32_t* v, int64_t count, int32_t* out_max, int32_t* out_min,
                              cudaStream_t st);

}  // namespace gwtf
