/*
 * amp_search.h — C ABI of the B200 strategy-search engine.
 *
 * Drop-in boundary for the batched candidate evaluation of AMP's planner
 * (reference `parplan`, arXiv 2210.07297).  The region this ABI replaces is
 * the worker pool + `evaluate_candidate` + `rank_records` inside
 * `parplan::plan` (reference proj/src/optimizer.cpp:200-231, declared at
 * proj/include/parplan/optimizer.hpp:74-75).  Everything around it
 * (config loading, the simulator run on the top `budget`, report writing)
 * stays host code in the caller.
 *
 * Conventions
 *   - Plain C: fixed-width integers, doubles, caller-owned pointers.  No C++
 *     exceptions and no torch types cross this boundary.
 *   - Every entry point returns AMP_OK (0) or a negative AMP_E_* status; the
 *     text is available from amp_search_last_error(ctx) (or
 *     amp_last_error() for context-free calls).
 *   - Per-candidate failures (pp > L, profile miss, parameter ceiling,
 *     invalid bandwidth) are DATA in amp_record.fail_code, never errors —
 *     matching the reference, which catches them per candidate into
 *     CandidateRecord.failure (optimizer.cpp:172-174).
 *   - Inputs are copied to the device at create time; the caller may free
 *     them afterwards.  Output buffers are caller-allocated host memory
 *     unless the function name ends in _device.
 *   - All floating-point results are bit-identical to the reference's
 *     IEEE-754 double arithmetic (no FMA contraction, same summation order).
 */
#ifndef AMP_SEARCH_H
#define AMP_SEARCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMP_SEARCH_ABI_VERSION 1

/* ---- status codes (returned) ------------------------------------------ */
#define AMP_OK 0
#define AMP_E_INVALID (-1)     /* bad argument / invalid problem            */
#define AMP_E_CUDA (-2)        /* CUDA runtime error                        */
#define AMP_E_OOM (-3)         /* device allocation failed                  */
#define AMP_E_UNSUPPORTED (-4) /* problem outside the supported envelope    */
#define AMP_E_NOT_BUILT (-5)   /* no sm_100a device / kernels unavailable   */
#define AMP_E_CANDIDATE (-6)   /* a strategy the search must evaluate failed
                                  (the reference throws there); the failing
                                  record is returned to the caller         */

/* ---- per-candidate failure codes (data) ------------------------------- */
/* Message texts the host rebuilds verbatim (reference file:line):          */
#define AMP_FAIL_NONE 0
/* "infeasible: pp = <pp> exceeds layer count <L>"  optimizer.cpp:149-152   */
#define AMP_FAIL_PP_GT_L 1
/* "profile miss: no entry for (layer=<l>, tmp=<tmp>, mbs=<mbs>) and
 *  analytic fallback is disabled"                    types.cpp:106-110     */
#define AMP_FAIL_PROFILE_MISS 2
/* "exceeds per-device parameter ceiling"            optimizer.cpp:165-167 */
#define AMP_FAIL_CEILING 3
/* "invalid p2p bandwidth <std::to_string(v)>"       cost_model.cpp:54-59  */
#define AMP_FAIL_P2P_BANDWIDTH 4
/* "invalid bandwidth <std::to_string(v)> in all-reduce group"
 *                                                   cost_model.cpp:47-50  */
#define AMP_FAIL_ALLREDUCE_BANDWIDTH 5

/* ---- problem description (SoA encoding of the reference inputs) ------- */
/*
 * ModelGraph   proj/include/parplan/types.hpp:41-54
 * Cluster      types.hpp:67-79 (diagonal is the +inf self-transfer sentinel;
 *              the value passed on the diagonal is ignored)
 * ProfileTable types.hpp:91-100, given as an entry list; later duplicates
 *              overwrite earlier ones exactly like ProfileTable::set.
 * CostModelOptions cost_model.hpp:41-52; PlanOptions optimizer.hpp:56-63.
 */
typedef struct amp_problem {
  int32_t n_layers;                  /* L >= 1                               */
  int32_t n_devices;                 /* |D| >= 1                             */
  int32_t gbs;                       /* global batch size >= 1               */
  int32_t fallback_enabled;          /* AnalyticFallback.enabled             */
  const double* param_count;         /* [L] LayerSpec.param_count            */
  const double* flops_per_sample;    /* [L] value when flops_present[l] != 0 */
  const uint8_t* flops_present;      /* [L] std::optional engaged? (NULL=none) */
  const double* activation_volumes;  /* [L-1] bytes per sample, i -> i+1     */
  const int32_t* node_id;            /* [|D|] node of device id d            */
  const double* bandwidth;           /* [|D|*|D|] row-major bytes/s          */
  int64_t n_profile_entries;
  const int32_t* profile_layer;      /* [n_profile_entries]                  */
  const int32_t* profile_tmp;
  const int32_t* profile_mbs;
  const double* profile_seconds;
  double bytes_per_param;            /* CostModelOptions.bytes_per_param     */
  double fallback_device_flops;      /* AnalyticFallback.device_flops        */
  double fallback_tmp_bandwidth;     /* AnalyticFallback.tmp_bandwidth       */
  int32_t has_max_params_per_device; /* PlanOptions.max_params_per_device ?  */
  int32_t reserved0;
  double max_params_per_device;
} amp_problem;

/*
 * Candidate space.  Candidates are the reference plan() list
 * (optimizer.cpp:202-207: pp asc, dp asc, tmp = |D|/(pp*dp), mbs in
 * divisors(gbs/dp) asc) — the "classes" — crossed with P placements per
 * class in class-major order: index = class * P + p.
 *   p == 0 : the reference heuristic placement (placement.cpp:27-66);
 *   p >= 1 : the heuristic device order shuffled by Fisher-Yates driven by
 *            splitmix64(seed ^ p).
 * With P == 1 the space is exactly the reference plan() space and index
 * order equals the reference ranking tie-break key (pp, dp, tmp, mbs).
 */
/* amp_search_config.flags */
/* Evaluate the reference's full tolerance-indexed DP table instead of only
 * the cells the result depends on (same results; for comparison).          */
#define AMP_FLAG_DENSE_DP 1
/* Solve one DP per candidate even when candidates share a signature (class,
 * per-boundary bandwidth codes).  By default the engine memoises the DP by
 * signature (exact: optimal_assignment is a pure function of it; SURVEY
 * §8(d)); this flag is for comparison runs.                                 */
#define AMP_FLAG_NO_DEDUP 2

typedef struct amp_search_config {
  uint64_t placements_per_class; /* P >= 1                                 */
  uint64_t seed;                 /* shuffle seed                            */
  int32_t device;                /* CUDA device ordinal                     */
  int32_t max_ctas;              /* 0 = auto (resident CTAs on all SMs)     */
  int32_t flags;                 /* AMP_FLAG_*                              */
  int32_t n_gpus;                /* 0 / 1: one GPU; n > 1: devices device ..
                                    device+n-1 driven by this one context
                                    (a thread per GPU, NCCL all-gather of
                                    the per-GPU top-k): amp_search_run
                                    shards its range with the LPT plan of
                                    amp_search_run_device_shard; the other
                                    entry points use the first device       */
} amp_search_config;

/* One evaluated candidate: CandidateRecord minus the vectors
 * (optimizer.hpp:48-54; CostBreakdown types.hpp:155-161). 64 bytes.       */
typedef struct amp_record {
  uint64_t index;         /* candidate index (class * P + p)                */
  double total;           /* CostBreakdown.total                            */
  double pipeline_time;   /* CostBreakdown.pipeline_time                    */
  double dpsync_time;     /* CostBreakdown.dpsync_time                      */
  int32_t pp, dp, tmp, mbs;
  int32_t fail_code;      /* AMP_FAIL_*                                     */
  int32_t fail_layer;     /* PROFILE_MISS: first missing layer              */
  double fail_value;      /* *_BANDWIDTH: offending bandwidth value         */
} amp_record;

/* Optional per-candidate vectors; strides from amp_search_max_pp():
 *   cuts        [n * (max_pp + 1)]  LayerAssignment.cut_boundaries
 *   stage_times [n * max_pp]        CostBreakdown.per_stage_times
 *   edge_times  [n * max_pp]        CostBreakdown.per_edge_times (pp-1 used)
 *   placement   [n * |D|]           Placement::flat() (rank -> device id)
 * Unused tail entries are set to -1 / NaN.  Any pointer may be NULL.     */
typedef struct amp_details {
  int32_t* cuts;
  double* stage_times;
  double* edge_times;
  int32_t* placement;
  double* simulated;   /* [n] simulate() iteration time (simulator.cpp:140-198),
                          NaN for failed candidates; runs the batched
                          simulator on the device      */
} amp_details;

/* Counters of the last amp_search_run* call (roofline accounting). */
typedef struct amp_stats {
  double kernel_ms;          /* device time of the evaluate kernel          */
  double total_ms;           /* device time of the whole run incl. top-k    */
  double dp_cells;           /* (i, j, m) DP cells computed                 */
  double dp_inner;           /* (i, j, m, cut) inner iterations executed    */
  double dp_inner_lt;        /* of which on the m < seg(cut,i) branch       */
  double fp64_ops;           /* algorithmic FP64 ops     */
  double bytes;              /* algorithmic HBM bytes                        */
  uint64_t candidates;       /* candidates evaluated                         */
  uint64_t dp_instances;     /* DP instances solved                          */
  int32_t launches;          /* kernels launched by the run                  */
  int32_t ctas;              /* CTAs of the DP kernel                        */
  double place_ms;           /* device time of K_place (all chunks)          */
  double dp_ms;              /* device time of K_dp (all chunks)             */
  double est_ms;             /* device time of K_est (all chunks)            */
  uint64_t dp_items;         /* candidates that went through K_dp (pp >= 3)  */
  int32_t dp_launches;       /* K_dp launches of the run                     */
  int32_t dp_group;          /* K_dp candidates per group (0: one at a time) */
  double dp_stage_ms;        /* device time of the DP stage kernels alone
                                (K_trie_tiles launches; CUDA events)        */
  int32_t dp_stage_launches; /* their launches                               */
  int32_t dp_fallback;       /* chunks whose trie capacity overflowed (their
                                signatures went through the per-signature
                                K_dp instead)                               */
} amp_stats;

typedef struct amp_ctx amp_ctx;

/* ---- context lifecycle ------------------------------------------------- */
int amp_search_create(amp_ctx** out, const amp_problem* problem,
                      const amp_search_config* config);
void amp_search_destroy(amp_ctx* ctx);
const char* amp_search_last_error(const amp_ctx* ctx);
/* Thread-local text of the last failed context-free call (create, dp). */
const char* amp_last_error(void);
int amp_search_abi_version(void);

/* ---- candidate space queries (host, no device work) -------------------- */
uint64_t amp_search_num_candidates(const amp_ctx* ctx);
int32_t amp_search_num_classes(const amp_ctx* ctx);
int32_t amp_search_max_pp(const amp_ctx* ctx);
int amp_search_class(const amp_ctx* ctx, int32_t cls, int32_t* pp, int32_t* dp,
                     int32_t* tmp, int32_t* mbs);
/* Work-weighted split of [0, num_candidates) into n_parts contiguous
 * ranges (bounds[n_parts + 1]); equal cumulative DP inner iterations.     */
int amp_search_partition(const amp_ctx* ctx, int32_t n_parts, uint64_t* bounds);

/* ---- evaluation --------------------------------------------------------- */
/* Evaluate candidates [begin, end).  Writes the k best under the key
 * (failed, total, index) — the reference rank_records order
 * (optimizer.cpp:178-196) — to topk[0 .. *n_topk).  If `all` is non-NULL
 * it receives every record in index order ([end - begin]); `all_details`
 * (nullable) the per-candidate vectors.  Host buffers.                    */
int amp_search_run(amp_ctx* ctx, uint64_t begin, uint64_t end, int32_t k,
                   amp_record* topk, int32_t* n_topk, amp_record* all,
                   const amp_details* all_details);

/* Re-evaluate an explicit list of candidate indices (e.g. the merged
 * global top-k) with full details.  Host buffers.                         */
int amp_search_evaluate(amp_ctx* ctx, const uint64_t* indices, int32_t n,
                        amp_record* out, const amp_details* details);

/* Device-resident variant for multi-GPU: writes exactly k records
 * (padded with fail_code = -1, index = UINT64_MAX) to device memory
 * d_topk on `stream` (cudaStream_t, NULL = legacy default stream).  No
 * host synchronisation.                                                   */
/* Estimate only (K_place -> K_est, no DP): candidates `indices` with the
 * caller's layer cuts cuts[i * (max_pp + 1) + 0 .. pp] (0 = c_0 < ... <
 * c_pp = n_layers).  The Megatron baseline path (optimizer.cpp:253-279:
 * uniform / parameter-balanced cuts through estimate(),
 * cost_model.cpp:176-212).  Host buffers, records in input order.          */
int amp_search_estimate(amp_ctx* ctx, const uint64_t* indices, const int32_t* cuts, int32_t n,
                        amp_record* out, const amp_details* details);
/* Evaluate caller placements: candidate i is class classes[i] with the
 * placement placements[i * |D| .. +|D|) (rank -> device id, a permutation)
 * instead of one of the P generated ones; with cuts == NULL the layer
 * partition is solved (DP), else the caller's cuts are estimated.  Used by
 * the annealing search (its domino-tiling proposals, placement.cpp:299-398)
 * and by any caller with its own placements.  Host buffers.                */
int amp_search_evaluate_placed(amp_ctx* ctx, const int32_t* classes, const int32_t* placements,
                               const int32_t* cuts, int32_t n, amp_record* out,
                               const amp_details* details);
int amp_search_run_device(amp_ctx* ctx, uint64_t begin, uint64_t end, int32_t k,
                          amp_record* d_topk, void* stream);
/* Shard `shard` of n_shards (multi-GPU; replaces the worker split of
 * optimizer.cpp:212-229 across GPUs): every class is cut into min(P, n)
 * contiguous placement blocks weighted by its work, and the blocks go
 * longest-first to the least-loaded shard (deterministic).  With P >= n all
 * shards carry the same class mix; with P = 1 (plan()) it is an LPT split
 * of the uneven DP instances.  The union over shards is the whole space and
 * the merged top-k equals the single-GPU one.  Device-resident like
 * amp_search_run_device.                                                  */
int amp_search_run_device_shard(amp_ctx* ctx, int32_t shard, int32_t n_shards, int32_t k,
                                amp_record* d_topk, void* stream);
/* Candidates in shard `shard` of n_shards. */
uint64_t amp_search_shard_size(const amp_ctx* ctx, int32_t shard, int32_t n_shards);
/* The shard's index ranges [ranges[2i], ranges[2i+1]) in its dispatch
 * order; *n_ranges = their number (ranges may be NULL to query it).      */
int amp_search_shard_ranges(const amp_ctx* ctx, int32_t shard, int32_t n_shards, uint64_t* ranges,
                            int32_t cap, int32_t* n_ranges);

/* Merge n_in device records — n_in / k lists of k records, each sorted by
 * the ranking key and padded at its end (e.g. the all-gathered per-GPU
 * outputs of amp_search_run_device), at most 1024 lists — into the k best
 * under the ranking key; deterministic.                                   */
int amp_search_merge_topk_device(amp_ctx* ctx, const amp_record* d_in, int32_t n_in,
                                 int32_t k, amp_record* d_out, void* stream);

int amp_search_last_stats(const amp_ctx* ctx, amp_stats* out);

/* ---- annealing search (placement.cpp:299-398, Algorithm 2) ------------ */
typedef struct amp_anneal_config {
  int32_t iterations;          /* >= 1                                      */
  int32_t budget;              /* top strategies ranked                     */
  uint64_t seed;               /* std::mt19937_64 seed                      */
  double initial_temperature;  /* reference default 1.0                     */
  double cooling;              /* 0.97                                      */
  double min_temperature;      /* 1e-3                                      */
  int32_t record_all;          /* record rejected evaluated states too      */
  int32_t neighbor_retries;    /* 20                                        */
} amp_anneal_config;

typedef struct amp_anneal_entry {
  amp_record estimated;        /* degrees, mbs, total / pipeline / dpsync    */
  int32_t iteration;           /* 0 = initial state                          */
  int32_t accepted;
  int32_t reserved[2];
} amp_anneal_entry;

/* The reference's annealing chain, bit for bit (same mt19937_64 draws,
 * domino tilings, temperatures and acceptances), with every proposal's DP
 * and estimate evaluated on the GPU (amp_search_evaluate_placed).  `record`
 * receives the recorded states in visit order ([cap]; cap >= iterations+1
 * always suffices), record_place [cap][|D|] and record_cuts
 * [cap][max_pp + 1] their placements and cuts (nullable); top[budget] the
 * record indices of the best `budget` states by (total, pp, dp, tmp, mbs)
 * (the reference's std::sort).  AMP_E_CANDIDATE: a strategy failed to
 * evaluate (profile miss ...) — the reference aborts there; `failed`
 * (nullable) receives its record.  The problem must be the one the context
 * was created from.                                                        */
int amp_search_anneal(amp_ctx* ctx, const amp_problem* problem, const amp_anneal_config* cfg,
                      amp_anneal_entry* record, int32_t* record_place, int32_t* record_cuts,
                      int32_t cap, int32_t* n_record, int32_t* top, int32_t* n_top,
                      double* initial_cost, amp_record* failed);

/* ---- standalone layer-partition DP (pipeline_dp.cpp:70-149) ----------- */
/* One instance: SegmentTimes over layer_times[L], `stages` stages, gas,
 * and EdgeCostFn tabulated as edge_costs[q * L + cut] for q in
 * [0, stages-1), cut in [1, L-1] (entry cut = 0 unused).                  */
typedef struct amp_dp_instance {
  int32_t n_layers;
  int32_t stages;
  int32_t gas;
  int32_t reserved;
  const double* layer_times;
  const double* edge_costs;
} amp_dp_instance;

/* Solve n instances on `device`.  cuts_out[n * cut_stride] receives
 * cut_boundaries (stages + 1 entries), cost_out[n] the DP cost
 * (AssignmentResult.cost).  Invalid instances (stages < 1, stages > L,
 * gas < 1) are reported per instance via status_out[n] (0 ok, 1 invalid),
 * mirroring the ValidationError of check_stage_count
 * (pipeline_dp.cpp:22-30).                                                */
int amp_dp_solve_batch(int32_t device, const amp_dp_instance* instances, int32_t n,
                       int32_t* cuts_out, int32_t cut_stride, double* cost_out,
                       int32_t* status_out);

/* Measured FP64 add throughput of `device` (DADD instructions/s over all
 * SMs), for the roofline denominator.                                     */
int amp_fp64_peak(int32_t device, double* dadd_per_s, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* AMP_SEARCH_H */
