/*
 * amp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference parplan hot path (candidate
 * enumeration, heuristic/shuffled placement, layer-time resolution, the
 * tolerance-indexed layer-partition DP, the cost estimate and the ranking
 * key).  It is the CPU checker for the CUDA engine: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * The product (paper_2210_07297_b200/libamp_search.so) never links it.
 *
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libparplan_ref.so, compiled from /root/reference sources by
 * oracle/Makefile) and the golden vectors under tests/golden/.
 */
#ifndef AMP_ORACLE_H
#define AMP_ORACLE_H

#include <stdint.h>

#include "../include/amp_search.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_ctx oracle_ctx;

oracle_ctx* oracle_create(const amp_problem* problem, uint64_t placements_per_class,
                          uint64_t seed);
void oracle_destroy(oracle_ctx* ctx);
uint64_t oracle_num_candidates(const oracle_ctx* ctx);
int32_t oracle_num_classes(const oracle_ctx* ctx);
int32_t oracle_max_pp(const oracle_ctx* ctx);
int oracle_class(const oracle_ctx* ctx, int32_t cls, int32_t* pp, int32_t* dp, int32_t* tmp,
                 int32_t* mbs);

/* LayerTimeResolver::layer_time; returns 0 on hit/fallback, 1 on miss. */
int oracle_layer_time(const oracle_ctx* ctx, int32_t layer, int32_t tmp, int32_t mbs,
                      double* out);

/* optimal_assignment core (pipeline_dp.cpp:70-149) with the EdgeCostFn
 * tabulated as edge_costs[q * L + cut].  Returns 0 ok, 1 invalid stage count
 * or gas.  Also reports the tolerance-domain size M and inner iterations. */
int oracle_optimal_assignment(const double* layer_times, int32_t L, int32_t stages, int32_t gas,
                              const double* edge_costs, int32_t* cuts, double* cost,
                              int32_t* domain_size, double* inner_iterations);

/* Tolerance domain (pipeline_dp.cpp:55-68); returns M, writes out[M]
 * (out must hold 1 + L(L+1)/2 doubles). */
int32_t oracle_tolerance_domain(const double* layer_times, int32_t L, double* out);

/* Placement of candidate `index` (rank -> device id, |D| entries). */
void oracle_placement(const oracle_ctx* ctx, uint64_t index, int32_t* rank_to_device);

/* evaluate_candidate (optimizer.cpp:141-176) for one candidate index. */
void oracle_evaluate(const oracle_ctx* ctx, uint64_t index, amp_record* rec, int32_t* cuts,
                     double* stage_times, double* edge_times);

/* Evaluate [begin, end) with `threads` pthreads (0 = 1). Vectors optional. */
void oracle_run(const oracle_ctx* ctx, uint64_t begin, uint64_t end, int32_t threads,
                amp_record* records, int32_t* cuts, double* stage_times, double* edge_times);

/* oracle_run with the DP memoised per worker by (class, boundary
 * bandwidths): the same records, cuts and times (SURVEY.md §8(d) full-N
 * memoised CPU oracle for large-N parity). */
void oracle_run_memo(const oracle_ctx* ctx, uint64_t begin, uint64_t end, int32_t threads,
                     amp_record* records, int32_t* cuts, double* stage_times, double* edge_times);

/* rank_records key (optimizer.cpp:178-196): writes the permutation that
 * sorts records by (failed, total, index). */
void oracle_rank(const amp_record* records, int64_t n, int64_t* order);

/* splitmix64. */
uint64_t oracle_splitmix64(uint64_t x);

#ifdef __cplusplus
}
#endif

#endif /* AMP_ORACLE_H */
