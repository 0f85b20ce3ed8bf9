// amp_common.cuh — device-side data layout shared by the kernels.
//
// HBM layout (all written once at amp_search_create, read-only afterwards):
//   PairDev[n_pairs]        one entry per distinct (tmp, mbs): the layer
//                           times, prefix sums, tolerance domain and segment
//                           index of SegmentTimes/tolerance_domain
//                           (reference pipeline_dp.cpp:39-91), built once
//                           per pair instead of once per candidate.
//   ClassDev[n_cls]         plan() candidate list (optimizer.cpp:202-207)
//                           with gas and the pair it uses.
//   times   [n_pairs][L]    f64 layer times (LayerTimeResolver, cost_model.cpp:74-86)
//   prefix  [n_pairs][L+1]  f64 prefix sums, left-to-right
//   domain  [n_pairs][nv]   f64 sorted unique segment sums (M valid)
//   seg     [n_pairs][(L+1)^2] u16 lower_bound index of prefix[b]-prefix[a]
//   bw      [|D|][|D|]      f64 link bandwidth, +inf diagonal
#pragma once

#include <stdint.h>

#include "../../include/amp_search.h"

namespace amp {

// Bounds assertions of the debug build (make lib EXTRA=-DAMP_BOUNDS): a
// failing check prints its site and traps.  compute-sanitizer is not
// available on the GPU pool; tools/gpu_bounds.sh runs the GPU tests on this
// build instead.
#ifdef AMP_BOUNDS
#define AMP_CHECK(cond, what)                                                      \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      printf("AMP_BOUNDS %s:%d %s (block %d thread %d)\n", __FILE__, __LINE__, what, \
             (int)blockIdx.x, (int)threadIdx.x);                                   \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define AMP_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

constexpr int kMaxLayers = 180;        // (L(L+1)/2 + 1) <= 16384 for the smem sort
constexpr int kSortCap = 16384;        // padded domain capacity (pow2)
constexpr int kEvalThreads = 384;      // evaluate kernel max block size

struct PairDev {
  int32_t tmp, mbs;
  int32_t M;            // tolerance domain size
  int32_t fail_code;    // AMP_FAIL_PROFILE_MISS / _ALLREDUCE_BANDWIDTH / 0
  int32_t fail_layer;   // first failing layer (segment_times order)
  int32_t monotone;     // all layer times >= 0 (DP split-loop fast path)
  double fail_value;
};

struct ClassDev {
  int32_t pp, dp, tmp, mbs;
  int32_t gas, pair;
  int32_t crow;  // row of the class's shape in the code table (EvalParams::ctab), -1: none
  int32_t pad1;
};

// Contiguous run of candidate indices of one class, handed out
// heaviest-class-first by the persistent evaluate kernel.
struct Segment {
  uint64_t first;   // first candidate index
  uint64_t count;   // number of candidates
  uint64_t offset;  // exclusive prefix of counts in dispatch order
  uint64_t out;     // position of `first` in the caller's output order
  uint64_t p0;      // placement index of `first` within its class
  int64_t cls;      // class of the whole segment
};

struct WEnt;     // per-stage cut table entry (amp_kernels.cuh)
struct ProgDev;  // pruned-DP program (amp_dp_sparse.cuh)
struct CandWork; // per-candidate pipeline record (amp_pipeline.cuh)

struct EvalParams {
  // problem
  int32_t L, D, gbs, max_pp;
  uint64_t P, seed;
  const double* param;      // [L]
  const double* act;        // [L-1]
  const double* bw;         // [D*D]
  const int32_t* base_order;  // [D] heuristic device order
  int32_t has_ceiling;
  int32_t n_pairs;
  double ceiling;
  double bpp;
  // tables
  const ClassDev* cls;
  const PairDev* pairs;
  const double* times;
  const double* prefix;
  const double* domain;
  const uint16_t* seg;
  int32_t nv_stride;        // domain stride per pair
  int32_t slice_in_smem;    // 1: DP stage slice in shared memory
  int32_t w_in_smem;        // 1: per-stage cut table in shared memory
  int32_t pad1;
  // work list
  const Segment* segs;
  int32_t n_segs;
  int32_t pad0;
  uint64_t n_work;
  int32_t chunk;               // work items taken per atomic fetch
  int32_t pad2;
  const uint64_t* index_list;  // explicit indices (evaluate) or NULL
  unsigned long long* counter;
  // scratch (per CTA)
  uint8_t* bp;              // backpointers, bp_stride bytes per CTA
  uint64_t bp_stride;
  double* slice;            // global stage slice when !slice_in_smem
  WEnt* wtab;               // global cut tables when !w_in_smem
  uint64_t slice_stride;    // doubles per CTA
  int32_t* place;           // placement, D per CTA
  // outputs
  amp_record* all;          // [n_work] in output order, or NULL
  int32_t* all_cuts;        // [n_work * (max_pp+1)]
  double* all_stage;        // [n_work * max_pp]
  double* all_edge;         // [n_work * max_pp]
  int32_t* all_place;       // [n_work * D]
  amp_record* cta_topk;     // [gridDim.x * k]
  int32_t k;
  int32_t max_M;
  // pruned DP (amp_dp_sparse.cuh)
  const ProgDev* progs;
  const int32_t* class_prog;  // [n_cls] program of each class
  const uint32_t* cells;
  const uint32_t* cellpred;
  const uint16_t* preds;
  const uint32_t* stage;
  double* vbuf;               // global value arrays when not in smem
  // pipeline chunk: work items [t0, t0 + n_chunk) of the run
  uint64_t t0;
  uint64_t n_chunk;
  CandWork* work;             // [n_chunk]
  int32_t* placeb;            // [n_chunk][D] rank -> device
  double* bwqb;               // [n_chunk][max_pp] stage-boundary bandwidths
  uint8_t* cutsb;             // [n_chunk][max_pp + 1]
  int32_t first_chunk;        // K_est: start CTA top-k lists empty
  int32_t pad3;
  int32_t max_cells;          // max_j |N_j| over programs
  int32_t max_prog_cells;     // max sum_j |N_j| over programs
  // K_dp multi (amp_dp_multi.cuh)
  int32_t max_n1;             // max |N_1|
  int32_t max_v;              // max_{j >= 2} |N_j|
  int32_t max_rest;           // max sum_{j >= 2} |N_j| (backpointer bytes per candidate)
  int32_t n_codes;            // distinct link bandwidths (0: codes disabled)
  const uint8_t* bwcode;      // [D*D] rank of each link's bandwidth among bwval, or NULL
  const double* bwval;        // [n_codes] distinct bandwidths, ascending
  const double* qtab;         // [n_cls][n_codes][L] edge cost act[c-1]*mbs / bwval[code]
  uint8_t* bwcb;              // [n_chunk][max_pp] stage-boundary bandwidth codes
  const uint2* cellrec;       // [cells] {cell, cellpred} (K_dp multi)
  uint64_t n_dp;              // chunk items [0, n_dp) may need K_dp (pp >= 3 first)
  int32_t cuts_given;         // 1: cutsb holds caller cuts for every item (estimate only)
  int32_t pad5;
  double* all_sim;            // [n_work] simulated iteration time (simulator.cpp:140-198) or NULL
  double* simbuf;             // per-warp scratch [gbs] for the pp > 32 simulation path
  // DP memoisation by signature (amp_dedup.cuh); NULL when off
  const uint32_t* rep_list;   // [n_rep] chunk items whose DP K_dp solves
  const uint32_t* rep_of;     // [n_dp] representative of every heavy item
  const uint64_t* n_rep;      // device count of representatives
  const double* prog_inner;   // [n_progs] unpadded inner iterations per program
  unsigned long long* exec_counters;  // [2]: DP instances solved, inner iterations executed
  const int32_t* given_place;  // [n_work][D] caller placements (rank -> device) or NULL
  // thread-mode traffic trims (amp_thread.cuh)
  uint64_t* placep;           // [n_chunk] placement as 16 x 4-bit nibbles, or NULL
  int32_t need_place_rows;    // K_place must also write placeb (warp K_est reads it)
  int32_t need_bwq;           // K_place must also write bwqb (kernels without edge tables)
  const uint8_t* cut2tab;     // [n_cls][n_codes] cut of the 2-stage DP (pp == 2 classes) or NULL
  int32_t n_cls_total;        // classes in the plan() list
  int32_t pad6;
  // stage_time / params_in_range over every layer range [a, b), summed from
  // 0.0 in layer order (the reference's loops, tabulated once per context)
  const double* rsum_t;       // [n_pairs][(L+1)^2] layer-time range sums, or NULL
  const double* rsum_p;       // [(L+1)^2] parameter range sums
  uint8_t* repcuts;           // [n_rep][max_pp + 1] cuts per signature run (memoised runs)
  int32_t bw_positive;        // every link bandwidth > 0 (coded): no all-reduce group can fail
  int32_t fuse_light;         // thread K_est places items [n_dp, n_chunk) itself (pp <= 2)
  uint64_t* sigkey;           // [n_chunk] DP signature key written by K_place_t, or NULL
  int32_t sig_code_bits;      // bits per boundary code in the key
  int32_t est_fast;           // K_est_t uses the unrolled shape kernels (amp_thread.cuh est_shape)
  int32_t need_bwcb;          // K_place stores the boundary codes (bwcb)
  int32_t fuse_hash;          // K_place_t inserts the signature keys itself (amp_dedup.cuh)
  // the signature hash table of this chunk (fuse_hash; see HashParams)
  unsigned long long* h_tkey;
  uint32_t* h_tval;
  uint32_t* h_slot_of;
  uint32_t* h_uniq;
  unsigned long long* h_nuniq;
  uint64_t h_mask, h_epoch, h_max_probe;
  int32_t h_eshift, pad10;
  // K_est shape kernels: signature run of item u = run_of_slot[run_slot[u]]
  // (the hash table after k_hash_runs) instead of the scattered rep_of[u]
  const uint32_t* run_slot;
  const uint32_t* run_of_slot;
  // per signature run of a dp == 1, pp >= 3 class: its pipeline time (the
  // whole estimate: one replica, no dpsync; NaN = parameter ceiling fails)
  const double* run_pipe;
  // K_place_t writes no work records: the shape K_est re-decodes its items
  // (nothing else reads them with the memoised DP and the fused hash insert)
  int32_t skip_work, pad11;
  // signature-mode K_dp (amp_dp_multi.cuh): the chunk's distinct signature
  // keys [*n_rep]; run only while *sig_guard != 0 (NULL: always)
  const uint64_t* sig_keys;
  const uint32_t* sig_guard;
  // gangs (k_dp<kSparseG>): each DP instance whose program has >= gang_min
  // inner iterations is solved by G CTAs (stage cells split G ways, one
  // cross-CTA barrier per stage); listed by k_gang_plan (NULL: off)
  uint32_t* gang_hdr;   // [0] gangs, [1] units, [2] unit dispenser
  uint32_t* gang_slot;  // [gangs] item slot (rep_list index, or item)
  uint32_t* gang_off;   // [gangs + 1] first unit of each gang
  uint32_t* gang_sync;  // [gangs][2] leader CTA (~0: not yet), stage parts finished
  double gang_min, gang_unit;
  int32_t gang_max, pad_gang;
  // hashed signature keys (class + codes wider than 63 bits): set when an
  // item's class / codes differ from its signature representative's (a
  // hash collision); K_est then reads the per-item cuts of the guarded
  // per-item K_dp instead of the signature's (NULL: exact keys)
  const uint32_t* memo_bad;
  // node-determined bandwidths (every link a function of its two nodes,
  // symmetric): make_comm_group's pairwise minimum over the nodes present
  // in the group instead of over its device pairs (warp K_est), or NULL
  const int32_t* node_of;     // [D] dense node index of each device
  const double* nodebw;       // [n_nodes][n_nodes] (diagonal: intra-node links)
  int32_t n_nodes, node_words;  // node bitmap words (32 nodes each)
  // |D| = 16: placement of every placement index p < perm_n (k_perm_table),
  // shared by the classes, or NULL
  const uint64_t* perm_tab;
  uint64_t perm_n;
  // |D| = 16 full shapes, codes < 16: the link codes of placement pl under
  // the shape of row crow, ctab[crow * perm_n + pl] = {x: the edge code of
  // every (boundary q, replica r) at 4 bits (q * dp + r) (min over shards),
  // y: the all-reduce group code of every stage j at 4 bits j (min over the
  // group's pairs)} (k_code_table), or NULL
  const ulonglong2* ctab;
};

// std::min(a, b) with the reference's argument order: (b < a) ? b : a.
__device__ __forceinline__ double std_min(double a, double b) { return b < a ? b : a; }
// std::max(a, b): (a < b) ? b : a.
__device__ __forceinline__ double std_max(double a, double b) { return a < b ? b : a; }
// std::max(0.0, x)
__device__ __forceinline__ double max0(double x) { return 0.0 < x ? x : 0.0; }

__device__ __forceinline__ void prefetch_l2(const void* a) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

// splitmix64; integer-only, identical on host.
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Ranking key of rank_records (optimizer.cpp:178-196): non-failed first,
// then total ascending, then (pp, dp, tmp, mbs[, p]) == candidate index.
// fail_code < 0 marks an empty slot that sorts after everything.
__host__ __device__ inline bool rank_less(const amp_record& a, const amp_record& b) {
  const int ca = a.fail_code < 0 ? 2 : (a.fail_code != 0 ? 1 : 0);
  const int cb = b.fail_code < 0 ? 2 : (b.fail_code != 0 ? 1 : 0);
  if (ca != cb) return ca < cb;
  if (ca == 0 && a.total != b.total) return a.total < b.total;
  return a.index < b.index;
}

}  // namespace amp
