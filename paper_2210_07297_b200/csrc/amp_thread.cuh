// amp_thread.cuh — K_place / K_est with one THREAD per candidate for
// clusters of at most 16 devices with coded bandwidths.
//
// The warp-per-candidate kernels (amp_pipeline.cuh) spread one candidate's
// few dozen sequential steps over 32 lanes; at |D| <= 16 most lanes idle or
// repeat the same scalar work (the splitmix64 chain, the stage loops).  Here
// a thread runs the reference's sequential code for its own candidate:
//  * the placement is a 16 x 4-bit nibble vector in one register;
//  * the Fisher–Yates draw r mod (k+1) uses a 32-bit Barrett step;
//  * the bandwidths are per-link u8 codes with integer minima (the
//    distinct-value table is sorted, so min code == code of the min);
//  * the edge costs come from the per-class tables of IEEE quotients.
// Every floating-point value is produced by the same operations in the
// same order as the warp kernels and the reference (sequential sums,
// strict comparisons), so records, cuts and the top-k are bit-identical
// (the GPU parity tests run both paths).
#pragma once

#include "amp_common.cuh"
#include "amp_dedup.cuh"
#include "amp_pipeline.cuh"

namespace amp {

constexpr int kThreadMaxD = 16;

__device__ __forceinline__ int nib(uint64_t v, int i) { return (int)((v >> (4 * i)) & 0xf); }

// r mod d for d in [2, 32]: (hi mod d) * (2^32 mod d) + (lo mod d), each
// 32-bit mod by a Barrett step with m = floor(2^32 / d) (quotient off by at
// most one, fixed by one conditional subtraction).
__device__ __forceinline__ uint32_t mod32(uint32_t x, uint32_t d, uint32_t m) {
  uint32_t r = x - __umulhi(x, m) * d;
  return r >= d ? r - d : r;
}
// (m, t32) = (floor(2^32 / d), 2^32 mod d) come from a per-CTA table: a
// 64-bit division by a runtime divisor is a ~100-instruction routine.
__device__ __forceinline__ uint32_t mod64_small(uint64_t r, uint32_t d, uint2 mt) {
  const uint32_t a = mod32((uint32_t)(r >> 32), d, mt.x), b = mod32((uint32_t)r, d, mt.x);
  return mod32(a * mt.y + b, d, mt.x);  // < d*d + d <= 1056
}

// ---------------------------------------------------------------------------
// K_place (thread per candidate)
// ---------------------------------------------------------------------------
// Shared state of the thread kernels' placement step (per CTA).
struct PlaceSmem {
  uint8_t code[kThreadMaxD * kThreadMaxD];
  uint64_t base_perm;
  uint2 magic[kThreadMaxD + 1];  // d -> (floor(2^32/d), 2^32 mod d)
};

__device__ void place_smem_init(const EvalParams& p, PlaceSmem& S) {
  const int D = p.D;
  for (int x = threadIdx.x; x < D * D; x += blockDim.x) S.code[x] = p.bwcode[x];
  if (threadIdx.x >= 2 && threadIdx.x <= kThreadMaxD)
    S.magic[threadIdx.x] = make_uint2((uint32_t)(0x100000000ull / threadIdx.x),
                                      (uint32_t)(0x100000000ull % threadIdx.x));
  if (threadIdx.x == 0) {
    uint64_t v = 0;
    for (int x = 0; x < D; ++x) v |= (uint64_t)p.base_order[x] << (4 * x);
    S.base_perm = v;
  }
}

// Boundary codes of a full-shape class (PP, DPn, TMP), loops unrolled
// (constant nibble shifts): the min over replicas and shards of each stage
// boundary's link codes (cost_model.cpp:164-174), appended to the DP
// signature key.  Positive bandwidths only (no boundary can fail).
template <int PP, int DPn, int TMP>
__device__ __forceinline__ uint64_t codes_shape(const EvalParams& p, const uint8_t* code, uint64_t perm,
                                                bool has_cw, ulonglong2 cw, uint64_t u, bool store,
                                                uint64_t key, int& code0) {
#pragma unroll
  for (int q = 0; q < PP - 1; ++q) {
    int cm = 255;
    if (has_cw) {  // the placement's per-replica edge codes (k_code_table)
#pragma unroll
      for (int r = 0; r < DPn; ++r) {
        const int cc = (int)((cw.x >> (4 * (q * DPn + r))) & 0xf);
        cm = cc < cm ? cc : cm;
      }
    } else {
#pragma unroll
      for (int r = 0; r < DPn && cm; ++r)
#pragma unroll
        for (int s = 0; s < TMP && cm; ++s) {
          const int cc = code[nib(perm, (q * DPn + r) * TMP + s) * 16 + nib(perm, ((q + 1) * DPn + r) * TMP + s)];
          cm = cc < cm ? cc : cm;
        }
    }
    if (q == 0) code0 = cm;
    key = (key << p.sig_code_bits) | (uint64_t)cm;
    if (store) {
      if (p.need_bwcb) p.bwcb[u * p.max_pp + q] = (uint8_t)cm;
      if (p.need_bwq) p.bwqb[u * p.max_pp + q] = p.bwval[cm];
    }
  }
  return key;
}

// The code-table entry of a placement under shape (PP, DPn, TMP): x = the
// edge code of every (boundary q, replica r), min over the shards
// (cost_model.cpp:164-174 before the min over replicas), y = the all-reduce
// group code of every stage (min over the group's device pairs,
// cost_model.cpp:122-143).  Codes < 16.
template <int PP, int DPn, int TMP>
__device__ __forceinline__ ulonglong2 ctab_entry(const uint8_t* code, uint64_t perm) {
  uint64_t x = 0, y = 0;
#pragma unroll
  for (int q = 0; q < PP - 1; ++q)
#pragma unroll
    for (int r = 0; r < DPn; ++r) {
      int cm = 255;
#pragma unroll
      for (int s = 0; s < TMP; ++s) {
        const int cc = code[nib(perm, (q * DPn + r) * TMP + s) * 16 + nib(perm, ((q + 1) * DPn + r) * TMP + s)];
        cm = cc < cm ? cc : cm;
      }
      x |= (uint64_t)cm << (4 * (q * DPn + r));
    }
  if (DPn > 1)
#pragma unroll
    for (int j = 0; j < PP; ++j) {
      int cm = 255;
#pragma unroll
      for (int s = 0; s < TMP; ++s)
#pragma unroll
        for (int r1 = 0; r1 < DPn; ++r1)
#pragma unroll
          for (int r2 = r1 + 1; r2 < DPn; ++r2) {
            const int cc = code[nib(perm, (j * DPn + r1) * TMP + s) * 16 + nib(perm, (j * DPn + r2) * TMP + s)];
            cm = cc < cm ? cc : cm;
          }
      y |= (uint64_t)cm << (4 * j);
    }
  return make_ulonglong2(x, y);
}

// K_place's work for chunk item u: decode, early failures, placement,
// boundary codes.  `store`: write placement / codes / values for the later
// kernels (K_dp, K_est); else only return them (fused light path).
// DT > 0: the device count as a compile-time constant (the Fisher-Yates
// loop unrolls: constant shifts, constant-divisor modulo).
// DECODE_ONLY: decode and the early failures only (K_est re-deriving a
// K_place item's work record: the placement comes from placep).
template <int DT, bool FAST = false, bool DECODE_ONLY = false>
__device__ __forceinline__ void place_one(const EvalParams& p, const PlaceSmem& S, uint64_t u,
                                          bool store, CandWork& w, uint64_t& perm, int& code0,
                                          uint64_t* sig = nullptr, int* seg_hint = nullptr,
                                          ulonglong2* cwo = nullptr) {
  if (sig) *sig = ~0ull;
  const int D = DT > 0 ? DT : p.D, maxpp = p.max_pp;
  uint64_t index, out, pl;
  int c;
  decode_item(p, p.t0 + u, index, out, c, pl, seg_hint);
  const ClassDev cl = p.cls[c];
  // the placement's code-table entry, issued with the pair load (it is used
  // only when the item does not fail early, but its address is valid)
  const bool has_cw = FAST && p.ctab != nullptr;
  ulonglong2 cwv = make_ulonglong2(0, 0);
  if (has_cw && (cl.pp > 1 || cl.dp > 1) && cl.crow >= 0) cwv = p.ctab[(uint64_t)cl.crow * p.P + pl];
  const PairDev pr = p.pairs[cl.pair];
  const int pp = cl.pp, dp = cl.dp, tmp = cl.tmp;
  int fc = 0, flayer = -1;
  double fval = 0.0;
  code0 = 0;
  perm = S.base_perm;
  if (pp > p.L) {  // optimizer.cpp:149-152
    fc = AMP_FAIL_PP_GT_L;
  } else if (pr.fail_code) {  // segment_times: first failing layer
    fc = pr.fail_code;
    flayer = pr.fail_layer;
    fval = pr.fail_value;
  }
  if (fc == 0 && !DECODE_ONLY) {
    // ---- placement: heuristic order (placement.cpp:37-49); p >= 1:
    //      Fisher-Yates driven by splitmix64(seed ^ p) ----------------------
    if constexpr (FAST) {
      // (the shape kernels run only with the placement table: P = 1 or the
      //  table of every placement index; no per-candidate shuffle)
      if (pl != 0 && !p.ctab && (store || pp != 1 || dp != 1)) perm = p.perm_tab[pl];
    } else if (p.given_place) {  // caller placement (anneal proposals, evaluate_placed)
      const int32_t* g = p.given_place + (p.t0 + u) * D;
      perm = 0;
      for (int x = 0; x < D; ++x) perm |= (uint64_t)g[x] << (4 * x);
    } else if (pl != 0 && (store || !FAST || pp != 1 || dp != 1)) {
      // (a fused pp = dp = 1 item's estimate does not depend on where its
      //  single stage sits: no edges, no all-reduce group — the shuffle is
      //  skipped when nothing stores the placement)
      if (p.perm_tab && pl < p.perm_n) {
        perm = p.perm_tab[pl];  // the shuffle of placement pl, shared by every class
      } else {
      uint64_t r = splitmix64(p.seed ^ pl);
      if (DT > 0) {
#pragma unroll
        for (int kk = DT - 1; kk >= 1; --kk) {
          const uint32_t d = (uint32_t)kk + 1u;  // constant: the compiler's divide-by-constant
          const uint32_t t32 = (uint32_t)(0x100000000ull % d);
          const uint32_t jj = (uint32_t)((((uint32_t)(r >> 32) % d) * t32 + ((uint32_t)r % d)) % d);
          // swap nibbles kk and jj: x = a ^ b flips both (x = 0 when jj == kk)
          const uint64_t x = ((perm >> (4 * kk)) ^ (perm >> (4 * jj))) & 0xf;
          perm ^= (x << (4 * kk)) | (x << (4 * jj));
          r = splitmix64(r);
        }
      } else {
        for (int kk = D - 1; kk >= 1; --kk) {
          const int jj = (int)mod64_small(r, (uint32_t)kk + 1u, S.magic[kk + 1]);
          const uint64_t x = ((perm >> (4 * kk)) ^ (perm >> (4 * jj))) & 0xf;  // (nibble swap)
          perm ^= (x << (4 * kk)) | (x << (4 * jj));
          r = splitmix64(r);
        }
      }
      }
    }
    if (store && p.placep) p.placep[u] = perm;
    if (has_cw && cwo) *cwo = cwv;
    if (store && p.need_place_rows) {
      int32_t* prow = p.placeb + u * D;
      for (int x = 0; x < D; ++x) prow[x] = nib(perm, x);
    }
    // ---- stage-boundary bandwidths: min over all replicas and shards
    //      (cost_model.cpp:164-174), as codes; the first invalid boundary
    //      fails like p2p_time in the DP's edge function -----------------
    int first_bad = -1;
    double bad_val = 0.0;
    uint64_t key = (uint64_t)c;  // DP signature (amp_dedup.cuh sig_key)
    if constexpr (FAST) {  // p.shape16: every class a full 16-device shape, bandwidths > 0
      switch (pp * 1024 + dp * 32 + tmp) {
#define AMP_SHAPE(a, b, c)                                                        \
  case a * 1024 + b * 32 + c:                                                     \
    key = codes_shape<a, b, c>(p, S.code, perm, has_cw, cwv, u, store, key, code0); \
    break;
        AMP_SHAPE(1, 1, 16) AMP_SHAPE(1, 2, 8) AMP_SHAPE(1, 4, 4) AMP_SHAPE(1, 8, 2) AMP_SHAPE(1, 16, 1)
        AMP_SHAPE(2, 1, 8) AMP_SHAPE(2, 2, 4) AMP_SHAPE(2, 4, 2) AMP_SHAPE(2, 8, 1)
        AMP_SHAPE(4, 1, 4) AMP_SHAPE(4, 2, 2) AMP_SHAPE(4, 4, 1)
        AMP_SHAPE(8, 1, 2) AMP_SHAPE(8, 2, 1)
        AMP_SHAPE(16, 1, 1)
#undef AMP_SHAPE
        default:
          __trap();  // (the host sets shape16 only for these shapes)
      }
    }
    for (int q = 0; !FAST && q < pp - 1; ++q) {
      int cm = 255;  // (code 0 is the smallest bandwidth: nothing can go lower)
      for (int r = 0; r < dp && cm; ++r)
        for (int s = 0; s < tmp && cm; ++s) {
          const int cc = S.code[nib(perm, (q * dp + r) * tmp + s) * D +
                                nib(perm, ((q + 1) * dp + r) * tmp + s)];
          cm = cc < cm ? cc : cm;
        }
      const double b = p.bwval[cm];
      if (q == 0) code0 = cm;
      key = (key << p.sig_code_bits) | (uint64_t)cm;
      if (store) {
        if (p.need_bwcb) p.bwcb[u * maxpp + q] = (uint8_t)cm;
        if (p.need_bwq) p.bwqb[u * maxpp + q] = b;
      }
      if (first_bad < 0 && !(b > 0)) {
        first_bad = q;
        bad_val = b;
      }
    }
    if (first_bad >= 0) {
      fc = AMP_FAIL_P2P_BANDWIDTH;
      fval = bad_val;
    }
    if (store && (p.sigkey || sig)) {  // zero codes pad the unused boundaries
      key <<= (uint64_t)p.sig_code_bits * (uint64_t)(maxpp - (pp > 0 ? pp : 1));
      key = (fc == 0 && pp >= 3) ? key : ~0ull;
      if (sig) *sig = key;
      else p.sigkey[u] = key;
    }
  } else if (store && p.sigkey && !sig) {
    p.sigkey[u] = ~0ull;
  }
  w.index = index;
  w.out = out;
  w.cls = c;
  w.fail_code = fc;
  w.fail_layer = flayer;
  w.pad = 0;
  w.fail_value = fval;
}

// 256 threads; -DAMP_PLACE_MINB=n caps the registers for n CTAs/SM (8
// measured slower).  Without it ptxas picks the count (40).
#ifdef AMP_PLACE_MINB
#define AMP_PLACE_BOUNDS __launch_bounds__(256, AMP_PLACE_MINB)
#else
#define AMP_PLACE_BOUNDS __launch_bounds__(256)
#endif
template <int DT, bool FAST = false>
__global__ void AMP_PLACE_BOUNDS k_place_t(EvalParams p) {
  __shared__ PlaceSmem S;
  place_smem_init(p, S);
  __syncthreads();
  // fused light path: K_est_t places the pp <= 2 tail itself
  const uint64_t n = p.fuse_light ? p.n_dp : p.n_chunk;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (p.fuse_hash) {
    // the signature hash insert (amp_dedup.cuh k_hash_insert) fused: the key
    // goes from registers into the table; warp-uniform trip count for the
    // warp-cooperative probe
    const int lane = threadIdx.x & 31, sh = p.h_eshift;
    const uint64_t tag = sh >= 64 ? 0 : (p.h_epoch << sh);
    int hint = -1;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n;
         base += stride) {
      const uint64_t u = base + lane;
      uint64_t key = kHashEmpty;
      if (u < n) {
        CandWork w;
        uint64_t perm;
        int code0;
        place_one<DT, FAST>(p, S, u, true, w, perm, code0, &key, &hint);
        if (!p.skip_work) p.work[u] = w;
      }
      const uint32_t slot = hash_insert_warp(key, u, lane, p.h_tkey, p.h_tval, p.h_uniq, p.h_nuniq,
                                             p.h_mask, tag, p.h_epoch, sh,
                                             p.h_max_probe);
      if (u < n) p.h_slot_of[u] = slot;
    }
    return;
  }
  int hint = -1;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
    CandWork w;
    uint64_t perm;
    int code0;
    place_one<DT, FAST>(p, S, u, true, w, perm, code0, nullptr, &hint);
    if (!p.skip_work) p.work[u] = w;
  }
}

// The placement of every placement index p in [0, n) as 16 x 4-bit
// nibbles (p = 0 the heuristic order, p >= 1 its
// Fisher-Yates shuffle driven by splitmix64(seed ^ p)).  It depends on p
// only — not on the class — so K_place / K_est of every class read it here
// instead of redoing the 15-step shuffle per candidate.  |D| = 16.
__global__ void k_perm_table(EvalParams p, uint64_t* out, uint64_t n) {
  __shared__ uint64_t base;
  if (threadIdx.x == 0) {
    uint64_t v = 0;
    for (int x = 0; x < p.D; ++x) v |= (uint64_t)p.base_order[x] << (4 * x);
    base = v;
  }
  __syncthreads();
  for (uint64_t pl = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; pl < n;
       pl += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t perm = base;
    if (pl != 0) {
      uint64_t r = splitmix64(p.seed ^ pl);
#pragma unroll
      for (int kk = 15; kk >= 1; --kk) {
        const uint32_t d = (uint32_t)kk + 1u;
        const uint32_t t32 = (uint32_t)(0x100000000ull % d);
        const uint32_t jj = (uint32_t)((((uint32_t)(r >> 32) % d) * t32 + ((uint32_t)r % d)) % d);
        const uint64_t x = ((perm >> (4 * kk)) ^ (perm >> (4 * jj))) & 0xf;
        perm ^= (x << (4 * kk)) | (x << (4 * jj));
        r = splitmix64(r);
      }
    }
    out[pl] = perm;
  }
}

// The code table (EvalParams::ctab): for every shape row and placement
// index, the placement's edge and all-reduce group codes (ctab_entry), so
// K_place / K_est of every class of that shape read one 16-byte entry
// instead of redoing the code minima per candidate.  |D| = 16, full shapes.
__global__ void k_code_table(EvalParams p, const int32_t* row_shape, int n_rows, ulonglong2* out) {
  __shared__ PlaceSmem S;
  place_smem_init(p, S);
  __syncthreads();
  const uint64_t P = p.P, n = (uint64_t)n_rows * P;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const int row = (int)(x / P);
    const uint64_t pl = x - (uint64_t)row * P;
    const uint64_t perm = pl == 0 ? S.base_perm : p.perm_tab[pl];
    ulonglong2 e = make_ulonglong2(0, 0);
    switch (row_shape[row]) {
#define AMP_SHAPE(a, b, c)            \
  case a * 1024 + b * 32 + c:         \
    e = ctab_entry<a, b, c>(S.code, perm); \
    break;
      AMP_SHAPE(1, 1, 16) AMP_SHAPE(1, 2, 8) AMP_SHAPE(1, 4, 4) AMP_SHAPE(1, 8, 2) AMP_SHAPE(1, 16, 1)
      AMP_SHAPE(2, 1, 8) AMP_SHAPE(2, 2, 4) AMP_SHAPE(2, 4, 2) AMP_SHAPE(2, 8, 1)
      AMP_SHAPE(4, 1, 4) AMP_SHAPE(4, 2, 2) AMP_SHAPE(4, 4, 1)
      AMP_SHAPE(8, 1, 2) AMP_SHAPE(8, 2, 1)
      AMP_SHAPE(16, 1, 1)
#undef AMP_SHAPE
      default:
        break;
    }
    out[x] = e;
  }
}

// ---------------------------------------------------------------------------
// K_est shape kernels: the estimate of one candidate of class shape
// (PP, DPn, TMP) (pp * dp * tmp == 16) with every loop unrolled — nibble
// extractions become constant shifts, the cut / stage values live in
// registers (the generic body indexes them at run time: local memory), and
// the replicas' independent table loads overlap.  The same operations in the
// same order as the generic body (which still serves detail outputs, given
// cuts and non-positive bandwidth tables), so results are bit-identical.
// The stage loop fuses stage_time, the first-maximum scan, the stage-sum
// chain of the slowest replica, the parameter ceiling and dpsync_time: each
// keeps its own sequential order, they only share the stage's two loads.
template <int PP, int DPn, int TMP>
__device__ __forceinline__ void est_shape(const EvalParams& p, const ulonglong2 cw, const CandWork& w,
                                          const ClassDev& cl, uint64_t u, bool fused, int code0, int& fc,
                                          double& pipeline, double& dpsync, uint32_t rs) {
  const int L = p.L, LP = L + 1, maxpp = p.max_pp;
  int cuts[PP + 1];
  if (PP >= 3) {  // the signature run's cuts (memoised DP) or this item's
    if (DPn == 1 && p.run_pipe) {
      // one replica whose boundary codes are the signature's: the whole
      // estimate is a function of the run (k_run_pipe, same operations),
      // stored by hash slot when the shape kernels look runs up by slot
      const double v = p.run_slot ? p.run_pipe[rs]
                                  : p.run_pipe[p.rep_of ? p.rep_of[u] : 0u];
      if (v != v) {
        fc = AMP_FAIL_CEILING;
      } else {
        pipeline = v;
        dpsync = 0.0;
      }
      return;
    }
    const uint64_t run = p.run_slot ? p.run_of_slot[rs] : p.rep_of ? p.rep_of[u] : ~0ull;
    const uint8_t* ci = run != ~0ull ? p.repcuts + run * (maxpp + 1) : p.cutsb + u * (maxpp + 1);
#pragma unroll
    for (int q = 0; q <= PP; ++q) cuts[q] = ci[q];
  } else if (PP == 2) {
    cuts[0] = 0;
    cuts[1] = p.cut2tab[(size_t)w.cls * p.n_codes + (fused ? code0 : p.bwcb[u * maxpp])];
    cuts[PP] = L;
  } else {
    cuts[0] = 0;
    cuts[PP] = L;
  }
  // slowest replica's edge sum (edge-sum monotonicity, see the generic body)
  const double* qt = p.qtab + (size_t)w.cls * p.n_codes * L;
  double emax = -CUDART_INF;
#pragma unroll
  for (int r = 0; r < (PP == 1 ? 1 : DPn); ++r) {
    double esum = 0.0;
#pragma unroll
    for (int q = 0; q < PP - 1; ++q) {
      const int cm = (int)((cw.x >> (4 * (q * DPn + r))) & 0xf);  // (min over the shards)
      esum = esum + qt[(size_t)cm * L + cuts[q + 1]];
    }
    emax = emax < esum ? esum : emax;
  }
#ifdef AMP_EST_DEBUG
  for (int q = 0; q <= PP; ++q)
    if (cuts[q] < 0 || cuts[q] > L || (q && cuts[q] < cuts[q - 1]))
      printf("est_fast: PP %d u=%llu bad cuts q=%d %d rep=%u\n", PP, (unsigned long long)u, q, cuts[q],
             p.rep_of ? p.rep_of[u] : 0u);
#endif
  const double* rt = p.rsum_t + (size_t)cl.pair * LP * LP;
  double slowest = 0.0, sum = emax, worst_p = 0.0, worst = 0.0;
#pragma unroll
  for (int j = 0; j < PP; ++j) {
    const int a = cuts[j] * LP + cuts[j + 1];
    const double stj = rt[a], spj = p.rsum_p[a];
    slowest = (j == 0 || slowest < stj) ? stj : slowest;  // std::max_element: first maximum
    sum = sum + stj;
    if (p.has_ceiling) worst_p = std_max(worst_p, spj / TMP);
    if (DPn != 1) {  // dpsync: the stage's minimum-bandwidth group (bw_positive)
      const int cm = (int)((cw.y >> (4 * j)) & 0xf);
      const double b = p.bwval[cm];
      const double message = spj * p.bpp / TMP;
      worst = std_max(worst, 2.0 * (double)(DPn - 1) * message / ((double)DPn * b));
    }
  }
  if (p.has_ceiling && worst_p > p.ceiling) {
    fc = AMP_FAIL_CEILING;
    return;
  }
  pipeline = (double)(cl.gas - 1) * slowest + sum;
  dpsync = worst;
}

// Per signature run of a dp == 1, pp >= 3 class: est_shape's estimate with
// one replica (its edge codes are the signature's boundary codes — the
// K_place minimum over replicas x shards with a single replica), so K_est
// reads one value per item.  Same operations and order as est_shape.
// out is indexed by run, or by the run's hash slot when slot_of_run is given
// (K_est then reads it through the item's slot: one dependent load less).
__global__ void k_run_pipe(EvalParams p, const uint64_t* rep_key, const unsigned long long* n_runs_d,
                           double* out, const uint32_t* slot_of_run) {
  const int nq = p.max_pp - 1, cb = p.sig_code_bits, L = p.L, LP = L + 1, maxpp = p.max_pp;
  const uint64_t cmask = (1ull << cb) - 1;
  const uint64_t n_runs = *n_runs_d;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_runs;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = rep_key[r];
    const int c = (int)(key >> (nq * cb));
    const ClassDev cl = p.cls[c];
    if (cl.dp != 1 || cl.pp < 3) continue;
    const uint8_t* ci = p.repcuts + r * (maxpp + 1);
    const double* qt = p.qtab + (size_t)c * p.n_codes * L;
    double esum = 0.0;
    for (int q = 0; q < cl.pp - 1; ++q) {
      const int code = (int)((key >> ((nq - 1 - q) * cb)) & cmask);
      esum = esum + qt[(size_t)code * L + ci[q + 1]];
    }
    double emax = -CUDART_INF;
    emax = emax < esum ? esum : emax;
    const double* rt = p.rsum_t + (size_t)cl.pair * LP * LP;
    double slowest = 0.0, sum = emax, worst_p = 0.0;
    for (int j = 0; j < cl.pp; ++j) {
      const int a = ci[j] * LP + ci[j + 1];
      const double stj = rt[a], spj = p.rsum_p[a];
      slowest = (j == 0 || slowest < stj) ? stj : slowest;
      sum = sum + stj;
      if (p.has_ceiling) worst_p = std_max(worst_p, spj / cl.tmp);
    }
    out[slot_of_run ? (uint64_t)slot_of_run[r] : r] =
        (p.has_ceiling && worst_p > p.ceiling) ? CUDART_NAN : (double)(cl.gas - 1) * slowest + sum;
  }
}

// One candidate through the shape kernels (p.est_fast: |D| == 16, every class
// with pp * dp * tmp == 16, positive bandwidths, range and 2-stage tables, no
// detail outputs, no given cuts).
template <int DT>
__device__ __forceinline__ void est_fast_item(const EvalParams& p, const PlaceSmem& PS, uint64_t u,
                                              amp_record& rec, bool& ok, int* seg_hint) {
  const bool fused = p.fuse_light && u >= p.n_dp;
  // a heavy item's signature-run slot, issued before its decode (the run's
  // cuts / estimate lookups hang off it)
  const uint32_t rs = (!fused && p.run_slot && u < p.n_dp) ? p.run_slot[u] : 0u;
  CandWork w;
  uint64_t perm = 0;
  int code0 = 0;
  ulonglong2 cw = make_ulonglong2(0, 0);  // the placement's link codes (k_code_table)
  if (fused) place_one<DT, true>(p, PS, u, false, w, perm, code0, nullptr, seg_hint, &cw);
  else if (p.skip_work) place_one<DT, true, true>(p, PS, u, false, w, perm, code0, nullptr, seg_hint);
  else w = p.work[u];
  const ClassDev cl = p.cls[w.cls];
  int fc = w.fail_code;
  double pipeline = CUDART_NAN, dpsync = CUDART_NAN;
  if (fc == 0) {
    // (a dp == 1, pp >= 3 item with the per-run estimate needs no placement)
    if (!fused && !(p.run_pipe && cl.dp == 1 && cl.pp >= 3))
      cw = p.ctab[(uint64_t)cl.crow * p.P + (w.index - (uint64_t)w.cls * p.P)];
    switch (cl.pp * 1024 + cl.dp * 32 + cl.tmp) {
#define AMP_SHAPE(a, b, c)                                                    \
  case a * 1024 + b * 32 + c:                                                 \
    est_shape<a, b, c>(p, cw, w, cl, u, fused, code0, fc, pipeline, dpsync, rs); \
    break;
      AMP_SHAPE(1, 1, 16) AMP_SHAPE(1, 2, 8) AMP_SHAPE(1, 4, 4) AMP_SHAPE(1, 8, 2) AMP_SHAPE(1, 16, 1)
      AMP_SHAPE(2, 1, 8) AMP_SHAPE(2, 2, 4) AMP_SHAPE(2, 4, 2) AMP_SHAPE(2, 8, 1)
      AMP_SHAPE(4, 1, 4) AMP_SHAPE(4, 2, 2) AMP_SHAPE(4, 4, 1)
      AMP_SHAPE(8, 1, 2) AMP_SHAPE(8, 2, 1)
      AMP_SHAPE(16, 1, 1)
#undef AMP_SHAPE
      default:
#ifdef AMP_EST_DEBUG
        printf("est_fast: shape %d %d %d u=%llu cls=%d fused=%d\n", cl.pp, cl.dp, cl.tmp,
               (unsigned long long)u, w.cls, (int)fused);
        fc = 99;
        break;
#else
        __trap();  // (the host enables est_fast only for these shapes)
#endif
    }
  }
  rec.index = w.index;
  rec.pp = cl.pp;
  rec.dp = cl.dp;
  rec.tmp = cl.tmp;
  rec.mbs = cl.mbs;
  rec.fail_code = fc;
  rec.fail_layer = fc == AMP_FAIL_PROFILE_MISS ? w.fail_layer : -1;
  rec.fail_value = fc == AMP_FAIL_P2P_BANDWIDTH ? w.fail_value : 0.0;
  ok = fc == 0;
  rec.pipeline_time = ok ? pipeline : CUDART_NAN;
  rec.dpsync_time = ok ? dpsync : CUDART_NAN;
  rec.total = ok ? pipeline + dpsync : CUDART_NAN;
  if (p.all) p.all[w.out] = rec;
}

// ---------------------------------------------------------------------------
// K_est (thread per candidate)
// ---------------------------------------------------------------------------
constexpr int kEstTWarps = 8;
#ifndef AMP_EST_PREFETCH
#define AMP_EST_PREFETCH 1
#endif

template <int DT, bool FAST = false>
#ifndef AMP_EST_MINB
#define AMP_EST_MINB 4  // (64 registers: 4 CTAs x 8 warps per SM)
#endif
__global__ void __launch_bounds__(kEstTWarps * 32, AMP_EST_MINB) k_est_t(EvalParams p) {
  __shared__ PlaceSmem PS;
  const uint8_t* codeS = PS.code;
  __shared__ int n_top;
  __shared__ amp_record stage_rec[kEstTWarps][32];  // records handed to the warp leader
  __shared__ amp_record wtop[kEstTWarps][32];       // per-warp top-k (no lock)
  __shared__ amp_record topS[32];
  const int D = p.D, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, maxpp = p.max_pp;
  const int L = p.L, LP = L + 1;
  amp_record* const gtop = p.cta_topk + (size_t)blockIdx.x * p.k;
  amp_record* mytop = p.k <= 32 ? topS : gtop;
  place_smem_init(p, PS);
  if (threadIdx.x == 0) {
    n_top = 0;
    if (!p.first_chunk) {  // CTA lists persist across chunks
      for (int x = 0; x < p.k; ++x) {
        if (gtop[x].fail_code < 0) break;
        if (mytop != gtop) mytop[x] = gtop[x];
        ++n_top;
      }
    }
  }
  __syncthreads();
  __shared__ int wcount[kEstTWarps];
  // Warp top-k threshold: the rank key (failed flag, total, index) an item
  // must beat (rank_less) to be handed to the leader — the warp list's k-th
  // entry once it is full, before that the CTA list's k-th entry persisted
  // from the previous chunk (an item that cannot beat it cannot reach the
  // CTA's top-k), else nothing (w_kf = 2).  The exact key (index included)
  // matters: a chunk of failing candidates would otherwise pass every item.
  // (the warp list's count and threshold live in shared memory:
  // registers are the kernel's occupancy limit)
  __shared__ unsigned long long w_ki[kEstTWarps];
  __shared__ double w_kt[kEstTWarps];
  __shared__ int w_kf[kEstTWarps];
  if (lane == 0) {
    wcount[wib] = 0;
    w_kf[wib] = 2;
    w_kt[wib] = CUDART_INF;
    w_ki[wib] = ~0ull;
    if (p.k > 0 && n_top == p.k) {
      const amp_record& e = mytop[p.k - 1];
      w_kf[wib] = e.fail_code < 0 ? 2 : (e.fail_code != 0 ? 1 : 0);
      w_kt[wib] = e.total;
      w_ki[wib] = e.index;
    }
  }
  __syncwarp();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  int seg_hint = -1;  // (decode_item: this thread's previous segment)
  // uniform trip count per warp (the top-k hand-off is warp-synchronous)
  const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  for (uint64_t wbase = first; wbase < p.n_chunk; wbase += stride) {
    const uint64_t u = wbase + lane;
    const bool live = u < p.n_chunk;
#if AMP_EST_PREFETCH
    {  // the next iteration's streamed inputs into L2 (no registers held)
      const uint64_t un = u + stride;
      if (un < p.n_chunk && !(p.fuse_light && un >= p.n_dp)) {
        if (!p.skip_work) prefetch_l2(p.work + un);
        if (p.placep) prefetch_l2(p.placep + un);
        if (p.run_slot && un < p.n_dp) prefetch_l2(p.run_slot + un);
        else if (p.rep_of && un < p.n_dp) prefetch_l2(p.rep_of + un);
      }
    }
#endif
    amp_record rec;
    int cuts[kThreadMaxD + 1];
    double st[kThreadMaxD], spar[kThreadMaxD];
    int pp = 0, best_r = -1;
    bool ok = false;
    if constexpr (FAST) {
      if (live) est_fast_item<DT>(p, PS, u, rec, ok, &seg_hint);
    } else if (live) {
      // fused light path: the pp <= 2 tail (never in K_dp) is placed here
      const bool fused = p.fuse_light && u >= p.n_dp;
      CandWork w;
      uint64_t perm = 0;
      int code0 = 0;
      if (fused) place_one<DT>(p, PS, u, false, w, perm, code0);
      else w = p.work[u];
      const ClassDev cl = p.cls[w.cls];
      pp = cl.pp;
      const int dp = cl.dp, tmp = cl.tmp, mbs = cl.mbs;
      int fc = w.fail_code;
      double fval = w.fail_value;
      double pipeline = CUDART_NAN, dpsync = CUDART_NAN;
      if (fc == 0) {
        if (fused) {
        } else if (p.placep) {
          perm = p.placep[u];
        } else {
          const int32_t* PL = p.placeb + u * D;
          for (int x = 0; x < D; ++x) perm |= (uint64_t)PL[x] << (4 * x);
        }
        // ---- cuts: K_dp (memoised: its signature's representative), or
        //      the k <= 2 DP here (light_cut2's operations, sequential) ---
        if (pp >= 3 || p.cuts_given) {
          // (memoised DP: the cuts of this candidate's signature run)
          const uint8_t* ci = (p.rep_of && !p.cuts_given && u < p.n_dp && !(p.memo_bad && *p.memo_bad))
                                  ? p.repcuts + (uint64_t)p.rep_of[u] * (maxpp + 1)
                                  : p.cutsb + u * (maxpp + 1);
          for (int q = 0; q <= pp; ++q) cuts[q] = ci[q];
        } else if (pp == 2 && p.cut2tab) {
          // the 2-stage DP depends on (class, boundary-0 code) only: tabulated
          // once per context by k_cut2_table (the same operations)
          cuts[0] = 0;
          cuts[1] = p.cut2tab[(size_t)w.cls * p.n_codes + (fused ? code0 : p.bwcb[u * maxpp])];
          cuts[2] = L;
        } else if (pp == 2) {
          const double* Pf = p.prefix + (size_t)cl.pair * LP;
          const double* Dm = p.domain + (size_t)cl.pair * p.nv_stride;
          const uint16_t* sg = p.seg + (size_t)cl.pair * LP * LP;
          const double g1 = (double)(cl.gas - 1);
          const double* qt =
              p.qtab + ((size_t)w.cls * p.n_codes + (fused ? code0 : p.bwcb[u * maxpp])) * L;
          const double dm0 = Dm[0], PLL = Pf[L], P0 = Pf[0];
          double best = CUDART_INF;
          int bc = -1;
          for (int c = 1; c < L; ++c) {
            const double t1 = Pf[c] - P0;
            const double sub = g1 * max0(t1 - Dm[sg[c * LP + L]]) + t1;
            const double t2 = PLL - Pf[c];
            const double term = t2 > dm0 ? g1 * (t2 - dm0) : 0.0;
            const double g = ((sub + term) + t2) + qt[c];
            if (g < best) {
              best = g;
              bc = c;
            }
          }
          cuts[0] = 0;
          cuts[1] = (int)(uint8_t)bc;
          cuts[2] = L;
        } else {
          cuts[0] = 0;
          cuts[1] = L;
        }
        // ---- stage_time (cost_model.cpp:88-98), params_in_range
        //      (types.cpp:34-40), per-device parameter ceiling -----------
        const double* tl = p.times + (size_t)cl.pair * L;
        double worst_p = 0.0;
        if (p.rsum_t) {  // the same sums, tabulated per layer range
          const double* rt = p.rsum_t + (size_t)cl.pair * LP * LP;
          for (int j = 0; j < pp; ++j) {
            st[j] = rt[cuts[j] * LP + cuts[j + 1]];
            spar[j] = p.rsum_p[cuts[j] * LP + cuts[j + 1]];
            if (p.has_ceiling) worst_p = std_max(worst_p, spar[j] / tmp);  // (only for the ceiling)
          }
        } else {
          for (int j = 0; j < pp; ++j) {
            double sum = 0.0, ps = 0.0;
            for (int l = cuts[j]; l < cuts[j + 1]; ++l) {
              sum += tl[l];
              ps += p.param[l];
            }
            st[j] = sum;
            spar[j] = ps;
            worst_p = std_max(worst_p, ps / tmp);
          }
        }
        if (p.has_ceiling && worst_p > p.ceiling) fc = AMP_FAIL_CEILING;
      }
      if (fc == 0) {
        // ---- pipeline term (cost_model.cpp:100-120, 145-162, 176-212) ---
        double slowest = st[0];  // std::max_element: first maximum
        for (int j = 1; j < pp; ++j)
          if (slowest < st[j]) slowest = st[j];
        const double g1 = (double)(cl.gas - 1);
        const double* qt = p.qtab + (size_t)w.cls * p.n_codes * L;
        double tr = -CUDART_INF;
        int rr = -1;
        // Without per-candidate edge details the slowest replica's value is
        // enough: t_r = g1*slowest + (((E_r + st_0) + st_1) + ...) is
        // non-decreasing in its edge sum E_r (IEEE additions round
        // monotonically), so max_r t_r = t at max_r E_r — one stage-sum chain
        // instead of one per replica.  (pp == 1: no edges, every replica
        // computes the same t; the strict-'>' scan keeps replica 0.)
        if (!p.all_edge) {
          double emax = -CUDART_INF;
          for (int r = 0; r < (pp == 1 ? 1 : dp); ++r) {
            double esum = 0.0;
            for (int q = 0; q < pp - 1; ++q) {
              int cm = 255;
              for (int s = 0; s < tmp && cm; ++s) {
                const int cc = codeS[nib(perm, (q * dp + r) * tmp + s) * D +
                                     nib(perm, ((q + 1) * dp + r) * tmp + s)];
                cm = cc < cm ? cc : cm;
              }
              esum = esum + qt[(size_t)cm * L + cuts[q + 1]];  // (act[cut-1]*mbs) / b
            }
            emax = emax < esum ? esum : emax;
          }
          double sum = emax;
          for (int j = 0; j < pp; ++j) sum = sum + st[j];
          tr = g1 * slowest + sum;
          rr = 0;  // (not reported without edge details)
        }
        for (int r = 0; p.all_edge && r < (pp == 1 ? 1 : dp); ++r) {
          double sum = 0.0;
          for (int q = 0; q < pp - 1; ++q) {
            int cm = 255;
            for (int s = 0; s < tmp && cm; ++s) {
              const int cc = codeS[nib(perm, (q * dp + r) * tmp + s) * D +
                                   nib(perm, ((q + 1) * dp + r) * tmp + s)];
              cm = cc < cm ? cc : cm;
            }
            sum = sum + qt[(size_t)cm * L + cuts[q + 1]];  // (act[cut-1]*mbs) / b
          }
          for (int j = 0; j < pp; ++j) sum = sum + st[j];
          const double t = g1 * slowest + sum;
          if (t > tr) {  // strict '>' over ascending r: first maximum
            tr = t;
            rr = r;
          }
        }
        // ---- dpsync_time (cost_model.cpp:122-143): groups (stage, shard) -
        double worst = 0.0;
        int bad_group = -1;
        double bad_value = 0.0;
        if (dp != 1 && p.bw_positive) {
          // no group can fail; within a stage every shard group carries the
          // same message, and the rounded time is non-increasing in b, so the
          // stage's maximum is the time of its minimum-bandwidth group: one
          // division per stage (same expression)
          for (int j = 0; j < pp; ++j) {
            int cm = 255;
            for (int s = 0; s < tmp && cm; ++s)
              for (int r1 = 0; r1 < dp && cm; ++r1) {
                const int d1 = nib(perm, (j * dp + r1) * tmp + s);
                for (int r2 = r1 + 1; r2 < dp && cm; ++r2) {
                  const int cc = codeS[d1 * D + nib(perm, (j * dp + r2) * tmp + s)];
                  cm = cc < cm ? cc : cm;
                }
              }
            const double b = p.bwval[cm];
            const double message = spar[j] * p.bpp / tmp;
            worst = std_max(worst, 2.0 * (double)(dp - 1) * message / ((double)dp * b));
          }
        } else if (dp != 1) {
          for (int j = 0, g = 0; j < pp; ++j)
            for (int s = 0; s < tmp; ++s, ++g) {
              int cm = 255;
              for (int r1 = 0; r1 < dp && cm; ++r1) {
                const int d1 = nib(perm, (j * dp + r1) * tmp + s);
                for (int r2 = r1 + 1; r2 < dp && cm; ++r2) {
                  const int cc = codeS[d1 * D + nib(perm, (j * dp + r2) * tmp + s)];
                  cm = cc < cm ? cc : cm;
                }
              }
              const double b = p.bwval[cm];
              if (!(b > 0)) {
                if (bad_group < 0) {
                  bad_group = g;
                  bad_value = b;
                }
              } else {
                const double message = spar[j] * p.bpp / tmp;
                worst = std_max(worst, 2.0 * (double)(dp - 1) * message / ((double)dp * b));
              }
            }
        }
        if (bad_group >= 0) {
          fc = AMP_FAIL_ALLREDUCE_BANDWIDTH;
          fval = bad_value;
        } else {
          pipeline = tr;
          dpsync = worst;
          best_r = rr;
        }
      }
      rec.index = w.index;
      rec.pp = pp;
      rec.dp = dp;
      rec.tmp = tmp;
      rec.mbs = mbs;
      rec.fail_code = fc;
      rec.fail_layer = fc == AMP_FAIL_PROFILE_MISS ? w.fail_layer : -1;
      rec.fail_value = fc == AMP_FAIL_P2P_BANDWIDTH || fc == AMP_FAIL_ALLREDUCE_BANDWIDTH ? fval : 0.0;
      ok = fc == 0;
      rec.pipeline_time = ok ? pipeline : CUDART_NAN;
      rec.dpsync_time = ok ? dpsync : CUDART_NAN;
      rec.total = ok ? pipeline + dpsync : CUDART_NAN;
      if (p.all) p.all[w.out] = rec;
      // the strategy (placement + DP cuts) is kept by the failures raised
      // after evaluate_candidate assigned it (optimizer.cpp:157-171: the
      // parameter ceiling, estimate's all-reduce bandwidth)
      const bool has_strategy = ok || fc == AMP_FAIL_CEILING || fc == AMP_FAIL_ALLREDUCE_BANDWIDTH;
      if (p.all_cuts) {
        int32_t* o = p.all_cuts + w.out * (maxpp + 1);
        for (int q = 0; q <= maxpp; ++q) o[q] = (has_strategy && q <= pp) ? cuts[q] : -1;
      }
      if (p.all_stage) {
        double* o = p.all_stage + w.out * maxpp;
        for (int q = 0; q < maxpp; ++q) o[q] = (ok && q < pp) ? st[q] : CUDART_NAN;
      }
      if (p.all_edge) {  // edges of the slowest replica (cost_model.cpp:203-207)
        double* o = p.all_edge + w.out * maxpp;
        for (int q = 0; q < maxpp; ++q) {
          double v = CUDART_NAN;
          if (ok && q + 1 < pp) {
            int cm = 255;
            for (int s = 0; s < tmp; ++s) {
              const int cc = codeS[nib(perm, (q * dp + best_r) * tmp + s) * D +
                                   nib(perm, ((q + 1) * dp + best_r) * tmp + s)];
              cm = cc < cm ? cc : cm;
            }
            v = p.act[cuts[q + 1] - 1] * mbs / p.bwval[cm];
          }
          o[q] = v;
        }
      }
      if (p.all_place) {
        int32_t* o = p.all_place + w.out * D;
        for (int x = 0; x < D; ++x) o[x] = has_strategy ? nib(perm, x) : -1;
      }
    }
    // ---- warp top-k (rank_records key): lanes that pass the cheap check
    //      against the warp list's k-th entry hand their record to the
    //      leader; the warp lists merge into the CTA list at the end --------
    if (p.k > 0) {
      bool cand = false;
      if (live) {
        const int rf = ok ? 0 : 1;
        const int kf = w_kf[wib];
        const double kt = w_kt[wib];
        cand = rf != kf ? rf < kf : (rf == 0 && rec.total != kt ? rec.total < kt : rec.index < w_ki[wib]);
        if (cand) stage_rec[wib][lane] = rec;
      }
      unsigned m = __ballot_sync(0xffffffffu, cand);
      __syncwarp();
      if (lane == 0 && m) {
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          topk_insert(wtop[wib], wcount[wib], p.k, stage_rec[wib][b]);
        }
        if (wcount[wib] == p.k) {
          w_kf[wib] = wtop[wib][p.k - 1].fail_code != 0;
          w_kt[wib] = wtop[wib][p.k - 1].total;
          w_ki[wib] = wtop[wib][p.k - 1].index;
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
  __syncthreads();
  if (threadIdx.x == 0 && p.k > 0) {  // CTA list (+ the persisted one) <- warp lists
    int n = n_top;
    for (int w = 0; w < kEstTWarps; ++w)
      for (int x = 0; x < wcount[w]; ++x) topk_insert(mytop, n, p.k, wtop[w][x]);
    n_top = n;
  }
  __syncthreads();
  // store the CTA list (padded to k) for the next chunk / the merge
  if (threadIdx.x == 0 && p.k > 0) {
    if (mytop != gtop)
      for (int x = 0; x < n_top; ++x) gtop[x] = mytop[x];
    for (int x = n_top; x < p.k; ++x) {
      amp_record e;
      e.index = ~0ull;
      e.total = e.pipeline_time = e.dpsync_time = CUDART_NAN;
      e.pp = e.dp = e.tmp = e.mbs = 0;
      e.fail_code = -1;
      e.fail_layer = -1;
      e.fail_value = 0.0;
      gtop[x] = e;
    }
  }
}

// Range sums of stage_time / params_in_range (cost_model.cpp:88-98,
// types.cpp:34-40): out[a*(L+1) + b] = ((0.0 + v[a]) + v[a+1]) + ... + v[b-1],
// the reference's loop order, for every range; block n_pairs is the params.
__global__ void k_range_sums(const double* times, const double* param, int L, int n_pairs,
                             double* rt, double* rp) {
  const int LP = L + 1;
  const int pr = blockIdx.x;
  const double* v = pr < n_pairs ? times + (size_t)pr * L : param;
  double* out = pr < n_pairs ? rt + (size_t)pr * LP * LP : rp;
  for (int a = threadIdx.x; a <= L; a += blockDim.x) {
    double sum = 0.0;
    out[a * LP + a] = 0.0;
    for (int b = a + 1; b <= L; ++b) {
      sum += v[b - 1];
      out[a * LP + b] = sum;
    }
  }
}

// The 2-stage DP (pipeline_dp.cpp:70-149 at k = 2; light_cut2's operations
// in order) for every pp == 2 class and every boundary code, once per
// context: its inputs are the class's tables and the code's edge row only.
__global__ void k_cut2_table(const EvalParams p, uint8_t* tab) {
  const int n = p.n_codes;
  const int L = p.L, LP = L + 1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < p.n_cls_total * n;
       t += gridDim.x * blockDim.x) {
    const int c = t / n, code = t % n;
    const ClassDev cl = p.cls[c];
    if (cl.pp != 2 || cl.pp > L) continue;
    const double* Pf = p.prefix + (size_t)cl.pair * LP;
    const double* Dm = p.domain + (size_t)cl.pair * p.nv_stride;
    const uint16_t* sg = p.seg + (size_t)cl.pair * LP * LP;
    const double g1 = (double)(cl.gas - 1);
    const double* qt = p.qtab + ((size_t)c * n + code) * L;
    const double dm0 = Dm[0], PLL = Pf[L], P0 = Pf[0];
    double best = CUDART_INF;
    int bc = -1;
    for (int cut = 1; cut < L; ++cut) {
      const double t1 = Pf[cut] - P0;
      const double sub = g1 * max0(t1 - Dm[sg[cut * LP + L]]) + t1;
      const double t2 = PLL - Pf[cut];
      const double term = t2 > dm0 ? g1 * (t2 - dm0) : 0.0;
      const double g = ((sub + term) + t2) + qt[cut];
      if (g < best) {
        best = g;
        bc = cut;
      }
    }
    tab[t] = (uint8_t)bc;
  }
}

}  // namespace amp
