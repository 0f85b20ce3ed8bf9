// amp_kernels.cuh — sm_100a kernels of the strategy search.
//
//   K0 k_pair_tables   one CTA per distinct (tmp, mbs): layer times
//                      (LayerTimeResolver, cost_model.cpp:74-86), prefix
//                      sums, tolerance domain (bitonic sort + unique in
//                      smem), segment index (pipeline_dp.cpp:39-91).
//   K1+K2 k_evaluate   persistent CTAs; per candidate: placement, stage
//                      boundary bandwidths, the tolerance-indexed DP as a
//                      shared-memory row wavefront (pipeline_dp.cpp:70-149),
//                      ceiling check, estimate (cost_model.cpp:176-212),
//                      record + CTA-local top-k.
//   K3 k_merge_topk    deterministic k-round block argmin of the CTA lists.
//
// Numerics: compiled with -fmad=false; every sum is evaluated in the
// reference's order (SURVEY.md §8(a) numerics contract).  min/max
// reductions are exact and may be reordered; argmin/argmax ties are broken
// toward the reference's sequential winner (lowest cut / lowest replica).
#pragma once

#include <math_constants.h>

#include "amp_common.cuh"
#include "amp_dp_sparse.cuh"

namespace amp {


// ---------------------------------------------------------------------------
// block helpers
// ---------------------------------------------------------------------------

// Block-wide min with std_min semantics (NaN never enters); all threads get it.
__device__ double block_min(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = std_min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? red[l] : CUDART_INF;
    for (int o = 16; o > 0; o >>= 1) v = std_min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

// Block-wide (max value, lowest index) over candidates; NaN/-1 idx skipped.
__device__ void block_argmax(double& v, int& idx, double* red, int* redi) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (oi >= 0 && (idx < 0 || ov > v || (ov == v && oi < idx))) {
      v = ov;
      idx = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    red[w] = v;
    redi[w] = idx;
  }
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? red[l] : -CUDART_INF;
    idx = l < (int)(blockDim.x >> 5) ? redi[l] : -1;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (oi >= 0 && (idx < 0 || ov > v || (ov == v && oi < idx))) {
        v = ov;
        idx = oi;
      }
    }
    if (l == 0) {
      red[0] = v;
      redi[0] = idx;
    }
  }
  __syncthreads();
  v = red[0];
  idx = redi[0];
  __syncthreads();
}

__device__ int block_min_int(int v, int* redi) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) redi[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? redi[l] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) redi[0] = v;
  }
  __syncthreads();
  v = redi[0];
  __syncthreads();
  return v;
}

// ---------------------------------------------------------------------------
// tolerance domain (pipeline_dp.cpp:55-68) + segment index (83-91)
// ---------------------------------------------------------------------------

// Builds the sorted unique domain of {0} U {P[b]-P[a]} into dom_out[0..M)
// and seg_out[a*(L+1)+b].  `vals` is smem scratch of npow2 doubles
// (npow2 >= 1 + L(L+1)/2, power of two).  Returns M (all threads).
__device__ int build_domain(const double* Pf, int L, double* vals, int npow2, double* dom_out,
                            uint16_t* seg_out, int* redi) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nv = 1 + L * (L + 1) / 2;
  for (int x = tid; x < npow2; x += nt) {
    double v = CUDART_INF;
    if (x == 0) {
      v = 0.0;
    } else if (x < nv) {
      // x-1 enumerates (a, b), a < b, row-major over a (same multiset as the
      // reference's push order; the order is irrelevant after sorting).
      int r = x - 1, a = 0, len = L;
      while (r >= len) {
        r -= len;
        ++a;
        --len;
      }
      const int b = a + 1 + r;
      v = Pf[b] - Pf[a];
    }
    vals[x] = v;
  }
  __syncthreads();
  // bitonic sort ascending
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int x = tid; x < (npow2 >> 1); x += nt) {
        const int lo = 2 * x - (x & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const double a = vals[lo], b = vals[hi];
        if ((a > b) == up) {
          vals[lo] = b;
          vals[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  // unique (exact ==): chunked scan, one contiguous chunk per thread
  const int chunk = (nv + nt - 1) / nt;
  const int c0 = tid * chunk, c1 = min(nv, c0 + chunk);
  int cnt = 0;
  for (int x = c0; x < c1; ++x)
    if (x == 0 || !(vals[x] == vals[x - 1])) ++cnt;
  // exclusive scan of cnt over threads (warp shuffles + smem)
  int incl = cnt;
  const int l = tid & 31, w = tid >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (l >= o) incl += y;
  }
  __syncthreads();
  if (l == 31) redi[w] = incl;
  __syncthreads();
  if (w == 0) {
    int s = l < (nt >> 5) ? redi[l] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (l >= o) s += y;
    }
    if (l < (nt >> 5)) redi[32 + l] = s;  // inclusive per warp
  }
  __syncthreads();
  int pos = incl - cnt + (w > 0 ? redi[32 + w - 1] : 0);
  const int M = redi[32 + (nt >> 5) - 1];
  for (int x = c0; x < c1; ++x)
    if (x == 0 || !(vals[x] == vals[x - 1])) dom_out[pos++] = vals[x];
  __syncthreads();
  // seg_index: lower_bound of each segment sum (exact member of the domain)
  for (int x = tid; x < (L + 1) * (L + 1); x += nt) {
    const int a = x / (L + 1), b = x % (L + 1);
    int idx = 0;
    if (a < b) {
      const double v = Pf[b] - Pf[a];
      int lo = 0, hi = M;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (dom_out[mid] < v) lo = mid + 1;
        else hi = mid;
      }
      idx = lo;
    }
    seg_out[x] = (uint16_t)idx;
  }
  __syncthreads();
  return M;
}

// ---------------------------------------------------------------------------
// K1: tolerance-indexed layer-partition DP (pipeline_dp.cpp:70-149)
// ---------------------------------------------------------------------------
//
// Stage slice C[i][m] (i in [0, L], m in [0, M)) lives in shared memory (or
// in a per-CTA global buffer for large M).  Each thread OWNS domain columns
// m and computes stage j of its column in place, rows i descending: row i at
// stage j reads rows cut < i of stage j-1 which, in the thread's own column,
// have not been overwritten yet.  The only cross-column read of the
// recurrence is cost[cut][j-1][max(seg(cut,i), m)] when m < seg(cut,i); that
// value, U(cut,i) = C[cut][seg(cut,i)], is uniform over m and is gathered
// once per stage into the table W[i][cut] = {t2, edge, U} together with the
// segment time t2 = prefix[i] - prefix[cut] and the stage's edge cost.  So a
// stage needs two barriers (table build, column sweep) instead of one per
// row, and the inner loop reads one uniform 32-byte entry plus (on the
// m >= seg branch) one own-column double.
//
// With non-negative layer times seg(cut, i) is non-increasing in cut, so for
// each (i, m) the cut range [j-1, i) splits at c* into an "m < seg" prefix
// (U branch) and an "m >= seg" suffix (own-column branch); c* is walked down
// incrementally as i decreases.  The two loops run in ascending cut order
// with a strict '<', so the smallest cut wins ties exactly like the
// reference (pipeline_dp.cpp:118-127).  Exactness of the branch forms:
//   m <  seg: t2 - dom[m] > 0, so max(0, .) = t2 - dom[m];
//   m >= seg: t2 - dom[m] <= 0, so (gas-1)*max(0, .) = +0.0 and
//             sub + 0.0 == sub (sub is never -0.0, t2 never -0.0).
// Backpointers (one byte per (j, i, m)) go to global scratch; thread 0
// backtracks from (L, k, m = 0).
struct __align__(16) WEnt {
  double t2;  // prefix[i] - prefix[cut]
  double e;   // edge cost at `cut` for the current stage boundary
  double u;   // C_{j-1}[cut][seg(cut, i)]
  double pad;
};

// Lexicographic (value, cut) argmin accumulator.  Several accumulators,
// each fed its cuts in ascending order, combined with comb(), equal the
// reference's single sequential strict-'<' scan (first cut attaining the
// minimum; NaN never selected); they break the DSETP->FSEL dependency chain.
struct ArgMin {
  double v;
  int c;
};
__device__ __forceinline__ void upd(ArgMin& a, double g, int c) {
  if (g < a.v) {
    a.v = g;
    a.c = c;
  }
}
__device__ __forceinline__ ArgMin comb(const ArgMin& a, const ArgMin& b) {
  return (b.v < a.v || (b.v == a.v && b.c < a.c)) ? b : a;
}

template <class EdgeFn>
__device__ double dp_solve(const int L, const int k, const int gas, const int M,
                           const double* __restrict__ Pf, const double* __restrict__ Dm,
                           const uint16_t* __restrict__ seg, const EdgeFn& edge, double* C,
                           WEnt* W, double* E, const bool monotone, uint8_t* __restrict__ bp,
                           int* cuts) {
  const double g1 = (double)(gas - 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int LP = L + 1;
  // base case j = 1 (102-107): t1 = between(0, i) = prefix[i] - prefix[0]
  for (int m = tid; m < M; m += nt) {
    const double dm = Dm[m];
    double* col = C + m;
    for (int i = 1; i <= L; ++i) {
      const double t1 = Pf[i] - Pf[0];
      col[i * M] = g1 * max0(t1 - dm) + t1;
    }
  }
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  for (int j = 2; j <= k; ++j) {
    // ---- per-stage uniform table W[i][cut], cut in [j-1, L), i in (cut, L]
    const int c0 = j - 1;
    for (int c = c0 + tid; c < L; c += nt) E[c] = edge(c, j - 2);
    __syncthreads();  // E ready; previous stage's columns complete
    for (int i = j + warp; i <= L; i += nwarp) {  // one warp per row
      const double Pi = Pf[i];
      for (int c = c0 + lane; c < i; c += 32) {
        WEnt w;
        w.t2 = Pi - Pf[c];
        w.e = E[c];
        w.u = C[c * M + seg[c * LP + i]];
        w.pad = 0.0;
        W[i * L + c] = w;
      }
    }
    __syncthreads();
    uint8_t* bpj = bp + (size_t)j * LP * M;
    for (int m = tid; m < M; m += nt) {
      const double dm = Dm[m];
      const double* Cm = C + m;
      double* Crow = C + L * M + m;           // C[i][m], i = L, L-1, ...
      uint8_t* brow = bpj + L * M + m;
      const WEnt* Wi = W + L * L;             // row i of the cut table
      const uint16_t* segi = seg + L;         // &seg[0 * LP + i]
      int cs = L;  // c*: first cut of the m >= seg suffix (non-increasing in i)
      for (int i = L; i >= j; --i, Crow -= M, brow -= M, Wi -= L, --segi) {
        double best = CUDART_INF;
        int bc = -1;
        if (monotone) {
          if (cs > i) cs = i;
          while (cs > c0 && (int)segi[(cs - 1) * LP] <= m) --cs;
          const WEnt* w = Wi + c0;
          const WEnt* wu = Wi + cs;
          int c = c0;
#pragma unroll 2
          for (; w < wu; ++w, ++c) {  // m < seg(c, i): U branch
            const double4 x = *reinterpret_cast<const double4*>(w);  // t2, e, u
            const double g = ((x.z + g1 * (x.x - dm)) + x.x) + x.y;
            if (g < best) {
              best = g;
              bc = c;
            }
          }
          const WEnt* we = Wi + i;
          const double* cp = Cm + c * M;
#pragma unroll 2
          for (; w < we; ++w, ++c, cp += M) {  // m >= seg(c, i): own column
            const double2 te = *reinterpret_cast<const double2*>(w);
            const double g = (*cp + te.x) + te.y;
            if (g < best) {
              best = g;
              bc = c;
            }
          }
        } else {  // general order (negative layer times): test per cut
          for (int c = c0; c < i; ++c) {
            const WEnt w = Wi[c];
            const int s = segi[c * LP];
            const double sub = s > m ? w.u : Cm[c * M];
            const double g = ((sub + g1 * max0(w.t2 - dm)) + w.t2) + w.e;
            if (g < best) {
              best = g;
              bc = c;
            }
          }
        }
        *Crow = best;
        *brow = (uint8_t)bc;
      }
    }
  }
  __syncthreads();
  double cost = 0.0;
  if (tid == 0) {
    cost = C[(size_t)L * M + 0];
    cuts[k] = L;
    int i = L, m = 0;
    for (int j = k; j >= 2; --j) {
      const int cut = bp[((size_t)j * LP + i) * M + m];
      cuts[j - 1] = cut;
      const int s = seg[cut * LP + i];
      m = s > m ? s : m;
      i = cut;
    }
    cuts[0] = 0;
  }
  __syncthreads();
  return cost;
}

// ---------------------------------------------------------------------------
// K0: per-(tmp, mbs) tables
// ---------------------------------------------------------------------------

struct TableParams {
  int32_t L, n_pairs, npow2;
  int32_t fallback_enabled;
  const int32_t* pair_tmp;      // [n_pairs]
  const int32_t* pair_mbs;      // [n_pairs]
  const double* cube;           // [n_pairs][L] profile seconds
  const uint8_t* cube_hit;      // [n_pairs][L]
  const double* flops;          // [L]
  const uint8_t* flops_ok;      // [L]
  const double* act;            // [L-1]
  double device_flops, tmp_bandwidth;
  PairDev* pairs;
  double* times;
  double* prefix;
  double* domain;
  uint16_t* seg;
  int32_t nv_stride;
};

__global__ void k_pair_tables(TableParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* vals = reinterpret_cast<double*>(smem_raw);
  double* Pf = vals + p.npow2;
  __shared__ int redi[64];
  const int pr = blockIdx.x, L = p.L, tid = threadIdx.x;
  const int tmp = p.pair_tmp[pr], mbs = p.pair_mbs[pr];
  double* times = p.times + (size_t)pr * L;
  // LayerTimeResolver::layer_time (cost_model.cpp:74-86): profile hit, else
  // analytic fallback (61-68) with allreduce_time (40-52), else miss.
  int my_fail = 0x7fffffff;  // (layer << 3) | code, min = first failing layer
  for (int l = tid; l < L; l += blockDim.x) {
    double t = 0.0;
    int code = 0;
    if (p.cube_hit[(size_t)pr * L + l]) {
      t = p.cube[(size_t)pr * L + l];
    } else if (!p.fallback_enabled || !p.flops_ok[l]) {
      code = AMP_FAIL_PROFILE_MISS;
    } else {
      const double vol = L <= 1 ? 0.0 : (l < L - 1 ? p.act[l] : p.act[l - 1]);
      const double message = vol * mbs;
      const double compute = (double)mbs * p.flops[l] / ((double)tmp * p.device_flops);
      double ar = 0.0;
      if (tmp != 1) {
        if (!(p.tmp_bandwidth > 0)) code = AMP_FAIL_ALLREDUCE_BANDWIDTH;
        else ar = 2.0 * (double)(tmp - 1) * message / ((double)tmp * p.tmp_bandwidth);
      }
      t = compute + ar;
    }
    times[l] = t;
    if (code) my_fail = min(my_fail, (l << 3) | code);
  }
  const int fail = block_min_int(my_fail, redi);
  if (tid == 0) {
    PairDev d;
    d.tmp = tmp;
    d.mbs = mbs;
    d.M = 0;
    d.fail_code = fail == 0x7fffffff ? 0 : (fail & 7);
    d.fail_layer = fail == 0x7fffffff ? -1 : (fail >> 3);
    d.monotone = 1;
    d.fail_value = d.fail_code == AMP_FAIL_ALLREDUCE_BANDWIDTH ? p.tmp_bandwidth : 0.0;
    p.pairs[pr] = d;
  }
  __syncthreads();
  if (fail != 0x7fffffff) return;  // every candidate of this pair fails
  // prefix sums, strictly left to right (pipeline_dp.cpp:39-44)
  if (tid == 0) {
    double s = 0.0;
    Pf[0] = 0.0;
    int mono = 1;  // non-negative layer times: seg(cut, i) monotone in cut
    for (int l = 0; l < L; ++l) {
      if (!(times[l] >= 0.0)) mono = 0;
      s = s + times[l];
      Pf[l + 1] = s;
    }
    p.pairs[pr].monotone = mono;
  }
  __syncthreads();
  for (int x = tid; x <= L; x += blockDim.x) p.prefix[(size_t)pr * (L + 1) + x] = Pf[x];
  const int M = build_domain(Pf, L, vals, p.npow2, p.domain + (size_t)pr * p.nv_stride,
                             p.seg + (size_t)pr * (L + 1) * (L + 1), redi);
  if (tid == 0) p.pairs[pr].M = M;
}

// ---------------------------------------------------------------------------
// K1+K2: persistent candidate evaluation
// ---------------------------------------------------------------------------

struct EdgeFromBandwidth {  // placement_edge_cost (optimizer.cpp:130-139)
  const double* act;
  const double* bwq;
  int mbs;
  __device__ double operator()(int cut, int q) const { return act[cut - 1] * mbs / bwq[q]; }
};

__device__ void topk_insert(amp_record* list, int& n, int k, const amp_record& r) {
  if (n == k && !rank_less(r, list[k - 1])) return;
  int pos = n < k ? n : k - 1;
  while (pos > 0 && rank_less(r, list[pos - 1])) {
    list[pos] = list[pos - 1];
    --pos;
  }
  list[pos] = r;
  if (n < k) ++n;
}

// ---------------------------------------------------------------------------
// K3: deterministic merge (k rounds of block argmin under rank_less)
// ---------------------------------------------------------------------------

// The input is n / k sorted lists of k records (CTA lists of K_est, or the
// all-gathered per-rank lists), each padded with empty slots at its end.
// k rounds of a block argmin over the list heads (a k-way merge), keys of
// the heads cached in shared memory.  Deterministic: ties cannot occur
// between distinct candidate indices.
constexpr int kMergeMaxLists = 1024;

__device__ __forceinline__ bool key_less(int ca, double ta, uint64_t ia, int cb, double tb,
                                         uint64_t ib) {
  if (ca != cb) return ca < cb;
  if (ca == 0 && ta != tb) return ta < tb;
  return ia < ib;
}

__global__ void k_merge_topk(const amp_record* in, int n, int k, amp_record* out,
                             unsigned char* /*unused*/) {
  __shared__ int hcls[kMergeMaxLists];
  __shared__ double htot[kMergeMaxLists];
  __shared__ uint64_t hidx[kMergeMaxLists];
  __shared__ int hpos[kMergeMaxLists];
  __shared__ int wbest[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nl = n / k;
  auto load_head = [&](int l) {
    const int pos = hpos[l];
    if (pos >= k) {
      hcls[l] = 3;  // exhausted: after everything
      htot[l] = 0.0;
      hidx[l] = ~0ull;
      return;
    }
    const amp_record& r = in[(size_t)l * k + pos];
    hcls[l] = r.fail_code < 0 ? 3 : (r.fail_code != 0 ? 1 : 0);
    htot[l] = r.total;
    hidx[l] = r.index;
  };
  for (int l = tid; l < nl; l += nt) {
    hpos[l] = 0;
    load_head(l);
  }
  __syncthreads();
  for (int round = 0; round < k; ++round) {
    int bl = -1;
    for (int l = tid; l < nl; l += nt)
      if (bl < 0 || key_less(hcls[l], htot[l], hidx[l], hcls[bl], htot[bl], hidx[bl])) bl = l;
    for (int o = 16; o > 0; o >>= 1) {
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ol >= 0 && (bl < 0 || key_less(hcls[ol], htot[ol], hidx[ol], hcls[bl], htot[bl], hidx[bl])))
        bl = ol;
    }
    if ((tid & 31) == 0) wbest[tid >> 5] = bl;
    __syncthreads();
    if (tid == 0) {
      int b = -1;
      for (int w = 0; w < (nt >> 5); ++w) {
        const int ol = wbest[w];
        if (ol >= 0 && (b < 0 || key_less(hcls[ol], htot[ol], hidx[ol], hcls[b], htot[b], hidx[b])))
          b = ol;
      }
      if (b >= 0 && hcls[b] != 3) {
        out[round] = in[(size_t)b * k + hpos[b]];
        ++hpos[b];
        load_head(b);
      } else {
        amp_record e;
        e.index = ~0ull;
        e.total = e.pipeline_time = e.dpsync_time = CUDART_NAN;
        e.pp = e.dp = e.tmp = e.mbs = 0;
        e.fail_code = -1;
        e.fail_layer = -1;
        e.fail_value = 0.0;
        out[round] = e;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// standalone DP batch (amp_dp_solve_batch)
// ---------------------------------------------------------------------------

struct DpBatchItem {
  int32_t L, stages, gas, status;
  const double* times;
  const double* edges;
};

struct EdgeFromTable {
  const double* e;
  int L;
  __device__ double operator()(int cut, int q) const { return e[(size_t)q * L + cut]; }
};

struct DpBatchParams {
  const DpBatchItem* items;
  int32_t n, max_L, max_k, npow2;
  int32_t cut_stride;
  int32_t* cuts_out;
  double* cost_out;
  uint8_t* bp;
  uint64_t bp_stride;
  double* slice;
  uint64_t slice_stride;
  double* domain;  // per-CTA scratch [npow2]
  uint16_t* seg;   // per-CTA scratch [(max_L+1)^2]
  WEnt* wtab;      // per-CTA scratch [(max_L+1) * max_L]
};

__global__ void k_dp_batch(DpBatchParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int redi[64];
  double* vals = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x;
  double* Pf = vals + p.npow2;
  double* E = Pf + p.max_L + 1;
  int* cuts = reinterpret_cast<int*>(E + p.max_L);
  WEnt* W = p.wtab + (size_t)blockIdx.x * (p.max_L + 1) * p.max_L;
  double* dom = p.domain + (size_t)blockIdx.x * p.npow2;
  uint16_t* seg = p.seg + (size_t)blockIdx.x * (p.max_L + 1) * (p.max_L + 1);
  double* C = p.slice + (size_t)blockIdx.x * p.slice_stride;
  uint8_t* bp = p.bp + (size_t)blockIdx.x * p.bp_stride;
  for (int inst = blockIdx.x; inst < p.n; inst += gridDim.x) {
    const DpBatchItem it = p.items[inst];
    if (it.status != 0) continue;
    const int L = it.L;
    __shared__ int mono;
    if (tid == 0) {
      double s = 0.0;
      Pf[0] = 0.0;
      mono = 1;
      for (int l = 0; l < L; ++l) {
        if (!(it.times[l] >= 0.0)) mono = 0;
        s = s + it.times[l];
        Pf[l + 1] = s;
      }
    }
    __syncthreads();
    int np2 = 2;
    while (np2 < 1 + L * (L + 1) / 2) np2 <<= 1;
    const int M = build_domain(Pf, L, vals, np2, dom, seg, redi);
    EdgeFromTable ef{it.edges, L};
    const double cost = dp_solve(L, it.stages, it.gas, M, Pf, dom, seg, ef, C, W, E, mono != 0, bp, cuts);
    if (tid == 0) {
      p.cost_out[inst] = cost;
      for (int q = 0; q <= it.stages; ++q) p.cuts_out[(size_t)inst * p.cut_stride + q] = cuts[q];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// FP64 add throughput probe (roofline denominator)
// ---------------------------------------------------------------------------

__global__ void k_dadd_peak(double* out, int iters, double a) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = x0 + a;
      x1 = x1 + a;
      x2 = x2 + a;
      x3 = x3 + a;
      x4 = x4 + a;
      x5 = x5 + a;
      x6 = x6 + a;
      x7 = x7 + a;
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 1234.5) out[0] = s;
}

}  // namespace amp
