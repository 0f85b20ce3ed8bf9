// amp_dp_sparse.cuh — the layer-partition DP restricted to the cells the
// answer depends on.
//
// The reference DP (pipeline_dp.cpp:70-149) fills cost[i][j][m] for every
// row i in [j, L] and tolerance index m in [0, M) at every stage j, then
// reads back only the chain that starts at (i = L, j = k, m = 0)
// (backtrack, 134-148).  A cell (i, m) of stage j reads, for each cut c in
// [j-1, i-1], exactly one cell of stage j-1: (c, max(seg(c, i), m)).  So the
// cells that can influence the result form the backward closure
//     N_k     = {(L, 0)}
//     N_{j-1} = {(c, max(seg(c, i), m)) : (i, m) in N_j, c in [j-1, i-1]}
// which depends only on the segment index table of the (tmp, mbs) pair and
// on k — not on placement, edges or gas.  Evaluating the unchanged
// recurrence (same operands, same cut order, same strict '<') on N_j only
// therefore yields bit-identical cuts and cost.  On the reference configs
// the closure is 1.7-5% of the dense table (measured).
//
// "Program" of one (pair, k), built on the device once per search context
// (K0b, two passes: count, then build):
//   cells[]     u32 (i << 16 | m) of N_1 .. N_k, each stage ordered by row
//               descending then m ascending (equal cut counts are adjacent)
//   cellpred[]  u32 per cell of N_j (j >= 2): offset of its predecessor list
//   preds[]     u16 per (cell, cut): index of (c, max(seg(c,i), m)) within
//               N_{j-1}, for c = j-1 .. i-1; each cell's list is padded to a
//               multiple of 4 entries so it can be read with 8-byte loads;
//               padding entries hold |N_{j-1}| (sentinel slot)
//   stage[]     u32 k+1 entries: start of N_j (j = 1..k) within the program's
//               cells, then the end
#pragma once

#include "amp_common.cuh"

namespace amp {

struct ProgDev {
  uint64_t pred_base;   // into preds[]
  uint64_t n_preds;     // total predecessor entries (= inner iterations)
  uint32_t cell_base;   // into cells[] / cellpred[]
  uint32_t stage_base;  // into stage[]
  uint32_t n_cells;     // sum_j |N_j|
  uint32_t max_cells;   // max_j |N_j|
  int32_t k, pair;
  int32_t ok;           // 0: |N_j| exceeds the u16 index range
  int32_t pad;
};

struct ProgBuildParams {
  int32_t L, n_progs, count_only, pad;
  const int32_t* prog_k;     // [n_progs]
  const int32_t* prog_pair;  // [n_progs]
  const PairDev* pairs;
  const uint16_t* seg;       // [n_pairs][(L+1)^2]
  uint32_t* scratch;         // [n_progs][2 * (L+1) * max_M] cell lists
  uint64_t scratch_stride;
  // count pass outputs
  uint32_t* stage_sizes;     // [n_progs][L+1]  |N_j| at [j]
  uint64_t* stage_preds;     // [n_progs][L+1]  predecessor entries of stage j (padded)
  uint64_t* stage_inner;     // [n_progs][L+1]  inner iterations of stage j (unpadded)
  // build pass inputs/outputs
  const ProgDev* progs;
  uint32_t* cells;
  uint32_t* cellpred;
  uint16_t* preds;
  const uint32_t* stage;     // stage starts (host-computed from the count pass)
  const uint64_t* pred_start;  // [n_progs][L+1] start of stage j's preds (relative)
};

// Exclusive block scan over n items in chunks of blockDim; emit(x, prefix)
// is called for every item.  Returns the total on every thread.
template <class F, class G>
__device__ uint64_t block_scan(int n, F value, G emit, uint64_t* sm) {
  const int tid = threadIdx.x, nt = blockDim.x, l = tid & 31, w = tid >> 5;
  uint64_t carry = 0;
  for (int base = 0; base < n; base += nt) {
    const int x = base + tid;
    const uint64_t v = x < n ? value(x) : 0;
    uint64_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (l >= o) incl += y;
    }
    if (l == 31) sm[w] = incl;
    __syncthreads();
    if (w == 0) {
      uint64_t s = l < (nt >> 5) ? sm[l] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (l >= o) s += y;
      }
      if (l < (nt >> 5)) sm[32 + l] = s;
    }
    __syncthreads();
    const uint64_t before = carry + (w > 0 ? sm[32 + w - 1] : 0) + incl - v;
    if (x < n) emit(x, before);
    carry += sm[32 + (nt >> 5) - 1];
    __syncthreads();
  }
  return carry;
}

// K0b: one CTA per program.  Dynamic smem: bitmap [(L+1) * W] u32 and its
// exclusive word prefix [(L+1) * W] u32 in row-descending scan order, plus
// the segment table [(L+1)^2] u16.
__global__ void k_build_progs(ProgBuildParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t scan_sm[64];
  __shared__ uint64_t red64[32];
  const int pg = blockIdx.x, L = p.L, LP = L + 1, tid = threadIdx.x, nt = blockDim.x;
  const int k = p.prog_k[pg];
  const PairDev pr = p.pairs[p.prog_pair[pg]];
  const int M = pr.M;
  const int W = (M + 31) >> 5;
  const int nw = LP * W;
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* wpre = bm + nw;
  uint16_t* seg = reinterpret_cast<uint16_t*>(wpre + nw);
  const uint16_t* gseg = p.seg + (size_t)p.prog_pair[pg] * LP * LP;
  for (int x = tid; x < LP * LP; x += nt) seg[x] = gseg[x];
  uint32_t* A = p.scratch + (size_t)pg * p.scratch_stride;
  uint32_t* B = A + p.scratch_stride / 2;
  if (tid == 0) A[0] = (uint32_t)L << 16;  // N_k = {(L, 0)}
  int n = 1;
  ProgDev pd{};
  if (!p.count_only) pd = p.progs[pg];
  __syncthreads();
  for (int j = k; j >= 1; --j) {
    if (p.count_only) {
      if (tid == 0) p.stage_sizes[(size_t)pg * LP + j] = n;
    } else {
      // write N_j (already in rank order) into the program
      uint32_t* out = p.cells + pd.cell_base + p.stage[pd.stage_base + j - 1];
      for (int x = tid; x < n; x += nt) out[x] = A[x];
    }
    if (j == 1) break;
    // ---- mark N_{j-1} ----------------------------------------------------
    for (int x = tid; x < nw; x += nt) bm[x] = 0;
    __syncthreads();
    uint64_t my_preds = 0, my_inner = 0;
    for (int x = tid; x < n; x += nt) {
      const uint32_t cell = A[x];
      const int i = cell >> 16, m = cell & 0xffff;
      my_preds += (uint64_t)((i - j + 1 + 3) & ~3);  // lists padded to 4 (8-byte loads)
      my_inner += (uint64_t)(i - j + 1);
      for (int c = j - 1; c < i; ++c) {
        const int s = seg[c * LP + i];
        const int mp = s > m ? s : m;
        atomicOr(&bm[c * W + (mp >> 5)], 1u << (mp & 31));
      }
    }
    // total predecessor entries of stage j
    for (int o = 16; o > 0; o >>= 1) {
      my_preds += __shfl_xor_sync(0xffffffffu, my_preds, o);
      my_inner += __shfl_xor_sync(0xffffffffu, my_inner, o);
    }
    if ((tid & 31) == 0) {
      red64[tid >> 5] = my_preds;
      red64[16 + (tid >> 5)] = my_inner;
    }
    __syncthreads();
    if (tid == 0) {
      uint64_t t = 0, ti = 0;
      for (int w = 0; w < (nt >> 5); ++w) {
        t += red64[w];
        ti += red64[16 + w];
      }
      if (p.count_only) {
        p.stage_preds[(size_t)pg * LP + j] = t;
        p.stage_inner[(size_t)pg * LP + j] = ti;
      }
    }
    // ---- rank structure: words in row-descending order ------------------
    // scan position o = (L - row) * W + w
    const uint64_t n_next = block_scan(
        nw, [&](int o) { return (uint64_t)__popc(bm[(L - o / W) * W + (o % W)]); },
        [&](int o, uint64_t before) { wpre[(L - o / W) * W + (o % W)] = (uint32_t)before; }, scan_sm);
    __syncthreads();
    // ---- predecessor lists of N_j (build pass) ---------------------------
    if (!p.count_only) {
      const uint64_t pbase = pd.pred_base + p.pred_start[(size_t)pg * LP + j];
      uint32_t* cpo = p.cellpred + pd.cell_base + p.stage[pd.stage_base + j - 1];
      block_scan(
          n, [&](int x) { return (uint64_t)(((A[x] >> 16) - j + 1 + 3) & ~3u); },
          [&](int x, uint64_t before) {
            const uint32_t cell = A[x];
            const int i = cell >> 16, m = cell & 0xffff;
            cpo[x] = (uint32_t)(p.pred_start[(size_t)pg * LP + j] + before);
            uint16_t* q = p.preds + pbase + before;
            for (int c = j - 1; c < i; ++c) {
              const int s = seg[c * LP + i];
              const int mp = s > m ? s : m;
              const int wi = c * W + (mp >> 5);
              const uint32_t below = bm[wi] & ((1u << (mp & 31)) - 1u);
              q[c - (j - 1)] = (uint16_t)(wpre[wi] + __popc(below));
            }
            // padding entries name the sentinel slot |N_{j-1}| (a +inf
            // value in K_dp multi, so padded cuts never win)
            for (int t = i - (j - 1); t < (((i - j + 1) + 3) & ~3); ++t)
              q[t] = (uint16_t)n_next;
          },
          scan_sm);
    }
    // ---- N_{j-1} list in rank order -------------------------------------
    for (int wi = tid; wi < nw; wi += nt) {
      uint32_t bits = bm[wi];
      uint32_t pos = wpre[wi];
      const int row = wi / W, m0 = (wi % W) << 5;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        B[pos++] = ((uint32_t)row << 16) | (uint32_t)(m0 + b);
      }
    }
    __syncthreads();
    uint32_t* t = A;
    A = B;
    B = t;
    n = (int)n_next;
  }
}

// ---------------------------------------------------------------------------
// K1 (pruned): per-candidate DP over the program of (pair, k)
// ---------------------------------------------------------------------------
//
// V[j & 1][x] holds cost(cell x of N_j); stage j reads V[(j-1) & 1] and
// writes V[j & 1], one barrier per stage.  E[j & 1][c] is stage j's edge cost
// at cut c (boundary j-2), computed one stage ahead.  bpS[x] is the argmin
// cut of cell x (global cell index within the program).
// One cut of the recurrence (pipeline_dp.cpp:122): with t2 = prefix[i] -
// prefix[c] and x = t2 - dom[m], (gas-1) * max(0, x) equals
// (t2 > dom[m]) ? (gas-1) * x : +0.0 exactly (for finite IEEE doubles
// a - b > 0 iff a > b, and NaN compares false on both sides).
__device__ __forceinline__ void cut_step(double sub, double Pi, double2 pe, double dm, double g1,
                                         int c, double& best, int& bc) {
  const double t2 = Pi - pe.x;
  const double term = t2 > dm ? g1 * (t2 - dm) : 0.0;
  const double g = ((sub + term) + t2) + pe.y;
  if (g < best) {
    best = g;
    bc = c;
  }
}

// V[j & 1][x] holds cost(cell x of N_j); stage j reads V[(j-1) & 1] and
// writes V[j & 1], one barrier per stage.  PE[j & 1][c] = {prefix[c],
// edge_j(c)} for stage j (boundary j-2), built one stage ahead.  bpS[x] is
// the argmin cut of cell x (global cell index within the program).
template <class EdgeFn>
__device__ double sparse_solve(const int L, const int k, const int gas,
                               const double* __restrict__ Pf, const double* __restrict__ Dm,
                               const ProgDev& pg, const uint32_t* __restrict__ cells,
                               const uint32_t* __restrict__ cellpred,
                               const uint16_t* __restrict__ preds,
                               const uint32_t* __restrict__ stage, const EdgeFn& edge,
                               double* V0, double* V1, double2* PE0, double2* PE1,
                               uint8_t* __restrict__ bpS, int* cuts) {
  const double g1 = (double)(gas - 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  const uint32_t* cl = cells + pg.cell_base;
  const uint32_t* cpd = cellpred + pg.cell_base;
  const uint16_t* pd = preds + pg.pred_base;
  const uint32_t* ss = stage + pg.stage_base;  // ss[j-1] = start of N_j, ss[k] = end
  // stage 1 (pipeline_dp.cpp:102-107) on N_1; V[1 & 1] = V1
  for (uint32_t x = ss[0] + tid; x < ss[1]; x += nt) {
    const uint32_t cell = cl[x];
    const int i = cell >> 16, m = cell & 0xffff;
    const double t1 = Pf[i] - Pf[0];
    V1[x - ss[0]] = g1 * max0(t1 - Dm[m]) + t1;
  }
  if (k >= 2)
    for (int c = 1 + tid; c < L; c += nt) PE0[c] = make_double2(Pf[c], edge(c, 0));  // stage 2
  __syncthreads();
  for (int j = 2; j <= k; ++j) {
    const double* Vp = (j & 1) ? V0 : V1;
    double* Vc = (j & 1) ? V1 : V0;
    const double2* PE = (j & 1) ? PE1 : PE0;
    if (j < k) {
      double2* PN = (j & 1) ? PE0 : PE1;
      for (int c = j + tid; c < L; c += nt) PN[c] = make_double2(Pf[c], edge(c, j - 1));
    }
    const uint32_t s0 = ss[j - 1], s1 = ss[j];
    const int c0 = j - 1;
    const int n = (int)(s1 - s0);
    if (n * 2 > nt) {
      // one thread per cell; predecessor indices read 4 at a time
      for (uint32_t x = s0 + tid; x < s1; x += nt) {
        const uint32_t cell = cl[x];
        const int i = cell >> 16, m = cell & 0xffff;
        const double dm = Dm[m], Pi = Pf[i];
        const uint2* q = reinterpret_cast<const uint2*>(pd + cpd[x]);
        double best = CUDART_INF;
        int bc = -1;
        int c = c0;
        for (; c + 3 < i; c += 4, ++q) {
          const uint2 w = __ldg(q);
          cut_step(Vp[w.x & 0xffff], Pi, PE[c], dm, g1, c, best, bc);
          cut_step(Vp[w.x >> 16], Pi, PE[c + 1], dm, g1, c + 1, best, bc);
          cut_step(Vp[w.y & 0xffff], Pi, PE[c + 2], dm, g1, c + 2, best, bc);
          cut_step(Vp[w.y >> 16], Pi, PE[c + 3], dm, g1, c + 3, best, bc);
        }
        if (c < i) {
          const uint2 w = __ldg(q);
          cut_step(Vp[w.x & 0xffff], Pi, PE[c], dm, g1, c, best, bc);
          if (c + 1 < i) cut_step(Vp[w.x >> 16], Pi, PE[c + 1], dm, g1, c + 1, best, bc);
          if (c + 2 < i) cut_step(Vp[w.y & 0xffff], Pi, PE[c + 2], dm, g1, c + 2, best, bc);
        }
        Vc[x - s0] = best;
        bpS[x] = (uint8_t)bc;
      }
    } else {
      // few cells (late stages): G lanes per cell split the cut loop by
      // residue, then a lexicographic (value, cut) butterfly combine — equal
      // to the sequential strict-'<' scan.
      int G = 2;
      while (G < 32 && n * G * 2 <= nt) G <<= 1;
      const int gl = tid & (G - 1);
      const int per = nt / G;
      for (int base = 0; base < n; base += per) {  // uniform trip count
        const int xi = base + tid / G;
        double best = CUDART_INF;
        int bc = -1;
        if (xi < n) {
          const uint32_t x = s0 + xi;
          const uint32_t cell = cl[x];
          const int i = cell >> 16, m = cell & 0xffff;
          const double dm = Dm[m], Pi = Pf[i];
          const uint16_t* q = pd + cpd[x] + gl;
          for (int c = c0 + gl; c < i; c += G, q += G)
            cut_step(Vp[__ldg(q)], Pi, PE[c], dm, g1, c, best, bc);
        }
        for (int o = G >> 1; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
          if (ov < best || (ov == best && oc < bc)) {
            best = ov;
            bc = oc;
          }
        }
        if (xi < n && gl == 0) {
          Vc[xi] = best;
          bpS[s0 + xi] = (uint8_t)bc;
        }
      }
    }
    __syncthreads();
  }
  double cost = 0.0;
  if (tid == 0) {
    cost = ((k & 1) ? V1 : V0)[0];
    cuts[k] = L;
    uint32_t x = ss[k - 1];  // N_k = {(L, 0)}
    for (int j = k; j >= 2; --j) {
      const int c = bpS[x];
      cuts[j - 1] = c;
      x = ss[j - 2] + pd[cpd[x] + (c - (j - 1))];
    }
    cuts[0] = 0;
  }
  __syncthreads();
  return cost;
}

}  // namespace amp
