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
// (K0b):
//   cells[]     u32 (i << 16 | m) of N_1 .. N_k, each stage ordered by row
//               descending then m ascending (equal cut counts are adjacent)
//   cellpred[]  u32 per cell of N_j (j >= 2): offset of its predecessor list
//   preds[]     u16 per (cell, cut): index of (c, max(seg(c,i), m)) within
//               N_{j-1}, for c = j-1 .. i-1; each cell's list is padded to a
//               multiple of 4 entries so it can be read with 8-byte loads;
//               padding entries hold |N_{j-1}| (sentinel slot)
//   stage[]     u32 k+1 entries: start of N_j (j = 1..k) within the program's
//               cells, then the end
// Two kernels: K0b-closure (one CTA per program, sequential over the stages)
// computes each N_j as a bitmap [row][m / 32] word-parallel:
//   row c of N_{j-1} = OR over the rows i > c of N_j of
//       (row i's bits above seg(c,i))  |  (bit seg(c,i) if row i has a bit <= seg(c,i))
// (= { max(seg(c,i), m) : (i, m) in N_j }), stores every stage's bitmap and
// its sizes; K0b-emit (one CTA per (program, stage, slice of 4096 cells),
// all in parallel) writes the cells, their list offsets and the predecessor
// indices (rank of (c, mp) in N_{j-1}: a word prefix plus a popcount).
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
  int32_t L, n_progs;
  const int32_t* prog_k;     // [n_progs]
  const int32_t* prog_pair;  // [n_progs]
  const PairDev* pairs;
  const uint16_t* seg;       // [n_pairs][(L+1)^2]
  uint32_t* bm;              // stage bitmaps: program g, stage j at bm_off[g] + (j-1) * (L+1) * W_g
  const uint64_t* bm_off;    // [n_progs]
  // closure outputs
  uint32_t* stage_sizes;     // [n_progs][L+1]  |N_j| at [j]
  uint64_t* stage_preds;     // [n_progs][L+1]  predecessor entries of stage j (padded)
  uint64_t* stage_inner;     // [n_progs][L+1]  inner iterations of stage j (unpadded)
  // emit inputs / outputs
  const ProgDev* progs;
  uint32_t* cells;
  uint32_t* cellpred;
  uint16_t* preds;
  const uint32_t* stage;     // stage starts (host-computed from the closure sizes)
  const uint64_t* pred_start;  // [n_progs][L+1] start of stage j's preds (relative)
  const uint4* items;        // emit work list {g, j, first cell, end cell}
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

constexpr uint32_t kEmitSlice = 4096;  // cells per K0b-emit CTA

__device__ __forceinline__ int pad4(int x) { return (x + 3) & ~3; }

// Bits of word w (m = 32 w .. 32 w + 31) strictly above m = s.
__device__ __forceinline__ uint32_t bits_above(int s, int w) {
  const int lo = w << 5;
  if (s < lo) return ~0u;
  if (s >= lo + 31) return 0u;
  return ~((2u << (s - lo)) - 1u);
}

// Exclusive word prefix of a stage bitmap in rank order (rows descending,
// words ascending): wpre[row * W + w] = cells before that word.  Returns the
// stage size.
__device__ uint32_t bitmap_rank(const uint32_t* bm, uint32_t* wpre, int L, int W, uint64_t* sm) {
  const int nw = (L + 1) * W;
  return (uint32_t)block_scan(
      nw, [&](int o) { return (uint64_t)__popc(bm[(L - o / W) * W + (o % W)]); },
      [&](int o, uint64_t before) { wpre[(L - o / W) * W + (o % W)] = (uint32_t)before; }, sm);
}

// K0b-closure: one CTA per program.  Dynamic smem: two stage bitmaps
// [(L+1) * W] u32, the segment table [(L+1)^2] u16, the non-empty rows of
// the current stage and their lowest m.
__global__ void __launch_bounds__(512) k_prog_closure(ProgBuildParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t red[3][32];
  __shared__ int n_rows;
  const int g = blockIdx.x, L = p.L, LP = L + 1, tid = threadIdx.x, nt = blockDim.x;
  const int k = p.prog_k[g];
  const int M = p.pairs[p.prog_pair[g]].M;
  const int W = (M + 31) >> 5, nw = LP * W;
  uint32_t* cur = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* nxt = cur + nw;
  uint16_t* seg = reinterpret_cast<uint16_t*>(nxt + nw);
  int* rows = reinterpret_cast<int*>(seg + ((LP * LP + 1) & ~1));  // [LP] non-empty rows, ascending
  int* rmin = rows + LP;                                            // [LP] lowest m of each listed row
  int* rlo = rmin + LP;                                             // [LP] lowest m of row i (-1: empty)
  const uint16_t* gseg = p.seg + (size_t)p.prog_pair[g] * LP * LP;
  for (int x = tid; x < LP * LP; x += nt) seg[x] = gseg[x];
  for (int x = tid; x < nw; x += nt) cur[x] = 0;
  __syncthreads();
  if (tid == 0) cur[L * W] = 1u;  // N_k = {(L, 0)}
  __syncthreads();
  for (int j = k; j >= 1; --j) {
    uint32_t* out = p.bm + p.bm_off[g] + (size_t)(j - 1) * nw;
    for (int x = tid; x < nw; x += nt) out[x] = cur[x];
    // sizes of N_j: cells, padded and unpadded predecessor entries
    uint64_t cn = 0, pn = 0, in = 0;
    for (int i = tid; i <= L; i += nt) {
      uint32_t c = 0;
      int lo = -1;
      for (int w = 0; w < W; ++w) {
        const uint32_t b = cur[i * W + w];
        if (b && lo < 0) lo = (w << 5) + __ffs(b) - 1;
        c += __popc(b);
      }
      rlo[i] = lo;
      cn += c;
      if (i >= j) {
        pn += (uint64_t)c * pad4(i - j + 1);
        in += (uint64_t)c * (i - j + 1);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      cn += __shfl_xor_sync(0xffffffffu, cn, o);
      pn += __shfl_xor_sync(0xffffffffu, pn, o);
      in += __shfl_xor_sync(0xffffffffu, in, o);
    }
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = cn;
      red[1][tid >> 5] = pn;
      red[2][tid >> 5] = in;
    }
    __syncthreads();
    if (tid == 0) {
      uint64_t a = 0, b = 0, c = 0;
      for (int w = 0; w < (nt >> 5); ++w) {
        a += red[0][w];
        b += red[1][w];
        c += red[2][w];
      }
      p.stage_sizes[(size_t)g * LP + j] = (uint32_t)a;
      if (j >= 2) {
        p.stage_preds[(size_t)g * LP + j] = b;
        p.stage_inner[(size_t)g * LP + j] = c;
      }
    }
    if (tid < 32) {  // the non-empty rows (ascending) and their lowest m
      int nr = 0;
      for (int b = 0; b <= L; b += 32) {
        const int i = b + (tid & 31);
        const bool ne = i <= L && rlo[i] >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, ne);
        if (ne) {
          const int at = nr + __popc(bal & ((1u << (tid & 31)) - 1u));
          rows[at] = i;
          rmin[at] = rlo[i];
        }
        nr += __popc(bal);
      }
      if (tid == 0) n_rows = nr;
    }
    __syncthreads();
    if (j == 1) break;
    // N_{j-1}: rows c in [j-1, L-1], word-parallel
    const int nr = n_rows;
    for (int x = tid; x < nw; x += nt) {
      const int c = x / W, w = x - c * W;
      uint32_t word = 0;
      if (c >= j - 1 && c < L) {
        for (int r = 0; r < nr; ++r) {
          const int i = rows[r];
          if (i <= c) continue;
          const int s = seg[c * LP + i];
          word |= cur[i * W + w] & bits_above(s, w);
          if ((s >> 5) == w && rmin[r] <= s) word |= 1u << (s & 31);
        }
      }
      nxt[x] = word;
    }
    __syncthreads();
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
  }
}

// K0b-emit: one CTA per work item {g, j, x0, x1}: the cells of N_j with rank
// in [x0, x1), their predecessor-list offsets and (j >= 2) the lists.
// Dynamic smem: bitmap + word prefix of N_j and of N_{j-1} [(L+1) * W] u32
// each, the segment table, the per-row list offsets of N_j.
__global__ void __launch_bounds__(512) k_prog_emit(ProgBuildParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t scan_sm[64];
  const uint4 it = p.items[blockIdx.x];
  const int g = (int)it.x, j = (int)it.y;
  const uint32_t x0 = it.z, x1 = it.w;
  const int L = p.L, LP = L + 1, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  const int M = p.pairs[p.prog_pair[g]].M;
  const int W = (M + 31) >> 5, nw = LP * W;
  uint32_t* bmj = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* wpj = bmj + nw;
  uint32_t* bmp = wpj + nw;
  uint32_t* wpp = bmp + nw;
  uint64_t* rowoff = reinterpret_cast<uint64_t*>(wpp + nw);  // (4 nw words: 8-byte aligned)  // [LP] first pred entry of row i's cells
  uint32_t* scell = reinterpret_cast<uint32_t*>(rowoff + LP);  // [kEmitSlice] the slice's cells
  uint32_t* scpo = scell + kEmitSlice;                           // [kEmitSlice] their list offsets
  uint16_t* seg = reinterpret_cast<uint16_t*>(scpo + kEmitSlice);
  const uint32_t* gbm = p.bm + p.bm_off[g] + (size_t)(j - 1) * nw;
  for (int x = tid; x < nw; x += nt) bmj[x] = gbm[x];
  if (j >= 2) {
    for (int x = tid; x < nw; x += nt) bmp[x] = gbm[x - nw];
    const uint16_t* gseg = p.seg + (size_t)p.prog_pair[g] * LP * LP;
    for (int x = tid; x < LP * LP; x += nt) seg[x] = gseg[x];
  }
  __syncthreads();
  const uint32_t n_cur = bitmap_rank(bmj, wpj, L, W, scan_sm);
  __syncthreads();
  uint32_t n_prev = 0;
  if (j >= 2) {
    n_prev = bitmap_rank(bmp, wpp, L, W, scan_sm);
    if (tid < 32) {  // rows descending: padded entries before each row's cells
      uint64_t carry = 0;
      for (int b = 0; b <= L; b += 32) {
        const int i = L - (b + lane);
        uint64_t v = 0;
        if (i >= j) {  // row i's cells: ranks [first(i), first(i - 1))
          const uint32_t c = (i > 0 ? wpj[(i - 1) * W] : n_cur) - wpj[i * W];
          v = (uint64_t)c * pad4(i - j + 1);
        }
        uint64_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
          const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (i >= 0) rowoff[i] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
  }
  __syncthreads();
  const ProgDev pd = p.progs[g];
  const uint32_t sbase = p.stage[pd.stage_base + j - 1];  // start of N_j within the program's cells
  uint32_t* cells = p.cells + pd.cell_base + sbase;
  uint32_t* cpo = p.cellpred + pd.cell_base + sbase;
  const uint64_t pstart = j >= 2 ? p.pred_start[(size_t)g * LP + j] : 0;
  // cells with rank in [x0, x1) (and their list offsets)
  for (int wi = tid; wi < nw; wi += nt) {
    uint32_t bits = bmj[wi];
    uint32_t pos = wpj[wi];
    if (!bits || pos >= x1 || pos + __popc(bits) <= x0) continue;
    const int row = wi / W, m0 = (wi % W) << 5;
    const uint32_t rfirst = wpj[row * W];  // rank of the row's first cell
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      if (pos >= x0 && pos < x1) {
        scell[pos - x0] = ((uint32_t)row << 16) | (uint32_t)(m0 + b);
        if (j >= 2) scpo[pos - x0] = (uint32_t)(pstart + rowoff[row] + (uint64_t)(pos - rfirst) * pad4(row - j + 1));
      }
      ++pos;
    }
  }
  __syncthreads();
  for (uint32_t x = x0 + tid; x < x1; x += nt) {
    cells[x] = scell[x - x0];
    if (j >= 2) cpo[x] = scpo[x - x0];
  }
  if (j < 2) return;
  // predecessor lists: 8 lanes per cell (4 cells per warp), each lane 4
  // cuts per pass (one 8-byte store)
  uint16_t* pbase = p.preds + pd.pred_base;
  const int sub = lane & 7;
  for (uint32_t x = x0 + (tid >> 3); x < x1; x += nt >> 3) {
    const uint32_t cell = scell[x - x0];
    const int i = cell >> 16, m = cell & 0xffff;
    const int n = i - j + 1, np = pad4(n);
    uint16_t* q = pbase + scpo[x - x0];
    for (int t0 = sub * 4; t0 < np; t0 += 32) {
      uint16_t v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int t = t0 + e;
        if (t < n) {
          const int c = j - 1 + t;
          const int s = seg[c * LP + i];
          const int mp = s > m ? s : m;
          const int wi = c * W + (mp >> 5);
          v[e] = (uint16_t)(wpp[wi] + __popc(bmp[wi] & ((1u << (mp & 31)) - 1u)));
        } else {
          v[e] = (uint16_t)n_prev;
        }
      }
      *reinterpret_cast<uint2*>(q + t0) =
          make_uint2((uint32_t)v[0] | ((uint32_t)v[1] << 16), (uint32_t)v[2] | ((uint32_t)v[3] << 16));
    }
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

// Gang version of sparse_solve: part g of G CTAs solves the cells
// [n g / G, n (g+1) / G) of every stage of one instance; the stage values
// V0 / V1 and the argmins bpS are the leader CTA's global scratch, shared by
// the gang (read through L2: other SMs write them), and *cnt counts the
// finished (part, stage) pairs: stage j starts once G (j - 1) are done
// (release add after the CTA barrier, acquire poll).  The leader (g = 0)
// backtracks after the last stage and returns the cost; the same cells,
// cuts and operations as sparse_solve, so the result is bit-identical.
__device__ __forceinline__ void gang_stage_done(uint32_t* cnt, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

template <class EdgeFn>
__device__ double sparse_solve_gang(const int L, const int k, const int gas,
                                    const double* __restrict__ Pf, const double* __restrict__ Dm,
                                    const ProgDev& pg, const uint32_t* __restrict__ cells,
                                    const uint32_t* __restrict__ cellpred,
                                    const uint16_t* __restrict__ preds,
                                    const uint32_t* __restrict__ stage, const EdgeFn& edge,
                                    double* V0, double* V1, double2* PE0, double2* PE1,
                                    uint8_t* bpS, int* cuts, int g, int G, uint32_t* cnt) {
  const double g1 = (double)(gas - 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  const uint32_t* cl = cells + pg.cell_base;
  const uint32_t* cpd = cellpred + pg.cell_base;
  const uint16_t* pd = preds + pg.pred_base;
  const uint32_t* ss = stage + pg.stage_base;
  {  // stage 1 (pipeline_dp.cpp:102-107), this part's cells of N_1
    const uint32_t n = ss[1] - ss[0], a = ss[0] + (uint32_t)((uint64_t)n * g / G),
                   b = ss[0] + (uint32_t)((uint64_t)n * (g + 1) / G);
    for (uint32_t x = a + tid; x < b; x += nt) {
      const uint32_t cell = cl[x];
      const int i = cell >> 16, m = cell & 0xffff;
      const double t1 = Pf[i] - Pf[0];
      V1[x - ss[0]] = g1 * max0(t1 - Dm[m]) + t1;
    }
  }
  if (k >= 2)
    for (int c = 1 + tid; c < L; c += nt) PE0[c] = make_double2(Pf[c], edge(c, 0));  // stage 2
  gang_stage_done(cnt, (uint32_t)G);
  for (int j = 2; j <= k; ++j) {
    const double* Vp = (j & 1) ? V0 : V1;
    double* Vc = (j & 1) ? V1 : V0;
    const double2* PE = (j & 1) ? PE1 : PE0;
    if (j < k) {
      double2* PN = (j & 1) ? PE0 : PE1;
      for (int c = j + tid; c < L; c += nt) PN[c] = make_double2(Pf[c], edge(c, j - 1));
    }
    const uint32_t s0 = ss[j - 1], n = ss[j] - s0;
    const uint32_t a = s0 + (uint32_t)((uint64_t)n * g / G), b = s0 + (uint32_t)((uint64_t)n * (g + 1) / G);
    const int c0 = j - 1, np = (int)(b - a);
    if (np * 2 > nt) {
      for (uint32_t x = a + tid; x < b; x += nt) {
        const uint32_t cell = cl[x];
        const int i = cell >> 16, m = cell & 0xffff;
        const double dm = Dm[m], Pi = Pf[i];
        const uint2* q = reinterpret_cast<const uint2*>(pd + cpd[x]);
        double best = CUDART_INF;
        int bc = -1;
        int c = c0;
        for (; c + 3 < i; c += 4, ++q) {
          const uint2 w = __ldg(q);
          cut_step(__ldcg(Vp + (w.x & 0xffff)), Pi, PE[c], dm, g1, c, best, bc);
          cut_step(__ldcg(Vp + (w.x >> 16)), Pi, PE[c + 1], dm, g1, c + 1, best, bc);
          cut_step(__ldcg(Vp + (w.y & 0xffff)), Pi, PE[c + 2], dm, g1, c + 2, best, bc);
          cut_step(__ldcg(Vp + (w.y >> 16)), Pi, PE[c + 3], dm, g1, c + 3, best, bc);
        }
        if (c < i) {
          const uint2 w = __ldg(q);
          cut_step(__ldcg(Vp + (w.x & 0xffff)), Pi, PE[c], dm, g1, c, best, bc);
          if (c + 1 < i) cut_step(__ldcg(Vp + (w.x >> 16)), Pi, PE[c + 1], dm, g1, c + 1, best, bc);
          if (c + 2 < i) cut_step(__ldcg(Vp + (w.y & 0xffff)), Pi, PE[c + 2], dm, g1, c + 2, best, bc);
        }
        Vc[x - s0] = best;
        bpS[x] = (uint8_t)bc;
      }
    } else {
      int GL = 2;  // lanes per cell (sparse_solve's few-cells branch)
      while (GL < 32 && np * GL * 2 <= nt) GL <<= 1;
      const int gl = tid & (GL - 1);
      const int per = nt / GL;
      for (int base = 0; base < np; base += per) {
        const int xi = base + tid / GL;
        double best = CUDART_INF;
        int bc = -1;
        if (xi < np) {
          const uint32_t x = a + xi;
          const uint32_t cell = cl[x];
          const int i = cell >> 16, m = cell & 0xffff;
          const double dm = Dm[m], Pi = Pf[i];
          const uint16_t* q = pd + cpd[x] + gl;
          for (int c = c0 + gl; c < i; c += GL, q += GL)
            cut_step(__ldcg(Vp + __ldg(q)), Pi, PE[c], dm, g1, c, best, bc);
        }
        for (int o = GL >> 1; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
          if (ov < best || (ov == best && oc < bc)) {
            best = ov;
            bc = oc;
          }
        }
        if (xi < np && gl == 0) {
          Vc[a + xi - s0] = best;
          bpS[a + xi] = (uint8_t)bc;
        }
      }
    }
    gang_stage_done(cnt, (uint32_t)G * (uint32_t)j);
  }
  double cost = 0.0;
  if (g == 0 && tid == 0) {
    cost = __ldcg(((k & 1) ? V1 : V0));
    cuts[k] = L;
    uint32_t x = ss[k - 1];
    for (int j = k; j >= 2; --j) {
      const int c = __ldcg(reinterpret_cast<const unsigned char*>(bpS) + x);
      cuts[j - 1] = c;
      x = ss[j - 2] + pd[cpd[x] + (c - (j - 1))];
    }
    cuts[0] = 0;
  }
  __syncthreads();
  return cost;
}

}  // namespace amp
