// amp_dp_multi.cuh — K_dp for B candidates of one class at a time.
//
// Every candidate of a class (pp, dp, tmp, mbs) runs the same pruned program
// (amp_dp_sparse.cuh): same cells, same predecessor lists, same prefix sums,
// tolerance domain and gas.  Only the stage-boundary bandwidths — hence the
// edge costs e(cut, q) — differ between placements.  So, for one (cell,
// cut) of the recurrence (pipeline_dp.cpp:114-131)
//
//     g = ((sub + (gas-1) * max(0, t2 - dom[m])) + t2) + edge(cut)
//
// the predecessor index, t2 = prefix[i] - prefix[cut] and the tolerance term
// (gas-1) * max(0, t2 - dom[m]) are the same for all B candidates; each
// candidate adds only its own sub (one gather), its own edge and the
// compare.  One thread owns one cell for all B candidates, so the shared
// part is issued once per B candidate-iterations:
//
//     shared  : pred index, LDS prefix[cut], DADD t2, DADD t2-dm, DSETP, DMUL
//     per cand: LDS sub, LDS edge, DADD, DADD, DADD, DSETP, argmin update
//
// Stage-1 values cost(i, 1, m) (pipeline_dp.cpp:102-107) depend on the
// class only, so they are computed once per class change and shared.
//
// Exactness: each candidate's values are produced by the same operations, in
// the same order, with the same operands as sparse_solve / the reference
// (strict '<' over ascending cuts; lexicographic (value, cut) combine in the
// split-cut path), so cuts and cost are bit-identical.
//
// Shared-memory layout (host mirror: multi_smem_bytes in amp_search.cu):
//   Vs[2][max_v][B]   f64  value arrays of stages j >= 2, interleaved by
//                          candidate (one 16-B load serves two candidates)
//   E[2][L][B]        f64  edge costs of the current / next stage
//   V1[max_n1]        f64  stage-1 values (class-shared)
//   Dm[max_M], Pf[L+1] f64
//   bp[2][max_rest][B] u8  argmin cut of every cell of stages j >= 2, per
//                          candidate (two buffers: the backtrack is deferred)
#pragma once

#include "amp_common.cuh"
#include "amp_dp_sparse.cuh"

namespace amp {

// One cut for B candidates.  STAGE2: the predecessor stage is stage 1,
// whose values are shared (V1, stride 1).
// Argmin update of one candidate: the scan's `if (g < best)` (strict '<':
// the lowest cut wins ties; NaN never wins).  (sm_100 has no FP64 min
// instruction — fmin compiles to DSETP + selects — so this form is cheapest.)
__device__ __forceinline__ void upd(double g, int c, double& best, int& bc) {
  if (g < best) {
    best = g;
    bc = c;
  }
}

template <int B, bool STAGE2>
__device__ __forceinline__ void multi_cut(const double* __restrict__ Vp,
                                          const double* __restrict__ Ec, int idx, double Pi,
                                          double pc, double dm, double g1, int c, double* best,
                                          int* bc) {
  const double t2 = Pi - pc;
  const double term = t2 > dm ? g1 * (t2 - dm) : 0.0;
  if (STAGE2) {
    const double st = Vp[idx] + term;
#pragma unroll
    for (int b = 0; b < B; b += 2) {
      const double2 e = *reinterpret_cast<const double2*>(Ec + b);
      upd((st + t2) + e.x, c, best[b], bc[b]);
      upd((st + t2) + e.y, c, best[b + 1], bc[b + 1]);
    }
  } else {
#pragma unroll
    for (int b = 0; b < B; b += 2) {
      const double2 s = *reinterpret_cast<const double2*>(Vp + (size_t)idx * B + b);
      const double2 e = *reinterpret_cast<const double2*>(Ec + b);
      upd(((s.x + term) + t2) + e.x, c, best[b], bc[b]);
      upd(((s.y + term) + t2) + e.y, c, best[b + 1], bc[b + 1]);
    }
  }
}

// Backpointers of one cell for the B candidates: bp[cell][b], one store.
template <int B>
__device__ __forceinline__ void store_bp(uint8_t* dst, const int* bc) {
  uint32_t w[(B + 3) / 4] = {};
#pragma unroll
  for (int b = 0; b < B; ++b) w[b / 4] |= (uint32_t)(bc[b] & 0xff) << (8 * (b % 4));
  if (B == 2) {
    *reinterpret_cast<uint16_t*>(dst) = (uint16_t)w[0];
  } else {
#pragma unroll
    for (int t = 0; t < (B + 3) / 4; ++t) reinterpret_cast<uint32_t*>(dst)[t] = w[t];
  }
}

// Stage j >= 2 of the group: cells [s0, s1) of the program.
template <int B, bool STAGE2>
__device__ __forceinline__ void multi_stage(const int j, const uint32_t s0, const uint32_t s1,
                                            const uint32_t rest0, const int max_rest,
                                            const uint2* __restrict__ cr,
                                            const uint16_t* __restrict__ pd, const double* Pf,
                                            const double* Dm, const double g1, const double* Vp,
                                            double* Vc, const double* E, uint8_t* bp,
                                            int* ctr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int c0 = j - 1;
  const int n = (int)(s1 - s0);
  if (n * 2 > nt) {
    // one thread per cell; warps take 32 consecutive cells at a time from a
    // shared counter (cells are ordered by row descending, i.e. by cut
    // count descending, so this is greedy longest-first scheduling and the
    // lanes of a chunk have similar cut counts); predecessor indices are
    // read 4 at a time
    const int lane = tid & 31;
    for (;;) {
      int base = 0;
      if (lane == 0) base = atomicAdd(ctr, 32);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= n) break;
      if (base + lane >= n) continue;
      const uint32_t x = s0 + base + lane;
      const uint2 rec = __ldg(cr + x);  // {cell, predecessor list offset}
      const int i = rec.x >> 16, m = rec.x & 0xffff;
      const double dm = Dm[m], Pi = Pf[i];
      const uint2* q = reinterpret_cast<const uint2*>(pd + rec.y);
      double best[B];
      int bc[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        best[b] = CUDART_INF;
        bc[b] = -1;
      }
      // 4 cuts per step, the next predecessor word loaded one step ahead
      uint2 w = __ldg(q);
      int c = c0;
      for (; c + 3 < i; c += 4) {
        const uint2 wn = __ldg(++q);
        multi_cut<B, STAGE2>(Vp, E + c * B, w.x & 0xffff, Pi, Pf[c], dm, g1, c, best, bc);
        multi_cut<B, STAGE2>(Vp, E + (c + 1) * B, w.x >> 16, Pi, Pf[c + 1], dm, g1, c + 1, best, bc);
        multi_cut<B, STAGE2>(Vp, E + (c + 2) * B, w.y & 0xffff, Pi, Pf[c + 2], dm, g1, c + 2, best, bc);
        multi_cut<B, STAGE2>(Vp, E + (c + 3) * B, w.y >> 16, Pi, Pf[c + 3], dm, g1, c + 3, best, bc);
        w = wn;
      }
      if (c < i) {
        multi_cut<B, STAGE2>(Vp, E + c * B, w.x & 0xffff, Pi, Pf[c], dm, g1, c, best, bc);
        if (c + 1 < i)
          multi_cut<B, STAGE2>(Vp, E + (c + 1) * B, w.x >> 16, Pi, Pf[c + 1], dm, g1, c + 1, best, bc);
        if (c + 2 < i)
          multi_cut<B, STAGE2>(Vp, E + (c + 2) * B, w.y & 0xffff, Pi, Pf[c + 2], dm, g1, c + 2, best, bc);
      }
      const uint32_t xl = x - s0;
#pragma unroll
      for (int b = 0; b < B; b += 2)
        *reinterpret_cast<double2*>(Vc + (size_t)xl * B + b) = make_double2(best[b], best[b + 1]);
      store_bp<B>(bp + (size_t)(x - rest0) * B, bc);
    }
  } else {
    // few cells (late stages): G lanes per cell split the cut loop by
    // residue, then a lexicographic (value, cut) butterfly per candidate —
    // equal to the sequential strict-'<' scan.
    int G = 2;
    while (G < 32 && n * G * 2 <= nt) G <<= 1;
    const int gl = tid & (G - 1);
    const int per = nt / G;
    for (int base = 0; base < n; base += per) {  // uniform trip count
      const int xi = base + tid / G;
      double best[B];
      int bc[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        best[b] = CUDART_INF;
        bc[b] = -1;
      }
      if (xi < n) {
        const uint2 rec = __ldg(cr + s0 + xi);
        const int i = rec.x >> 16, m = rec.x & 0xffff;
        const double dm = Dm[m], Pi = Pf[i];
        const uint16_t* q = pd + rec.y + gl;
        for (int c = c0 + gl; c < i; c += G, q += G)
          multi_cut<B, STAGE2>(Vp, E + c * B, __ldg(q), Pi, Pf[c], dm, g1, c, best, bc);
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        for (int o = G >> 1; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best[b], o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc[b], o);
          if (ov < best[b] || (ov == best[b] && oc < bc[b])) {
            best[b] = ov;
            bc[b] = oc;
          }
        }
      }
      if (xi < n && gl == 0) {
        const uint32_t x = s0 + xi;
#pragma unroll
        for (int b = 0; b < B; b += 2)
          *reinterpret_cast<double2*>(Vc + (size_t)xi * B + b) = make_double2(best[b], best[b + 1]);
        store_bp<B>(bp + (size_t)(x - rest0) * B, bc);
      }
    }
  }
}

// Persistent CTAs over batches of B chunk items: CTA c takes batches c,
// c + grid, ... (the dispatch order interleaves all classes heaviest first,
// so the static split is balanced) and prefetches the next batch's work
// records while it solves the current one.  A batch is split into
// same-class groups (one group in the steady state).  The backtrack of a
// group is deferred into stage 2 of the next group (double-buffered
// backpointers), where it overlaps with the other warps' cells.
template <int B>
__global__ void __launch_bounds__(B >= 8 ? 512 : 256, (B <= 2 ? 3 : (B >= 8 ? 1 : 2))) k_dp_multi(EvalParams p) {
  static_assert(B % 2 == 0 && B <= 16, "B must be even (16-byte value/edge loads)");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int WW = sizeof(CandWork) / 8;  // 8-byte words per work record
  __shared__ __align__(16) CandWork wq[2][B];
  __shared__ int ctr[2];
  __shared__ uint64_t gus[B];  // chunk positions of the current group's members
  const int L = p.L, LP = L + 1, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  const int maxpp = p.max_pp, max_v = p.max_v, max_rest = p.max_rest;
  const bool bt_warp = (tid >> 5) == (nt >> 5) - 1;  // runs deferred backtracks
  // dynamic smem carve-up (host mirror: multi_smem_bytes)
  // (value arrays carry a +inf sentinel slot; Pf / E are padded by 3 cuts
  // for the whole-4-cut steps)
  double* Vs0 = reinterpret_cast<double*>(smem_raw);
  double* Vs1 = Vs0 + (size_t)(max_v + 1) * B;
  double* E0 = Vs1 + (size_t)(max_v + 1) * B;
  double* E1 = E0 + (size_t)(L + 3) * B;
  double* V1 = E1 + (size_t)(L + 3) * B;
  double* Dm = V1 + (p.max_n1 + 1);
  double* Pf = Dm + p.max_M;
  uint8_t* const bpb = reinterpret_cast<uint8_t*>(Pf + LP + 3);  // [2][max_rest][B]

  // slots: chunk items that may need the DP (pp >= 3 first), or with
  // memoisation the distinct signatures (signature mode: class and boundary
  // codes come from the key, amp_trie.cuh K_sig_init; only when the trie is
  // off, or — sig_guard — when its device capacity was exceeded)
  if (p.sig_guard && *p.sig_guard == 0) return;
  const bool sigm = p.sig_keys != nullptr;
  const int sig_nq = maxpp - 1, sig_cb = p.sig_code_bits;
  const uint64_t n_items = (p.rep_list || sigm) ? *p.n_rep : p.n_dp;
  auto item_of = [&](uint64_t slot) -> uint64_t { return (p.rep_list && !sigm) ? p.rep_list[slot] : slot; };
  const uint64_t nbatch = (n_items + B - 1) / B;
  uint64_t bi = blockIdx.x;
  if (bi >= nbatch) return;
  auto word = [&](uint64_t batch, int w) -> uint64_t {
    const uint64_t slot = batch * B + w / WW;
    if (slot >= n_items) return 0;
    if (sigm)  // a CandWork of class key >> codes, fail_code 0 (word 2: cls | fail_code << 32)
      return (w % WW) == 2 ? (p.sig_keys[slot] >> (sig_nq * sig_cb)) : 0;
    return reinterpret_cast<const uint64_t*>(p.work + item_of(slot))[w % WW];
  };
  if (tid < B * WW) reinterpret_cast<uint64_t*>(wq[0])[tid] = word(bi, tid);
  if (tid < 3 * B) {  // edge padding (cuts L .. L+2), never rewritten
    E0[L * B + tid] = 0.0;
    E1[L * B + tid] = 0.0;
  }
  __syncthreads();

  int cur_cls = -1;  // class whose Pf / Dm / V1 are in smem
  // deferred backtrack (uniform except pend_u, the member of this lane)
  int pend_n = 0, pend_k = 0, pend_buf = 0;
  uint32_t pend_cell = 0, pend_stage = 0;
  uint64_t pend_pred = 0, pend_u = 0, pend_slot = 0;
  int bpsel = 0;
  auto backtrack = [&]() {  // pipeline_dp.cpp:134-148, lane r < pend_n
    const uint32_t* cpd = p.cellpred + pend_cell;
    const uint16_t* pd = p.preds + pend_pred;
    const uint32_t* ss = p.stage + pend_stage;
    const uint32_t rest0 = ss[1];
    // memoised runs write the signature's cuts at its run index (compact,
    // L2-resident for K_est); otherwise at the chunk item
    uint8_t* co = p.repcuts ? p.repcuts + pend_slot * (maxpp + 1) : p.cutsb + pend_u * (maxpp + 1);
    const uint8_t* bpr = bpb + (size_t)pend_buf * B * max_rest + lane;
    co[pend_k] = (uint8_t)L;
    uint32_t x = ss[pend_k - 1];  // N_k = {(L, 0)}
    for (int j = pend_k; j >= 2; --j) {
      const int c = bpr[(size_t)(x - rest0) * B];
      co[j - 1] = (uint8_t)c;
      x = ss[j - 2] + pd[cpd[x] + (c - (j - 1))];
    }
    co[0] = 0;
  };

  for (int it = 0;; ++it) {
    const int cur = it & 1;
    const uint64_t bnext = bi + gridDim.x;
    uint64_t pre = 0;  // next batch's records, stored after this batch
    if (tid < B * WW && bnext < nbatch) pre = word(bnext, tid);
    const uint64_t ubase = bi * B;
    const int bn = (int)(n_items - ubase < (uint64_t)B ? n_items - ubase : B);
    unsigned todo = 0;
    for (int b = 0; b < bn; ++b)
      if (wq[cur][b].fail_code == 0) todo |= 1u << b;  // failed before the DP
    while (todo) {
      // ---- next same-class group (every thread computes it) -------------
      const int gcls = wq[cur][__ffs(todo) - 1].cls;
      unsigned gm = 0;
      for (int b = 0; b < bn; ++b)
        if (((todo >> b) & 1u) && wq[cur][b].cls == gcls) gm |= 1u << b;
      todo &= ~gm;
      const int ng = __popc(gm);
      auto slot_of = [&](int r) -> uint64_t {  // r >= ng repeats member 0
        unsigned m = gm;
        for (int q = r < ng ? r : 0; q > 0; --q) m &= m - 1;
        return ubase + (uint64_t)(__ffs(m) - 1);
      };
      auto member = [&](int r) -> uint64_t {  // r >= ng repeats member 0
        unsigned m = gm;
        for (int q = r < ng ? r : 0; q > 0; --q) m &= m - 1;
        return item_of(ubase + (uint64_t)(__ffs(m) - 1));
      };
      const ClassDev cl = p.cls[gcls];
      const int k = cl.pp;
      if (k <= 2) continue;  // solved in K_est (light_cut2)
      const ProgDev pg = p.progs[p.class_prog[gcls]];
      if (p.exec_counters && tid == 0) {  // executed work (roofline accounting)
        atomicAdd(&p.exec_counters[0], (unsigned long long)ng);
        atomicAdd(&p.exec_counters[1],
                  (unsigned long long)(p.prog_inner[p.class_prog[gcls]] * ng));
      }
      const uint32_t* cl_ = p.cells + pg.cell_base;
      const uint2* cr = p.cellrec + pg.cell_base;
      const uint16_t* pd = p.preds + pg.pred_base;
      const uint32_t* ss = p.stage + pg.stage_base;
      const double g1 = (double)(cl.gas - 1);
      if (gcls != cur_cls) {
        // ---- class change: Pf, Dm, stage-1 values (pipeline_dp.cpp:102-107)
        // (the previous group's stages ended with a barrier)
        const double* gdom = p.domain + (size_t)cl.pair * p.nv_stride;
        const int M = p.pairs[cl.pair].M;
        for (int x = tid; x < M; x += nt) Dm[x] = gdom[x];
        for (int x = tid; x < LP + 3; x += nt) Pf[x] = p.prefix[(size_t)cl.pair * LP + (x < LP ? x : L)];
        __syncthreads();
        for (uint32_t x = ss[0] + tid; x < ss[1]; x += nt) {
          const uint32_t cell = cl_[x];
          const int i = cell >> 16, m = cell & 0xffff;
          const double t1 = Pf[i] - Pf[0];
          V1[x - ss[0]] = g1 * max0(t1 - Dm[m]) + t1;
        }
        if (tid == 0) V1[ss[1] - ss[0]] = CUDART_INF;  // sentinel slot
        cur_cls = gcls;
      }
      const uint32_t rest0 = ss[1];
      const double mbs = (double)cl.mbs;
      uint8_t* bp = bpb + (size_t)bpsel * B * max_rest;
      // edge cost e(cut, q) = act[cut-1]*mbs / bw[q] (placement_edge_cost,
      // optimizer.cpp:130-139): a lookup in the class's table of the same
      // quotients when the bandwidths are coded, else the division
      const double* qt = p.qtab ? p.qtab + (size_t)gcls * p.n_codes * L : nullptr;
      auto edge = [&](uint64_t uu, int c, int q) -> double {
        if (sigm)
          return qt[(size_t)((p.sig_keys[uu] >> ((sig_nq - 1 - q) * sig_cb)) & ((1ull << sig_cb) - 1)) * L + c];
        if (qt) return qt[(size_t)p.bwcb[uu * maxpp + q] * L + c];
        return p.act[c - 1] * mbs / p.bwqb[uu * maxpp + q];
      };
      // edges of stage 2 (boundary 0): E0[c][b], c in [1, L-1]
      for (int x = tid; x < (L - 1) * B; x += nt) {
        const int c = 1 + x / B, b = x % B;
        E0[c * B + b] = edge(member(b), c, 0);
      }
      if (tid < B) gus[tid] = member(tid);
      if (tid == 0) ctr[0] = ctr[1] = 0;
      __syncthreads();
      for (int j = 2; j <= k; ++j) {
        double* Vc = (j & 1) ? Vs1 : Vs0;
        const double* Vp = (j & 1) ? Vs0 : Vs1;
        const double* E = (j & 1) ? E1 : E0;
        if (j < k) {  // next stage's edges (boundary j-1), c in [j, L-1]
          double* EN = (j & 1) ? E0 : E1;
          for (int x = tid; x < (L - j) * B; x += nt) {
            const int c = j + x / B, b = x % B;
            EN[c * B + b] = edge(gus[b], c, j - 1);
          }
        }
        if (j > 2 && tid == 0) ctr[(j + 1) & 1] = 0;  // stage j-1's counter is free
        if (j == 2 && pend_n) {  // previous group's backtrack, overlapped
          if (bt_warp && lane < pend_n) backtrack();
          pend_n = 0;
        }
        const uint32_t s0 = ss[j - 1], s1 = ss[j];
        if (tid < B) Vc[(size_t)(s1 - s0) * B + tid] = CUDART_INF;  // sentinel slot
        if (j == 2)
          multi_stage<B, true>(j, s0, s1, rest0, max_rest, cr, pd, Pf, Dm, g1, V1, Vc, E, bp,
                               &ctr[0]);
        else
          multi_stage<B, false>(j, s0, s1, rest0, max_rest, cr, pd, Pf, Dm, g1, Vp, Vc, E,
                                bp, &ctr[j & 1]);
        __syncthreads();
      }
      pend_n = ng;
      pend_k = k;
      pend_buf = bpsel;
      pend_cell = pg.cell_base;
      pend_pred = pg.pred_base;
      pend_stage = pg.stage_base;
      pend_u = member(lane);
      pend_slot = slot_of(lane);
      bpsel ^= 1;
    }
    if (bnext >= nbatch) break;
    if (tid < B * WW) reinterpret_cast<uint64_t*>(wq[cur ^ 1])[tid] = pre;
    bi = bnext;
    __syncthreads();
  }
  if (pend_n && bt_warp && lane < pend_n) backtrack();
}

}  // namespace amp

namespace amp {

// {cell, cellpred} records for K_dp multi (one 8-byte load per cell).
__global__ void k_pack_cells(const uint32_t* cells, const uint32_t* cellpred, uint2* rec,
                             uint64_t n) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x)
    rec[x] = make_uint2(cells[x], cellpred[x]);
}

}  // namespace amp
