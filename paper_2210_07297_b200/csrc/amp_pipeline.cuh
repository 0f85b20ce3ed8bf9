// amp_pipeline.cuh — candidate evaluation as three batched kernels per chunk
// of work items (replaces the one-CTA-per-candidate monolith):
//
//   K_place  warp per candidate: decode (segment -> class, placement index),
//            early failures (pp > L, profile miss), placement (heuristic
//            order, splitmix64 Fisher-Yates; lane = rank for |D| <= 32),
//            min_edge_bandwidth per stage boundary (cost_model.cpp:164-174)
//            and the DP edge function's p2p_time check.
//   K_dp     persistent CTAs, one candidate at a time: only the layer-partition
//            DP (pruned or dense) -> cuts.  No serial phases between stages.
//   K_est    warp per candidate: stage sums and params_in_range, parameter
//            ceiling (optimizer.cpp:159-169), estimate (cost_model.cpp:176-212),
//            record, CTA top-k (rank_records key).
//
// Latency-bound scalar work (splitmix chain, divisions, shuffles) now
// overlaps across dozens of independent warps per SM instead of stalling the
// three idle warps of a DP CTA.
#pragma once

#include "amp_common.cuh"
#include "amp_dp_sparse.cuh"

namespace amp {

struct CandWork {
  uint64_t index;     // candidate index
  uint64_t out;       // position in the caller's output order
  int32_t cls;
  int32_t fail_code;  // 0 ok, AMP_FAIL_*
  int32_t fail_layer;
  int32_t pad;
  double fail_value;
};

// ---------------------------------------------------------------------------
// work decode: item t of the run -> candidate
// ---------------------------------------------------------------------------
// hint (optional): the segment of this thread's previous item.  Grid-stride
// loops visit increasing t, and a stride is shorter than a class segment, so
// the segment is found by stepping forward from the hint (usually zero or
// one step) instead of a dependent-load binary search per item.
__device__ __forceinline__ void decode_item(const EvalParams& p, uint64_t t, uint64_t& index,
                                            uint64_t& out, int& cls, uint64_t& pl,
                                            int* hint = nullptr) {
  if (p.index_list) {
    index = p.index_list[t];
    out = t;
    cls = (int)(index / p.P);
    pl = index % p.P;
    return;
  }
  int lo;
  if (hint && *hint >= 0 && __ldg(&p.segs[*hint].offset) <= t) {
    lo = *hint;
    while (lo + 1 < p.n_segs && __ldg(&p.segs[lo + 1].offset) <= t) ++lo;
  } else {
    lo = 0;
    int hi = p.n_segs - 1;  // last segment with offset <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&p.segs[mid].offset) <= t) lo = mid;
      else hi = mid - 1;
    }
  }
  if (hint) *hint = lo;
  const Segment& sg = p.segs[lo];
  const uint64_t d = t - sg.offset;
  index = sg.first + d;
  out = sg.out + d;
  pl = sg.p0 + d;
  cls = (int)sg.cls;
}

// ---------------------------------------------------------------------------
// K_place
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_place(EvalParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int D = p.D, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // |D| <= 32: bandwidth matrix (or its code matrix) and one rank->device
  // row per warp in smem
  double* bwS = reinterpret_cast<double*>(smem_raw);
  int* placeS = reinterpret_cast<int*>(bwS + (D <= 32 ? D * D : 0)) + wib * 32;
  uint8_t* codeS = reinterpret_cast<uint8_t*>(placeS - wib * 32 + 32 * (blockDim.x >> 5));
  const double* BW = p.bw;
  const uint8_t* CODE = p.bwcode;
  if (D <= 32) {
    for (int x = threadIdx.x; x < D * D; x += blockDim.x) {
      bwS[x] = p.bw[x];
      if (p.bwcode) codeS[x] = p.bwcode[x];
    }
    BW = bwS;
    if (p.bwcode) CODE = codeS;
    __syncthreads();
  }
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t u = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; u < p.n_chunk; u += nw) {
    uint64_t index, out, pl;
    int c;
    decode_item(p, p.t0 + u, index, out, c, pl);
    const ClassDev cl = p.cls[c];
    const PairDev pr = p.pairs[cl.pair];
    const int pp = cl.pp, dp = cl.dp, tmp = cl.tmp;
    int fc = 0, flayer = -1;
    double fval = 0.0;
    if (pp > p.L) {  // optimizer.cpp:149-152
      fc = AMP_FAIL_PP_GT_L;
    } else if (pr.fail_code) {  // segment_times: first failing layer
      fc = pr.fail_code;
      flayer = pr.fail_layer;
      fval = pr.fail_value;
    }
    int32_t* prow = p.placeb + u * D;
    if (fc == 0) {
      // ---- placement: heuristic order (placement.cpp:37-49); p >= 1:
      //      Fisher-Yates driven by splitmix64(seed ^ p) ------------------
      if (p.given_place) {  // caller placement (anneal proposals, evaluate_placed)
        const int32_t* g = p.given_place + (p.t0 + u) * D;
        for (int x = lane; x < D; x += 32) prow[x] = g[x];
        if (D <= 32) placeS[lane] = lane < D ? g[lane] : -1;
        __syncwarp();
      } else if (D <= 32) {
        int v = lane < D ? p.base_order[lane] : -1;
        if (pl != 0) {
          // lane kk keeps the draw of step kk, then reduces it once:
          // r mod d == ((hi mod d) * (2^32 mod d) + (lo mod d)) mod d
          uint64_t r = splitmix64(p.seed ^ pl), mine = 0;
          for (int kk = D - 1; kk >= 1; --kk) {
            mine = lane == kk ? r : mine;
            r = splitmix64(r);
          }
          const uint32_t d = (uint32_t)lane + 1u;
          const uint32_t hi = (uint32_t)(mine >> 32) % d, lo = (uint32_t)mine % d;
          const uint32_t t32 = (uint32_t)((1ull << 32) % d);
          const int jk = (int)((hi * t32 + lo) % d);
          for (int kk = D - 1; kk >= 1; --kk) {
            const int jj = __shfl_sync(0xffffffffu, jk, kk);
            const int src = lane == kk ? jj : (lane == jj ? kk : lane);
            v = __shfl_sync(0xffffffffu, v, src);
          }
        }
        placeS[lane] = v;
        if (lane < D) prow[lane] = v;
        __syncwarp();
      } else {
        for (int x = lane; x < D; x += 32) prow[x] = p.base_order[x];
        __syncwarp();
        if (pl != 0 && lane == 0) {
          uint64_t r = splitmix64(p.seed ^ pl);
          for (int kk = D - 1; kk >= 1; --kk) {
            const int jj = (int)(r % (uint64_t)(kk + 1));
            const int t = prow[kk];
            prow[kk] = prow[jj];
            prow[jj] = t;
            r = splitmix64(r);
          }
        }
        __syncwarp();
      }
      const int* PL = D <= 32 ? placeS : prow;
      // ---- stage-boundary bandwidths (min over all replicas and shards) --
      int first_bad = 0x7fffffff;
      double bad_val = 0.0;
      for (int q0 = 0; q0 < pp - 1; q0 += 32) {
        const int q = q0 + lane;
        double b = CUDART_INF;
        if (q < pp - 1) {
          if (CODE) {
            // codes rank the distinct bandwidths, so the minimum code is the
            // code of the minimum bandwidth (no NaN: checked at create)
            int cm = 255;
            for (int r = 0; r < dp; ++r)
              for (int s = 0; s < tmp; ++s) {
                const int cc = CODE[(size_t)PL[(q * dp + r) * tmp + s] * D +
                                    PL[((q + 1) * dp + r) * tmp + s]];
                cm = cc < cm ? cc : cm;
              }
            b = p.bwval[cm];
            p.bwcb[u * p.max_pp + q] = (uint8_t)cm;
          } else {
            for (int r = 0; r < dp; ++r)
              for (int s = 0; s < tmp; ++s)
                b = std_min(b, BW[(size_t)PL[(q * dp + r) * tmp + s] * D +
                                  PL[((q + 1) * dp + r) * tmp + s]]);
          }
          p.bwqb[u * p.max_pp + q] = b;
        }
        // p2p_time throws on the first invalid boundary inside the DP's
        // edge function (cost_model.cpp:54-59)
        const unsigned bad = __ballot_sync(0xffffffffu, q < pp - 1 && !(b > 0));
        if (bad && first_bad == 0x7fffffff) {
          const int l0 = __ffs(bad) - 1;
          first_bad = q0 + l0;
          bad_val = __shfl_sync(0xffffffffu, b, l0);
        }
      }
      if (first_bad != 0x7fffffff) {
        fc = AMP_FAIL_P2P_BANDWIDTH;
        fval = bad_val;
      }
    }
    if (lane == 0) {
      CandWork w;
      w.index = index;
      w.out = out;
      w.cls = c;
      w.fail_code = fc;
      w.fail_layer = flayer;
      w.pad = 0;
      w.fail_value = fval;
      p.work[u] = w;
    }
  }
}

// ---------------------------------------------------------------------------
// K_dp
// ---------------------------------------------------------------------------
enum : int { kDenseSS = 0, kDenseSG = 1, kDenseGS = 2, kDenseGG = 3, kSparseS = 4, kSparseG = 5 };

#ifndef AMP_DP_BATCH
#define AMP_DP_BATCH 4
#endif
constexpr int kDpBatch = AMP_DP_BATCH;

struct DpShared {
  uint64_t u;
  int done, ok;
  int cls, pair;
  ClassDev cl;
  PairDev pr;
  uint32_t leader, pad;
};

// The gang list of a K_dp launch: every item whose program has >= gang_min
// inner iterations, with G = clamp(inner / gang_unit, 2, gang_max) parts;
// units (gang, part) numbered gang-major (one CTA).
__global__ void __launch_bounds__(1024) k_gang_plan(EvalParams p) {
  __shared__ uint32_t s_c[32], s_g[32], s_nb, s_nu;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  const uint64_t n_items = (p.sig_guard && *p.sig_guard == 0) ? 0 : (p.rep_list ? *p.n_rep : p.n_dp);
  if (tid == 0) s_nb = s_nu = 0;
  __syncthreads();
  for (uint64_t base = 0; base < n_items; base += blockDim.x) {
    const uint64_t slot = base + tid;
    uint32_t G = 0;
    if (slot < n_items) {
      const uint64_t u = p.rep_list ? p.rep_list[slot] : slot;
      const CandWork& wk = p.work[u];
      if (wk.fail_code == 0) {
        const double inner = p.prog_inner[p.class_prog[wk.cls]];
        if (inner >= p.gang_min)
          G = (uint32_t)min(p.gang_max, max(2, (int)(inner / p.gang_unit)));
      }
    }
    // block exclusive scans of (G > 0) and G
    uint32_t c = G ? 1u : 0u, gi = G;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, c, o), z = __shfl_up_sync(0xffffffffu, gi, o);
      if (lane >= o) {
        c += y;
        gi += z;
      }
    }
    if (lane == 31) {
      s_c[w] = c;
      s_g[w] = gi;
    }
    __syncthreads();
    uint32_t pc = 0, pgi = 0, tc = 0, tg = 0;
    for (int x = 0; x < nw; ++x) {
      if (x < w) {
        pc += s_c[x];
        pgi += s_g[x];
      }
      tc += s_c[x];
      tg += s_g[x];
    }
    if (G) {
      const uint32_t b = s_nb + pc + c - 1;
      p.gang_slot[b] = (uint32_t)slot;
      p.gang_off[b] = s_nu + pgi + gi - G;
      p.gang_sync[2 * b] = ~0u;
      p.gang_sync[2 * b + 1] = 0;
    }
    __syncthreads();
    if (tid == 0) {
      s_nb += tc;
      s_nu += tg;
    }
    __syncthreads();
  }
  if (tid == 0) {
    p.gang_off[s_nb] = s_nu;
    p.gang_hdr[0] = s_nb;
    p.gang_hdr[1] = s_nu;
    p.gang_hdr[2] = 0;
  }
}



// MODE selects the DP implementation and where its working set lives
// (compile-time so the compiler emits LDS/STS instead of generic loads):
//   kDenseSS/SG/GS/GG  full tolerance-indexed table; stage slice / cut table
//                      in (S)hared or (G)lobal memory
//   kSparseS/G         pruned program (amp_dp_sparse.cuh); value arrays and
//                      backpointers in shared / global memory
// kSparseG (large L, e.g. 96 layers x 1024 GPUs): few, very uneven DP
// instances, so each candidate gets a full 1024-thread CTA.
template <int MODE>
__global__ void __launch_bounds__(MODE == kSparseG ? 1024 : (MODE == kSparseS ? 256 : kEvalThreads),
                                  MODE == kSparseG ? 1 : (MODE == kSparseS ? 4 : 2))
    k_dp(EvalParams p) {
  constexpr bool SPARSE = MODE >= kSparseS;
  constexpr bool SLICE_SMEM = MODE == kDenseSS || MODE == kDenseSG;
  constexpr bool W_SMEM = MODE == kDenseSS || MODE == kDenseGS;
  constexpr bool V_SMEM = MODE == kSparseS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ DpShared sh;
  const int L = p.L, LP = L + 1, tid = threadIdx.x, nt = blockDim.x;
  const int maxM = p.max_M, maxpp = p.max_pp;
  // dynamic smem carve-up (host mirror: dp_smem_bytes in amp_search.cu)
  unsigned char* sp = smem_raw;
  double* C = nullptr;
  WEnt* W = nullptr;
  double *V0 = nullptr, *V1 = nullptr;
  uint8_t* bp = p.bp + (size_t)blockIdx.x * p.bp_stride;
  if (SPARSE) {
    if (V_SMEM) {
      V0 = reinterpret_cast<double*>(sp);
      sp += sizeof(double) * 2 * (size_t)p.max_cells;
      bp = reinterpret_cast<uint8_t*>(sp);
      sp += (p.max_prog_cells + 15) & ~15;
    } else {
      V0 = p.vbuf + (size_t)blockIdx.x * 2 * p.max_cells;
    }
    V1 = V0 + p.max_cells;
  } else {
    if (SLICE_SMEM) {
      C = reinterpret_cast<double*>(sp);
      sp += sizeof(double) * (size_t)LP * maxM;
    } else {
      C = p.slice + (size_t)blockIdx.x * p.slice_stride;
    }
    if (W_SMEM) {
      W = reinterpret_cast<WEnt*>(sp);
      sp += sizeof(WEnt) * (size_t)LP * L;
    } else {
      W = p.wtab + (size_t)blockIdx.x * LP * L;
    }
  }
  double* Dm = reinterpret_cast<double*>(sp);
  sp += sizeof(double) * maxM;
  double* Pf = reinterpret_cast<double*>(sp);
  sp += sizeof(double) * LP;
  sp = smem_raw + ((sp - smem_raw + 15) & ~15);
  double* E = reinterpret_cast<double*>(sp);  // dense: E[L]; sparse: 2 x double2[L]
  sp += sizeof(double) * 4 * L;
  CandWork* wq = reinterpret_cast<CandWork*>(sp);  // [kDpBatch]
  sp += sizeof(CandWork) * kDpBatch;
  int* cuts = reinterpret_cast<int*>(sp);
  sp += sizeof(int) * (maxpp + 2);
  // (integer offset from smem_raw keeps the shared address space visible)
  uint16_t* seg = reinterpret_cast<uint16_t*>(smem_raw + ((sp - smem_raw + 15) & ~15));

  // memoised runs (p.rep_list): slot s solves signature s through its
  // representative item rep_list[s] and writes its cuts at repcuts[s]; a
  // guarded launch (sig_guard) runs only while *sig_guard != 0
  if (p.sig_guard && *p.sig_guard == 0) return;
  const uint64_t n_items = p.rep_list ? *p.n_rep : p.n_dp;
  if (tid == 0) {
    sh.cls = -1;
    sh.pair = -1;
  }
  // ---- gangs first (k_gang_plan): units (gang, part) in gang-major order
  //      from their own counter; the first part of a gang publishes its CTA,
  //      whose scratch holds the gang's stage values and argmins.  Every
  //      CTA a part waits on holds a unit of the same gang, and only the
  //      last gang being dealt can lack parts, so the gangs cannot deadlock.
  if constexpr (MODE == kSparseG) {
    if (p.gang_hdr) {
      const uint32_t NB = p.gang_hdr[0], NU = p.gang_hdr[1];
      for (;;) {
        if (tid == 0) sh.u = atomicAdd(&p.gang_hdr[2], 1u);
        __syncthreads();
        const uint32_t un = (uint32_t)sh.u;
        if (un >= NU) break;
        int lo = 0, hi = (int)NB - 1;  // the last gang whose first unit is <= un
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (p.gang_off[mid] <= un) lo = mid;
          else hi = mid - 1;
        }
        const int g = (int)(un - p.gang_off[lo]), G = (int)(p.gang_off[lo + 1] - p.gang_off[lo]);
        const uint64_t slot = p.gang_slot[lo];
        const uint64_t u = p.rep_list ? p.rep_list[slot] : slot;
        const CandWork w = p.work[u];
        uint32_t* gs = p.gang_sync + 2 * (size_t)lo;
        if (tid == 0) {
          uint32_t ld = blockIdx.x;
          if (g == 0) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gs), "r"(ld) : "memory");
          } else {
            for (;;) {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(ld) : "l"(gs) : "memory");
              if (ld != ~0u) break;
              __nanosleep(64);
            }
          }
          sh.leader = ld;
        }
        if (w.cls != sh.cls) {
          __syncthreads();
          if (tid == 0) {
            sh.cls = w.cls;
            sh.cl = p.cls[w.cls];
            sh.pr = p.pairs[sh.cl.pair];
          }
        }
        __syncthreads();
        const ClassDev cl = sh.cl;
        const int pp = cl.pp;
        if (sh.pair != cl.pair) {
          const double* gdom = p.domain + (size_t)cl.pair * p.nv_stride;
          for (int x = tid; x < sh.pr.M; x += nt) Dm[x] = gdom[x];
          for (int x = tid; x < LP; x += nt) Pf[x] = p.prefix[(size_t)cl.pair * LP + x];
          __syncthreads();
          if (tid == 0) sh.pair = cl.pair;
        }
        const uint32_t ldr = sh.leader;
        double* GV0 = p.vbuf + (size_t)ldr * 2 * p.max_cells;
        uint8_t* gbp = p.bp + (size_t)ldr * p.bp_stride;
        EdgeFromBandwidth ef{p.act, p.bwqb + u * maxpp, cl.mbs};
        const ProgDev pg = p.progs[p.class_prog[w.cls]];
        sparse_solve_gang(L, pp, cl.gas, Pf, Dm, pg, p.cells, p.cellpred, p.preds, p.stage, ef, GV0,
                          GV0 + p.max_cells, reinterpret_cast<double2*>(E), reinterpret_cast<double2*>(E) + L,
                          gbp, cuts, g, G, gs + 1);
        if (g == 0) {
          uint8_t* co = p.repcuts ? p.repcuts + slot * (maxpp + 1) : p.cutsb + u * (maxpp + 1);
          for (int q = tid; q <= pp; q += nt) co[q] = (uint8_t)cuts[q];
          if (p.exec_counters && tid == 0) {
            atomicAdd(&p.exec_counters[0], 1ull);
            atomicAdd(&p.exec_counters[1], (unsigned long long)p.prog_inner[p.class_prog[w.cls]]);
          }
        }
        __syncthreads();
      }
    }
  }
  // work is taken kDpBatch items at a time: one atomic and one coalesced
  // load of the work records and bandwidth rows per batch
  int bi = 0, bn = 0;
  uint64_t bbase = 0;
  for (;;) {
    if (bi >= bn) {
      if (tid == 0) {
        const unsigned long long u0 = atomicAdd(p.counter, (unsigned long long)kDpBatch);
        sh.u = u0;
        sh.done = u0 >= n_items;  // items [n_dp, n_chunk) are pp <= 2 (K_est)
      }
      __syncthreads();
      if (sh.done) break;
      bbase = sh.u;
      bn = n_items - bbase < (uint64_t)kDpBatch ? (int)(n_items - bbase) : kDpBatch;
      bi = 0;
      constexpr int WW = (int)(sizeof(CandWork) / 8);
      uint64_t* dst = reinterpret_cast<uint64_t*>(wq);
      for (int x = tid; x < bn * WW; x += nt) {
        const uint64_t it = p.rep_list ? p.rep_list[bbase + x / WW] : bbase + x / WW;
        dst[x] = reinterpret_cast<const uint64_t*>(p.work + it)[x % WW];
      }
      __syncthreads();
    }
    const int my = bi++;
    const CandWork& w = wq[my];
    if (w.fail_code != 0) continue;  // failed before the DP (uniform)
    if (MODE == kSparseG && p.gang_hdr && p.prog_inner[p.class_prog[w.cls]] >= p.gang_min)
      continue;  // solved by its gang (above)
    const uint64_t slot = bbase + my;
    const uint64_t u = p.rep_list ? p.rep_list[slot] : slot;
    if (p.exec_counters && tid == 0) {  // executed work (roofline accounting)
      atomicAdd(&p.exec_counters[0], 1ull);
      atomicAdd(&p.exec_counters[1], (unsigned long long)p.prog_inner[p.class_prog[w.cls]]);
    }
    if (w.cls != sh.cls) {  // uniform: everybody reads the same smem
      __syncthreads();
      if (tid == 0) {
        sh.cls = w.cls;
        sh.cl = p.cls[w.cls];
        sh.pr = p.pairs[sh.cl.pair];
      }
      __syncthreads();
    }
    const ClassDev cl = sh.cl;
    const PairDev pr = sh.pr;
    const int pp = cl.pp, M = pr.M;
    const double* bwq = p.bwqb + u * maxpp;  // read by the edge function (L1)
    if (sh.pair != cl.pair) {  // Dm/Pf (and the dense seg table) persist in smem
      const double* gdom = p.domain + (size_t)cl.pair * p.nv_stride;
      for (int x = tid; x < M; x += nt) Dm[x] = gdom[x];
      for (int x = tid; x < LP; x += nt) Pf[x] = p.prefix[(size_t)cl.pair * LP + x];
      if (!SPARSE) {
        const uint16_t* gseg = p.seg + (size_t)cl.pair * LP * LP;
        for (int x = tid; x < LP * LP; x += nt) seg[x] = gseg[x];
      }
      __syncthreads();
      if (tid == 0) sh.pair = cl.pair;
    }
    EdgeFromBandwidth ef{p.act, bwq, cl.mbs};
    if (SPARSE) {
      const ProgDev pg = p.progs[p.class_prog[sh.cls]];
      sparse_solve(L, pp, cl.gas, Pf, Dm, pg, p.cells, p.cellpred, p.preds, p.stage, ef, V0, V1,
                   reinterpret_cast<double2*>(E), reinterpret_cast<double2*>(E) + L, bp, cuts);
    } else {
      dp_solve(L, pp, cl.gas, M, Pf, Dm, seg, ef, C, W, E, pr.monotone != 0, bp, cuts);
    }
    uint8_t* co = p.repcuts ? p.repcuts + slot * (maxpp + 1) : p.cutsb + u * (maxpp + 1);
    for (int q = tid; q <= pp; q += nt) co[q] = (uint8_t)cuts[q];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K_est
// ---------------------------------------------------------------------------
constexpr int kEstWarps = 8;

// simulate() (reference simulator.cpp:140-198) for one candidate, by its
// warp.  run_replica's event loop (75-136) keeps every stage in micro-batch
// order and every link FIFO, so its event times obey
//     C[j][u]  = max(C[j][u-1], TE[j-1][u]) + t_j      (compute end)
//     TE[j][u] = max(TE[j][u-1], C[j][u]) + e_j(r)     (transfer end)
// with C[j][-1] = TE[j][-1] = 0 and TE[-1][u] = 0: the start of an event is
// the time of the later of its two triggers, and each end time is one DADD
// of that start, exactly as the event loop pushes `now + duration`.
// finish = C[pp-1][gas-1]; makespan = max over replicas (std::max order);
// iteration time = makespan + dpsync.  pp <= 32: lane j owns stage j and the
// warp sweeps the (stage, micro-batch) wavefront (TE passed by shfl_up);
// pp > 32: lane 0 sweeps stage by stage over a per-warp array of the
// incoming ready times.
__device__ double sim_iteration(const EvalParams& p, const ClassDev& cl, const int* PL,
                                const int* cutsW, const double* stW, double dpsync, int lane,
                                double* scratch) {
  const int pp = cl.pp, dp = cl.dp, tmp = cl.tmp, gas = cl.gas, D = p.D;
  auto edge = [&](int q, int r) {  // replica_edge_times (cost_model.cpp:145-162)
    const double volume = p.act[cutsW[q + 1] - 1] * cl.mbs;
    double b = CUDART_INF;
    for (int s = 0; s < tmp; ++s)
      b = std_min(b, p.bw[(size_t)PL[(q * dp + r) * tmp + s] * D + PL[((q + 1) * dp + r) * tmp + s]]);
    return volume / b;
  };
  double makespan = 0.0;
  for (int r = 0; r < dp; ++r) {
    double fin = 0.0;
    if (pp <= 32) {
      const int j = lane;
      const double t = j < pp ? stW[j] : 0.0;
      const double e = j < pp - 1 ? edge(j, r) : 0.0;
      double C = 0.0, TE = 0.0;
      for (int step = 0; step < gas + pp - 1; ++step) {
        const double Rin = __shfl_up_sync(0xffffffffu, TE, 1);  // TE[j-1][step-j]
        const int u = step - j;
        if (j < pp && u >= 0 && u < gas) {
          const double R = j == 0 ? 0.0 : Rin;
          C = (C < R ? R : C) + t;
          if (j < pp - 1) TE = (TE < C ? C : TE) + e;
        }
      }
      fin = __shfl_sync(0xffffffffu, C, pp - 1);
    } else {
      if (lane == 0) {
        for (int u = 0; u < gas; ++u) scratch[u] = 0.0;
        double C = 0.0;
        for (int j = 0; j < pp; ++j) {
          const double t = stW[j];
          const double e = j < pp - 1 ? edge(j, r) : 0.0;
          double TE = 0.0;
          C = 0.0;
          for (int u = 0; u < gas; ++u) {
            const double R = scratch[u];
            C = (C < R ? R : C) + t;
            if (j < pp - 1) {
              TE = (TE < C ? C : TE) + e;
              scratch[u] = TE;
            }
          }
        }
        fin = C;
      }
      fin = __shfl_sync(0xffffffffu, fin, 0);
    }
    makespan = makespan < fin ? fin : makespan;  // std::max(makespan, run_replica(...))
  }
  return makespan + dpsync;
}

// The layer-partition DP for k = 2 stages (pipeline_dp.cpp:70-149): stage 2
// has the single cell (L, 0); its cut c reads stage-1 cell
// (c, max(seg(c, L), 0)) = (c, seg(c, L)).  Lane-strided cuts, each lane
// keeps its first strict minimum, then a lexicographic (value, cut)
// butterfly — the sequential strict-'<' scan.  Same operations and operand
// order as sparse_solve / the reference.
__device__ int light_cut2(const EvalParams& p, const ClassDev& cl, int cls, uint64_t u, int lane) {
  const int L = p.L, LP = L + 1;
  const double* Pf = p.prefix + (size_t)cl.pair * LP;
  const double* Dm = p.domain + (size_t)cl.pair * p.nv_stride;
  const uint16_t* sg = p.seg + (size_t)cl.pair * LP * LP;
  const double g1 = (double)(cl.gas - 1);
  const double bq = p.bwqb[u * p.max_pp];
  // edge costs: the class's table of the same quotients when coded
  const double* qt = p.qtab ? p.qtab + ((size_t)cls * p.n_codes + p.bwcb[u * p.max_pp]) * L
                            : nullptr;
  const double dm0 = Dm[0], PL = Pf[L], P0 = Pf[0];
  double best = CUDART_INF;
  int bc = -1;
  for (int c = 1 + lane; c < L; c += 32) {
    const double t1 = Pf[c] - P0;
    const double sub = g1 * max0(t1 - Dm[sg[c * LP + L]]) + t1;  // cost(c, 1, seg(c, L))
    const double t2 = PL - Pf[c];
    const double term = t2 > dm0 ? g1 * (t2 - dm0) : 0.0;
    const double e = qt ? qt[c] : p.act[c - 1] * cl.mbs / bq;  // placement_edge_cost
    const double g = ((sub + term) + t2) + e;
    if (g < best) {
      best = g;
      bc = c;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
    if (ov < best || (ov == best && oc < bc)) {
      best = ov;
      bc = oc;
    }
  }
  return bc;
}

// Per-warp smem scratch of K_est.
struct EstWarp {
  double ebuf[32];
  int place[32];
};

__global__ void __launch_bounds__(kEstWarps * 32, 2) k_est(EvalParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int lock;
  __shared__ int n_top;
  // the k-th entry only improves, so these may be read without the lock
  // as a conservative reject filter
  __shared__ double kth_total;
  __shared__ int kth_failed;
  __shared__ unsigned long long kth_index;  // (failed k-th: failed items order by index)
  const int D = p.D, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, maxpp = p.max_pp;
  // smem: [bw matrix if |D| <= 32] [st, spar per warp: 2 * maxpp] [cuts per warp]
  //       [EstWarp per warp] [CTA top-k, k <= 32]
  unsigned char* sp = smem_raw;
  double* bwS = reinterpret_cast<double*>(sp);
  if (D <= 32) sp += sizeof(double) * D * D;
  double* stW = reinterpret_cast<double*>(sp) + wib * 2 * maxpp;
  double* sparW = stW + maxpp;
  sp += sizeof(double) * 2 * maxpp * kEstWarps;
  int* cutsW = reinterpret_cast<int*>(sp) + wib * (maxpp + 2);
  sp += sizeof(int) * (maxpp + 2) * kEstWarps;
  // node bitmaps of the node-pair all-reduce minimum: present, >= 2 devices
  unsigned* nodeP = reinterpret_cast<unsigned*>(sp) + wib * 2 * p.node_words;
  unsigned* nodeM = nodeP + p.node_words;
  if (p.nodebw) sp += sizeof(unsigned) * 2 * p.node_words * kEstWarps;
  sp = smem_raw + ((sp - smem_raw + 15) & ~15);
  EstWarp* ew = reinterpret_cast<EstWarp*>(sp) + wib;
  sp += sizeof(EstWarp) * kEstWarps;
  amp_record* topS = reinterpret_cast<amp_record*>(sp);
  amp_record* const gtop = p.cta_topk + (size_t)blockIdx.x * p.k;
  amp_record* mytop = p.k <= 32 ? topS : gtop;
  const double* BW = p.bw;
  if (D <= 32) {
    for (int x = threadIdx.x; x < D * D; x += blockDim.x) bwS[x] = p.bw[x];
    BW = bwS;
  }
  if (threadIdx.x == 0) {
    lock = 0;
    n_top = 0;
    kth_total = CUDART_INF;
    kth_failed = 2;
    kth_index = ~0ull;
    if (!p.first_chunk) {  // CTA lists persist across chunks
      for (int x = 0; x < p.k; ++x) {
        if (gtop[x].fail_code < 0) break;
        if (mytop != gtop) mytop[x] = gtop[x];
        ++n_top;
      }
      if (p.k > 0 && n_top == p.k) {
        kth_failed = mytop[p.k - 1].fail_code != 0;
        kth_total = mytop[p.k - 1].total;
        kth_index = mytop[p.k - 1].index;
      }
    }
  }
  __syncthreads();
  const uint64_t nw = (uint64_t)gridDim.x * kEstWarps;
  for (uint64_t u = (uint64_t)blockIdx.x * kEstWarps + wib; u < p.n_chunk; u += nw) {
    const CandWork w = p.work[u];
    const ClassDev cl = p.cls[w.cls];
    const int pp = cl.pp, dp = cl.dp, tmp = cl.tmp, mbs = cl.mbs;
    int fc = w.fail_code;
    double fval = w.fail_value;
    double pipeline = CUDART_NAN, dpsync = CUDART_NAN;
    int best_r = -1;
    const int* PL = ew->place;
    if (fc == 0) {
      if (pp >= 3 || p.cuts_given) {
        // (memoised DP: the cuts of this candidate's signature representative)
        // (memoised DP: the cuts of this candidate's signature run)
        const uint8_t* ci = (p.rep_of && !p.cuts_given && u < p.n_dp && !(p.memo_bad && *p.memo_bad))
                                ? p.repcuts + (uint64_t)p.rep_of[u] * (maxpp + 1)
                                : p.cutsb + u * (maxpp + 1);
        for (int q = lane; q <= pp; q += 32) cutsW[q] = ci[q];
      } else {
        // pp <= 2 never reaches K_dp: single stage, or the two-stage DP
        // solved here by the warp (light_cut2)
        const int c1 = pp == 2 ? light_cut2(p, cl, w.cls, u, lane) : p.L;
        if (lane == 0) {
          cutsW[0] = 0;
          cutsW[1] = pp == 2 ? (int)(uint8_t)c1 : p.L;
          if (pp == 2) cutsW[2] = p.L;
        }
      }
      const int32_t* prow = p.placeb + u * D;
      if (D <= 32) {
        if (lane < D) ew->place[lane] = prow[lane];
      } else {
        PL = prow;
      }
      __syncwarp();
      // ---- stage_time (cost_model.cpp:88-98), params_in_range (types.cpp:34-40)
      const double* tl = p.times + (size_t)cl.pair * p.L;
      double worst_p = 0.0;
      for (int j = lane; j < pp; j += 32) {
        double sum = 0.0, ps = 0.0;
        for (int l = cutsW[j]; l < cutsW[j + 1]; ++l) {
          sum += tl[l];
          ps += p.param[l];
        }
        stW[j] = sum;
        sparW[j] = ps;
        worst_p = std_max(worst_p, ps / tmp);
      }
      // ---- per-device parameter ceiling (optimizer.cpp:159-169) ---------
      for (int o = 16; o > 0; o >>= 1)
        worst_p = std_max(worst_p, __shfl_xor_sync(0xffffffffu, worst_p, o));
      __syncwarp();
      if (p.has_ceiling && worst_p > p.ceiling) fc = AMP_FAIL_CEILING;
    }
    if (fc == 0) {
      // ---- estimate: pipeline term (cost_model.cpp:176-212) -------------
      double slowest_stage = stW[0];  // std::max_element: first maximum
      for (int j = 1; j < pp; ++j)
        if (slowest_stage < stW[j]) slowest_stage = stW[j];
      const double g1 = (double)(cl.gas - 1);
      double tr = -CUDART_INF;
      int rr = -1;
      const int ne = pp - 1;
      if (dp * ne <= 32) {
        // replica_edge_times (145-162): lane (r, q) computes edge q of
        // replica r, then lane r sums its edges in order
        if (lane < dp * ne) {
          const int r = lane / ne, q = lane - r * ne;
          const int cut = cutsW[q + 1];
          const double volume = p.act[cut - 1] * mbs;
          double b = CUDART_INF;
          for (int s = 0; s < tmp; ++s)
            b = std_min(b, BW[(size_t)PL[(q * dp + r) * tmp + s] * D +
                              PL[((q + 1) * dp + r) * tmp + s]]);
          ew->ebuf[lane] = volume / b;
        }
        __syncwarp();
        if (lane < dp) {
          double sum = 0.0;
          for (int q = 0; q < ne; ++q) sum = sum + ew->ebuf[lane * ne + q];
          for (int j = 0; j < pp; ++j) sum = sum + stW[j];
          const double t = g1 * slowest_stage + sum;  // pipeline_time (100-120)
          if (t > tr) {
            tr = t;
            rr = lane;
          }
        }
      } else {
        for (int r = lane; r < dp; r += 32) {
          double sum = 0.0;
          for (int q = 0; q < ne; ++q) {
            const int cut = cutsW[q + 1];
            const double volume = p.act[cut - 1] * mbs;
            double b = CUDART_INF;
            for (int s = 0; s < tmp; ++s)
              b = std_min(b, BW[(size_t)PL[(q * dp + r) * tmp + s] * D +
                                PL[((q + 1) * dp + r) * tmp + s]]);
            sum = sum + volume / b;
          }
          for (int j = 0; j < pp; ++j) sum = sum + stW[j];
          const double t = g1 * slowest_stage + sum;
          if (t > tr) {  // strict '>' over ascending r: first maximum
            tr = t;
            rr = r;
          }
        }
      }
      for (int o = 16; o > 0; o >>= 1) {  // max, lowest replica on ties
        const double ov = __shfl_xor_sync(0xffffffffu, tr, o);
        const int oi = __shfl_xor_sync(0xffffffffu, rr, o);
        if (oi >= 0 && (rr < 0 || ov > tr || (ov == tr && oi < rr))) {
          tr = ov;
          rr = oi;
        }
      }
      // ---- dpsync_time (122-143): groups (stage j, shard s) -------------
      double worst = 0.0;
      int bad_group = 0x7fffffff;
      double bad_value = 0.0;
      if (dp != 1) {
        const int ngroups = pp * tmp;
        if (ngroups * dp <= 32) {
          // lane (g, r1): pairwise minimum over r2 > r1 (make_comm_group 23-38)
          const int g = lane / dp, r1 = lane % dp;
          double b = CUDART_INF;
          if (g < ngroups) {
            const int j = g / tmp, s = g % tmp;
            const int d1 = PL[(j * dp + r1) * tmp + s];
            for (int r2 = r1 + 1; r2 < dp; ++r2)
              b = std_min(b, BW[(size_t)d1 * D + PL[(j * dp + r2) * tmp + s]]);
          }
          for (int o = 1; o < dp; o <<= 1) {  // min over the dp lanes of a group
            const double ob = __shfl_down_sync(0xffffffffu, b, o);
            if (r1 + o < dp) b = std_min(b, ob);
          }
          if (g < ngroups && r1 == 0) {
            const double message = sparW[g / tmp] * p.bpp / tmp;
            if (!(b > 0)) {
              bad_group = g;
              bad_value = b;
            } else {
              worst = 2.0 * (double)(dp - 1) * message / ((double)dp * b);
            }
          }
        } else {
          for (int g = 0; g < ngroups; ++g) {
            const int j = g / tmp, s = g % tmp;
            double b = CUDART_INF;
            if (p.nodebw) {
              // node-determined symmetric links: the minimum over the device
              // pairs of the group (cost_model.cpp:23-38) equals the minimum
              // over its node pairs plus the intra-node link of every node
              // holding >= 2 of its devices (min is exact in any order)
              const int NW = p.node_words, NN = p.n_nodes;
              for (int x = lane; x < NW; x += 32) nodeP[x] = nodeM[x] = 0u;
              __syncwarp();
              for (int r = lane; r < dp; r += 32) {
                const int n = p.node_of[PL[(j * dp + r) * tmp + s]];
                const unsigned bit = 1u << (n & 31);
                if (atomicOr(&nodeP[n >> 5], bit) & bit) atomicOr(&nodeM[n >> 5], bit);
              }
              __syncwarp();
              for (int n1 = lane; n1 < NW * 32; n1 += 32) {
                if (!((nodeP[n1 >> 5] >> (n1 & 31)) & 1u)) continue;
                const double* row = p.nodebw + (size_t)n1 * NN;
                if ((nodeM[n1 >> 5] >> (n1 & 31)) & 1u) b = std_min(b, row[n1]);
                for (int w = n1 >> 5; w < NW; ++w) {
                  unsigned m = nodeP[w];
                  if (w == (n1 >> 5)) m &= (n1 & 31) == 31 ? 0u : ~((2u << (n1 & 31)) - 1u);
                  while (m) {
                    const int n2 = w * 32 + __ffs(m) - 1;
                    m &= m - 1;
                    b = std_min(b, row[n2]);
                  }
                }
              }
              __syncwarp();
            } else {
              for (int r1 = lane; r1 < dp; r1 += 32) {
                const int d1 = PL[(j * dp + r1) * tmp + s];
                for (int r2 = r1 + 1; r2 < dp; ++r2)
                  b = std_min(b, BW[(size_t)d1 * D + PL[(j * dp + r2) * tmp + s]]);
              }
            }
            for (int o = 16; o > 0; o >>= 1) b = std_min(b, __shfl_xor_sync(0xffffffffu, b, o));
            if (lane == 0) {
              const double message = sparW[j] * p.bpp / tmp;
              if (!(b > 0)) {
                if (g < bad_group) {
                  bad_group = g;
                  bad_value = b;
                }
              } else {
                worst = std_max(worst, 2.0 * (double)(dp - 1) * message / ((double)dp * b));
              }
            }
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          worst = std_max(worst, __shfl_xor_sync(0xffffffffu, worst, o));
          const int og = __shfl_xor_sync(0xffffffffu, bad_group, o);
          const double ov = __shfl_xor_sync(0xffffffffu, bad_value, o);
          if (og < bad_group) {
            bad_group = og;
            bad_value = ov;
          }
        }
      }
      if (bad_group != 0x7fffffff) {
        fc = AMP_FAIL_ALLREDUCE_BANDWIDTH;
        fval = bad_value;
      } else {
        pipeline = tr;
        dpsync = worst;
        best_r = rr;
      }
    }
    // ---- batched simulator ---------------------------
    double simv = CUDART_NAN;
    if (p.all_sim && fc == 0)  // fc is warp-uniform
      simv = sim_iteration(p, cl, PL, cutsW, stW, dpsync, lane,
                           p.simbuf + ((size_t)blockIdx.x * kEstWarps + wib) * p.gbs);
    if (p.all_sim && lane == 0) p.all_sim[w.out] = simv;
    // ---- record ---------------------------------------------------------
    amp_record rec;
    rec.index = w.index;
    rec.pp = pp;
    rec.dp = dp;
    rec.tmp = tmp;
    rec.mbs = mbs;
    rec.fail_code = fc;
    rec.fail_layer = fc == AMP_FAIL_PROFILE_MISS ? w.fail_layer : -1;
    rec.fail_value = fc == AMP_FAIL_P2P_BANDWIDTH || fc == AMP_FAIL_ALLREDUCE_BANDWIDTH ? fval : 0.0;
    const bool ok = fc == 0;
    rec.pipeline_time = ok ? pipeline : CUDART_NAN;
    rec.dpsync_time = ok ? dpsync : CUDART_NAN;
    rec.total = ok ? pipeline + dpsync : CUDART_NAN;
    if (lane == 0) {
      if (p.all) p.all[w.out] = rec;
      if (p.k > 0) {
        // CTA top-k under a smem spinlock; most records fail the cheap
        // pre-check against the current k-th entry without taking the lock
        const int kf = *(volatile int*)&kth_failed;
        const double kt = *(volatile double*)&kth_total;
        const int rf = ok ? 0 : 1;
        // (failed items: the index decides; the k-th only improves, so a
        // stale read is looser, never stricter)
        const unsigned long long ki = *(volatile unsigned long long*)&kth_index;
        const bool reject = rf > kf || (rf == 0 && kf == 0 && rec.total > kt) ||
                            (rf == 1 && kf == 1 && rec.index > ki);
        if (!reject) {
          while (atomicCAS(&lock, 0, 1) != 0) __nanosleep(32);
          __threadfence_block();
          int n = *(volatile int*)&n_top;
          topk_insert(mytop, n, p.k, rec);
          *(volatile int*)&n_top = n;
          if (n == p.k) {
            *(volatile int*)&kth_failed = mytop[p.k - 1].fail_code != 0;
            *(volatile double*)&kth_total = mytop[p.k - 1].total;
            *(volatile unsigned long long*)&kth_index = mytop[p.k - 1].index;
          }
          __threadfence_block();
          atomicExch(&lock, 0);
        }
      }
    }
    // (the strategy survives the failures raised after it was assigned,
    // optimizer.cpp:157-171: the parameter ceiling, the all-reduce bandwidth)
    const bool has_strategy = ok || fc == AMP_FAIL_CEILING || fc == AMP_FAIL_ALLREDUCE_BANDWIDTH;
    if (p.all_cuts) {
      int32_t* o = p.all_cuts + w.out * (maxpp + 1);
      for (int q = lane; q <= maxpp; q += 32) o[q] = (has_strategy && q <= pp) ? cutsW[q] : -1;
    }
    if (p.all_stage) {
      double* o = p.all_stage + w.out * maxpp;
      for (int q = lane; q < maxpp; q += 32) o[q] = (ok && q < pp) ? stW[q] : CUDART_NAN;
    }
    if (p.all_edge) {
      double* o = p.all_edge + w.out * maxpp;
      for (int q = lane; q < maxpp; q += 32) {
        double v = CUDART_NAN;
        if (ok && q + 1 < pp) {
          const int cut = cutsW[q + 1];
          double b = CUDART_INF;
          for (int s = 0; s < tmp; ++s)
            b = std_min(b, BW[(size_t)PL[(q * dp + best_r) * tmp + s] * D +
                              PL[((q + 1) * dp + best_r) * tmp + s]]);
          v = p.act[cut - 1] * mbs / b;
        }
        o[q] = v;
      }
    }
    if (p.all_place) {
      int32_t* o = p.all_place + w.out * D;
      for (int x = lane; x < D; x += 32) o[x] = has_strategy ? PL[x] : -1;
    }
    __syncwarp();
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

}  // namespace amp
