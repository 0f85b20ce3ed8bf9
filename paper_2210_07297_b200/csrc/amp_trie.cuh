// amp_trie.cuh — the layer-partition DP shared across signature prefixes.
//
// Stage j of the DP (pipeline_dp.cpp:114-131) reads stage j-1 and the edge
// costs of boundary j-2 only.  So the values and argmins of stage j are a
// function of the class and of the boundary codes c_0 .. c_{j-2}: every
// signature (class, c_0 .. c_{k-2}) with the same first j-1 codes has the
// same stage-j table.  After the signature sort (amp_dedup.cuh) the
// representatives are in key order, i.e. lexicographic in (class, c_0,
// c_1, ...).  The signatures sharing a prefix of length d therefore form a
// run; the runs are the nodes of a trie, and stage j is solved once per node
// of depth j-1 instead of once per signature.  The operations per cell and
// cut are those of the per-candidate kernels (same operands, same order,
// same strict '<'), so every cut is bit-identical (tested against
// AMP_FLAG_NO_DEDUP).
//
// Layout: the nodes of one depth are class-contiguous.  The stage-j table of
// class c is cell-major over its K nodes — value / argmin of (cell x, node
// n) at base_c + x*K + (n - nb_c) — so the threads of a warp share a cell
// (program record, predecessor list, prefix, domain: broadcast loads, no
// divergence in the cut loop) and touch consecutive nodes (coalesced).
//
//   K_flag(d)    head flags of the depth-d runs        -> scan -> nid_d (1-based)
//   K_nodes(d)   first signature and parent of every node, class node ranges
//   (host)       one read of the ranges; table bases, per-stage item lists
//   K_stage(j)   one thread per (class, cell of N_j, node of depth j-1)
//   K_back       one thread per signature: walk its trie path, write its cuts
#pragma once

#include "amp_common.cuh"
#include "amp_dp_sparse.cuh"

namespace amp {

constexpr int kTrieMaxCls = 256;  // classes per stage list held in smem

struct TrieParams {
  // signatures (run heads of the sorted keys)
  const uint64_t* n_rep;      // device count
  const uint64_t* rep_key;    // [n_rep]
  const uint32_t* rep_list;   // [n_rep] chunk item of each signature
  int32_t nq, cb;             // codes per key, bits per code
  int32_t L, max_pp;
  int32_t n_cls, pad0;
  uint64_t stride;            // n_rep (row stride of the per-depth arrays)
  uint32_t* nid;              // [nq + 1][stride]  node id (1-based) at depth d
  uint32_t* first;            // [nq + 1][stride]  first signature of each node
  uint32_t* parent;           // [nq + 1][stride]  node of depth d-1 it extends
  uint32_t* flags;            // [stride] scratch
  uint32_t* range;            // [nq + 1][n_cls][2]  node range [nb, ne) of each class
  // host-computed tables (after one read of `range`)
  const uint64_t* vbase;      // [nq + 1][n_cls]  value-table base of (depth, class)
  const uint64_t* bbase;      // [nq + 1][n_cls]  argmin-table base of (depth, class)
  const int32_t* st_cls;      // [max_pp + 1][n_cls]  classes of stage j's item list
  const uint64_t* st_item;    // [max_pp + 1][n_cls + 1]  exclusive item bases
  const int32_t* st_n;        // [max_pp + 1]  classes in stage j's list
  // problem tables
  const ClassDev* cls;
  const int32_t* class_prog;
  const ProgDev* progs;
  const uint32_t* stage;
  const uint2* cellrec;
  const uint16_t* preds;
  const double* prefix;
  const double* domain;
  int32_t nv_stride, n_codes;
  const double* qtab;         // [n_cls][n_codes][L]
  const double* v1g;          // stage-1 values per class (v1off)
  const uint64_t* v1off;      // [n_cls]
  // stage storage
  double* vals[2];            // ping-pong by stage parity
  uint8_t* bp;                // argmins of all stages
  uint8_t* repcuts;           // [n_rep][max_pp + 1] cuts per signature run
};

__device__ __forceinline__ int key_cls(const TrieParams& p, uint64_t k) {
  return (int)(k >> (p.nq * p.cb));
}
__device__ __forceinline__ int key_code(const TrieParams& p, uint64_t k, int q) {
  return (int)((k >> ((p.nq - 1 - q) * p.cb)) & ((1ull << p.cb) - 1));
}

// head flags of the depth-d runs (d codes + the class)
__global__ void k_trie_flag(TrieParams p, int d) {
  const uint64_t n = *p.n_rep;
  const int sh = (p.nq - d) * p.cb;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x)
    p.flags[r] = (r == 0 || (p.rep_key[r] >> sh) != (p.rep_key[r - 1] >> sh)) ? 1u : 0u;
}

// first signature and parent of every depth-d node; node range of each
// class (the failed / pp <= 2 run, key ~0, belongs to no class)
__global__ void k_trie_nodes(TrieParams p, int d) {
  const uint64_t n = *p.n_rep;
  const uint32_t* nid = p.nid + (size_t)d * p.stride;
  uint32_t* first = p.first + (size_t)d * p.stride;
  uint32_t* parent = p.parent + (size_t)d * p.stride;
  uint32_t* range = p.range + (size_t)d * p.n_cls * 2;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t node = nid[r] - 1;
    if (r == 0 || nid[r] != nid[r - 1]) {  // node head
      first[node] = (uint32_t)r;
      parent[node] = d >= 2 ? p.nid[(size_t)(d - 1) * p.stride + r] - 1 : 0;
    }
    const uint64_t key = p.rep_key[r];
    if (key == ~0ull) continue;
    const int c = key_cls(p, key);
    // the class's first signature opens its node range, its last closes it
    if (r == 0 || key_cls(p, p.rep_key[r - 1]) != c) range[2 * c] = node;
    if (r + 1 == n || p.rep_key[r + 1] == ~0ull || key_cls(p, p.rep_key[r + 1]) != c)
      range[2 * c + 1] = node + 1;
  }
}

// Per-class facts of one stage, cached in shared memory.
struct TrieSlot {
  uint64_t ibase;      // first item of the class in the stage
  uint64_t vbase, bbase, vbase_p;  // table bases at depth d, d (argmins), d-1
  uint64_t v1off;
  uint32_t nb, K, nb_p, K_p;       // node ranges at depth d and d-1
  uint32_t cell0, pred_base_lo, pred_base_hi, pad;  // program: first cell of N_j, preds
  int32_t c, pair, gas, chunks;    // class, its (tmp, mbs) pair, gas, node chunks
};

#ifndef AMP_TRIE_NB
#define AMP_TRIE_NB 4
#endif
constexpr int kTrieNB = AMP_TRIE_NB;  // nodes per thread: they share the cell's work

// Stage j: one thread per (class, cell x of N_j, chunk of kTrieNB nodes of
// depth j-1).  Per cut the predecessor index, t2 and the tolerance term are
// shared by the thread's nodes; each node adds its parent's value and its
// own edge (the per-candidate kernels' operations and order).
#ifndef AMP_TRIE_UNROLL
#define AMP_TRIE_UNROLL 2
#endif
#ifndef AMP_TRIE_MINB
#define AMP_TRIE_MINB 2
#endif
constexpr int kTrieUnroll = AMP_TRIE_UNROLL;
__global__ void __launch_bounds__(256, AMP_TRIE_MINB) k_trie_stage(TrieParams p, int j, uint64_t total,
                                                    unsigned long long* exec) {
  __shared__ TrieSlot slot[kTrieMaxCls];
  __shared__ uint64_t ibase[kTrieMaxCls + 1];
  const int nc = p.st_n[j];
  const int d = j - 1, L = p.L, LP = L + 1;
  for (int x = threadIdx.x; x <= nc; x += blockDim.x) {
    ibase[x] = p.st_item[(size_t)j * (p.n_cls + 1) + x];
    if (x == nc) continue;
    TrieSlot t;
    const int c = p.st_cls[(size_t)j * p.n_cls + x];
    const ClassDev cl = p.cls[c];
    const ProgDev pg = p.progs[p.class_prog[c]];
    const uint32_t* rg = p.range + ((size_t)d * p.n_cls + c) * 2;
    t.ibase = ibase[x];
    t.c = c;
    t.pair = cl.pair;
    t.gas = cl.gas;
    t.nb = rg[0];
    t.K = rg[1] - rg[0];
    t.chunks = (t.K + kTrieNB - 1) / kTrieNB;
    t.vbase = p.vbase[(size_t)d * p.n_cls + c];
    t.bbase = p.bbase[(size_t)d * p.n_cls + c];
    if (j > 2) {
      const uint32_t* rgp = p.range + ((size_t)(d - 1) * p.n_cls + c) * 2;
      t.nb_p = rgp[0];
      t.K_p = rgp[1] - rgp[0];
      t.vbase_p = p.vbase[(size_t)(d - 1) * p.n_cls + c];
    } else {
      t.nb_p = 0;
      t.K_p = 1;
      t.vbase_p = 0;
    }
    t.v1off = p.v1off[c];
    t.cell0 = pg.cell_base + p.stage[pg.stage_base + j - 1];
    t.pred_base_lo = (uint32_t)pg.pred_base;
    t.pred_base_hi = (uint32_t)(pg.pred_base >> 32);
    t.pad = 0;
    slot[x] = t;
  }
  __syncthreads();
  unsigned long long mine = 0;
  const double* Vprev = p.vals[(j - 1) & 1];
  double* Vcur = p.vals[j & 1];
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nc - 1;  // class slot: last with ibase <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ibase[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const TrieSlot& S = slot[lo];
    const uint64_t off = t - S.ibase;
    const uint32_t x = (uint32_t)(off / (uint32_t)S.chunks);
    const uint32_t n0 = (uint32_t)(off % (uint32_t)S.chunks) * kTrieNB;  // local node
    const int nn = (int)min((uint32_t)kTrieNB, S.K - n0);
    const uint2 rec = p.cellrec[S.cell0 + x];
    const int i = rec.x >> 16, m = rec.x & 0xffff;
    const uint16_t* q = p.preds + (((uint64_t)S.pred_base_hi << 32) | S.pred_base_lo) + rec.y;
    const double* Pf = p.prefix + (size_t)S.pair * LP;
    const double dm = p.domain[(size_t)S.pair * p.nv_stride + m];
    const double Pi = Pf[i];
    const double g1 = (double)(S.gas - 1);
    const double* Vp[kTrieNB];
    const double* E[kTrieNB];
    double best[kTrieNB];
    int bc[kTrieNB];
#pragma unroll
    for (int b = 0; b < kTrieNB; ++b) {
      const uint32_t node = S.nb + n0 + (b < nn ? b : 0);  // pad with the first node
      const uint64_t key = p.rep_key[p.first[(size_t)d * p.stride + node]];
      E[b] = p.qtab + ((size_t)S.c * p.n_codes + key_code(p, key, j - 2)) * L;
      if (j == 2) {
        Vp[b] = p.v1g + S.v1off;
      } else {
        const uint32_t pn = p.parent[(size_t)d * p.stride + node] - S.nb_p;
        Vp[b] = Vprev + S.vbase_p + pn;
      }
      best[b] = CUDART_INF;
      bc[b] = -1;
    }
    const uint32_t Kp = S.K_p;
#pragma unroll kTrieUnroll
    for (int cut = j - 1; cut < i; ++cut) {  // pipeline_dp.cpp:114-131
      const double t2 = Pi - Pf[cut];
      const double term = t2 > dm ? g1 * (t2 - dm) : 0.0;
      const size_t idx = (size_t)q[cut - (j - 1)] * Kp;
#pragma unroll
      for (int b = 0; b < kTrieNB; ++b) {
        const double g = ((Vp[b][idx] + term) + t2) + E[b][cut];
        if (g < best[b]) {
          best[b] = g;
          bc[b] = cut;
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kTrieNB; ++b) {
      if (b >= nn) break;
      const uint64_t o = (uint64_t)x * S.K + n0 + b;
      Vcur[S.vbase + o] = best[b];
      p.bp[S.bbase + o] = (uint8_t)bc[b];
    }
    mine += (unsigned long long)(i - (j - 1)) * nn;
  }
  if (exec) {  // executed inner iterations (roofline accounting): one
               // global atomic per warp (a 64-bit smem atomicAdd is a CAS loop)
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(exec, mine);
  }
}

// One thread per signature: backtrack (pipeline_dp.cpp:134-148) along its
// trie path and write the cuts of its representative item.
__global__ void k_trie_back(TrieParams p) {
  const uint64_t n = *p.n_rep;
  const int L = p.L;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = p.rep_key[r];
    if (key == ~0ull) continue;  // failed / pp <= 2 items (K_est)
    const int c = key_cls(p, key);
    const ClassDev cl = p.cls[c];
    const int k = cl.pp;
    const ProgDev pg = p.progs[p.class_prog[c]];
    const uint32_t* ss = p.stage + pg.stage_base;
    uint8_t* co = p.repcuts + r * (p.max_pp + 1);  // compact, by signature run
    co[k] = (uint8_t)L;
    uint32_t x = ss[k - 1];  // N_k = {(L, 0)}
    for (int j = k; j >= 2; --j) {
      const int d = j - 1;
      const uint32_t* rg = p.range + ((size_t)d * p.n_cls + c) * 2;
      const uint32_t node = p.nid[(size_t)d * p.stride + r] - 1;
      const uint64_t o = (uint64_t)(x - ss[j - 1]) * (rg[1] - rg[0]) + (node - rg[0]);
      const int cut = p.bp[p.bbase[(size_t)d * p.n_cls + c] + o];
      co[j - 1] = (uint8_t)cut;
      const uint2 rec = p.cellrec[pg.cell_base + x];
      x = ss[j - 2] + p.preds[pg.pred_base + rec.y + (cut - (j - 1))];
    }
    co[0] = 0;
  }
}

// Stage-1 values of every heavy class (pipeline_dp.cpp:102-107), once per
// context: v1g[v1off[c] + x] for the cells x of the class program's N_1.
__global__ void k_trie_v1(const ClassDev* cls, const int32_t* class_prog, const ProgDev* progs,
                          const uint32_t* stage, const uint32_t* cells, const double* prefix,
                          const double* domain, int nv_stride, int L, const int32_t* heavy,
                          int n_heavy, const uint64_t* v1off, double* v1g) {
  for (int h = blockIdx.x; h < n_heavy; h += gridDim.x) {
    const int c = heavy[h];
    const ClassDev cl = cls[c];
    const ProgDev pg = progs[class_prog[c]];
    const uint32_t* ss = stage + pg.stage_base;
    const double* Pf = prefix + (size_t)cl.pair * (L + 1);
    const double* Dm = domain + (size_t)cl.pair * nv_stride;
    const double g1 = (double)(cl.gas - 1);
    for (uint32_t x = ss[0] + threadIdx.x; x < ss[1]; x += blockDim.x) {
      const uint32_t cell = cells[pg.cell_base + x];
      const int i = cell >> 16, m = cell & 0xffff;
      const double t1 = Pf[i] - Pf[0];
      v1g[v1off[c] + (x - ss[0])] = g1 * max0(t1 - Dm[m]) + t1;
    }
  }
}

}  // namespace amp
