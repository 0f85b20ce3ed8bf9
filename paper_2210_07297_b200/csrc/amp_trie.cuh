// amp_trie.cuh — the layer-partition DP shared across signature prefixes.
//
// Stage j of the DP (pipeline_dp.cpp:114-131) reads stage j-1 and the edge
// costs of boundary j-2 only, so the stage-j table of a candidate is a
// function of its class and of its boundary codes c_0 .. c_{j-2}.  The
// distinct signatures (class, c_0 .. c_{pp-2}) of a chunk (amp_dedup.cuh)
// are the leaves of a trie whose depth-d nodes are the distinct prefixes
// (class, c_0 .. c_{d-1}); stage j is solved once per node of depth j-1
// instead of once per signature.  Per cell and cut the operations are those
// of pipeline_dp.cpp:118-127 (same operands, same order, same strict '<'),
// so every cut is bit-identical to the reference (tested against the
// one-DP-per-candidate kernel).
//
// Everything is built and scheduled on the device — no host round trip:
//   K_sig_init     the hash table's distinct keys -> signature list (hash
//                  order), slot -> signature map, root of each signature,
//                  depth-1 child marks
//   per depth d = 1 .. nq:
//     K_level_up   per-CTA sums of the child marks          (fixed grid)
//     K_level_down exclusive scan -> depth-d node ids in (parent, code)
//                  order: lexicographic, class-contiguous, children of a
//                  parent adjacent.  The last CTA plans the level: per
//                  class node range, tiles, value / argmin table bases
//                  (device bump allocation; capacity overflow raises `ovf`
//                  and the signature-mode K_dp (amp_dp_multi.cuh) solves the
//                  chunk instead)
//     K_level_assign each signature's depth-d node; marks for depth d+1
//     K_trie_tiles   stage j = d+1.  One CTA per tile = (class, run of <= TN
//                  consecutive depth-d nodes).  The tile's parents are
//                  consecutive depth-(d-1) nodes; their stage-(j-1) tables
//                  are staged in shared memory (transposed, odd stride: the
//                  lanes of a warp read distinct banks), with the class's
//                  edge rows and prefix sums.  Thread = (cell of N_j, group
//                  of 4 nodes): per cut the predecessor index, t2 and the
//                  tolerance term are shared by the 4 nodes.
//   K_trie_back    one thread per signature: backtrack (pipeline_dp.cpp:
//                  134-148) along its trie path, write its cuts.
#pragma once

#include "amp_common.cuh"
#include "amp_dp_sparse.cuh"

namespace amp {

constexpr int kTrieMaxD1 = 64;       // depths 0 .. nq (keys are <= 63 bits, >= 1 bit per code)
constexpr int kTrieThreads = 256;    // K_trie_tiles block
constexpr int kTrieNB = 4;           // nodes per thread (share the cell's work)
constexpr int kScanGrid = 296;       // CTAs of the level scans
constexpr int kScanThreads = 512;
constexpr int kTrieSmem = 46 * 1024; // K_trie_tiles dynamic smem budget (4 CTAs / SM)

// Level state, in device memory (reset by K_sig_init every chunk).
struct TrieState {
  uint32_t cnt[kTrieMaxD1];        // nodes per depth (depth 0: the heavy classes)
  uint64_t node_off[kTrieMaxD1];   // start of depth d's nodes in the node arrays
  uint32_t ntiles[kTrieMaxD1];     // tiles of stage d+1
  unsigned long long bp_bump;      // argmin bytes allocated
  uint32_t ovf;                    // capacity exceeded: signature-mode K_dp instead
  uint32_t ticket;                 // last-CTA election of K_level_down
};

// Per (class, stage j) facts of the class's pruned program (host-built).
struct TrieStage {
  uint32_t cell0;   // first cell of N_j in cellrec (absolute)
  uint32_t n;       // |N_j|
  uint32_t iters;   // (cell, cut) pairs of stage j (unpadded)
  uint32_t tn;      // nodes per K_trie_tiles tile
};

struct TrieParams {
  // signatures: the distinct keys of the chunk's hash table
  const unsigned long long* n_sig;  // device count
  const uint32_t* uniq;             // [n_sig] slots
  const unsigned long long* tkey;
  uint32_t* tval;                   // slot -> first item, rewritten to slot -> signature
  int32_t key_shift;                // epoch tag position (64: none)
  int32_t nq, cb, U, L, max_pp, n_cls, n_roots;
  uint64_t* sig_key;                // [n] class | codes
  uint32_t* rep_item;               // [n] first item of each signature
  uint32_t* nid;                    // [n] node at the current depth (local id)
  const int32_t* root_rank;         // [n_cls] rank among the roots (-1: not heavy)
  const int32_t* root_cls;          // [n_roots] class of each root
  TrieState* st;
  uint8_t* pres;                    // child marks [cnt[d-1] * U]
  uint32_t* cid;                    // their scan: child node id
  uint64_t pres_cap;
  uint32_t* partial;                // [kScanGrid]
  uint32_t* npar;                   // node arrays (absolute index node_off[d] + id)
  uint16_t* ncls;
  uint8_t* ncode;
  uint64_t node_cap;
  // level plans [kTrieMaxD1][n_cls] (tbase: [kTrieMaxD1][n_cls + 1])
  uint32_t* nb;
  uint32_t* nK;
  uint64_t* vbase;
  uint64_t* bbase;
  uint32_t* tbase;
  const TrieStage* tstage;          // [n_cls][max_pp + 1]
  double* varena[2];                // values of depth d in varena[d & 1]
  uint64_t vcap;                    // doubles per arena
  uint8_t* bparena;                 // argmins of every depth
  uint64_t bpcap;
  // problem tables
  const ClassDev* cls;
  const uint2* cellrec;
  const uint16_t* preds;
  const ProgDev* progs;
  const int32_t* class_prog;
  const double* prefix;
  const double* domain;
  int32_t nv_stride, n_codes;
  const double* qtab;               // [n_cls][n_codes][L]
  const double* v1g;                // stage-1 values per class (v1off)
  const uint64_t* v1off;
  uint8_t* repcuts;                 // [n_sig][max_pp + 1] cuts per signature
  unsigned long long* exec;         // [2]: DP instances, inner iterations (or NULL)
};

__device__ __forceinline__ int trie_cls(const TrieParams& p, uint64_t k) { return (int)(k >> (p.nq * p.cb)); }
__device__ __forceinline__ int trie_code(const TrieParams& p, uint64_t k, int q) {
  return (int)((k >> ((p.nq - 1 - q) * p.cb)) & (uint64_t)(p.U - 1));
}

// signature list, slot -> signature, roots, depth-1 marks; resets the state
__global__ void k_sig_init(TrieParams p) {
  const uint64_t n = *p.n_sig;
  if (p.st && blockIdx.x == 0 && threadIdx.x == 0) {  // (no state: trie off)
    p.st->cnt[0] = (uint32_t)p.n_roots;
    p.st->node_off[0] = 0;
    p.st->bp_bump = 0;
    p.st->ovf = 0;
    p.st->ticket = 0;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = p.uniq[i];
    const unsigned long long k = p.tkey[s];
    const uint64_t key = p.key_shift >= 64 ? k : (k & ((1ull << p.key_shift) - 1));
    p.sig_key[i] = key;
    p.rep_item[i] = p.tval[s];
    p.tval[s] = (uint32_t)i;
    if (p.pres) {
      const int c = trie_cls(p, key);
      const int r = p.root_rank[c];
      p.nid[i] = (uint32_t)r;
      if (p.cls[c].pp - 1 >= 1) p.pres[(uint64_t)r * p.U + trie_code(p, key, 0)] = 1;
    }
  }
}

__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v, uint32_t* sm) {
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  uint32_t t = 0;
  for (int x = 0; x < nw; ++x) t += sm[x];
  return t;
}

__device__ __forceinline__ uint64_t level_entries(const TrieParams& p, int d) {
  const uint64_t n = (uint64_t)p.st->cnt[d - 1] * (uint64_t)p.U;
  return n < p.pres_cap ? n : p.pres_cap;
}

__global__ void __launch_bounds__(kScanThreads) k_level_up(TrieParams p, int d) {
  __shared__ uint32_t sm[32];
  if (p.st->ovf) return;
  const uint64_t n = level_entries(p, d);
  const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint64_t b = (uint64_t)blockIdx.x * per, e = b + per < n ? b + per : n;
  uint32_t s = 0;
  for (uint64_t x = b + threadIdx.x; x < e; x += blockDim.x) s += p.pres[x];
  s = block_sum_u32(s, sm);
  if (threadIdx.x == 0) p.partial[blockIdx.x] = s;
}

// Scan of the child marks -> depth-d nodes; clears the marks it reads; the
// last CTA plans the level.
__global__ void __launch_bounds__(kScanThreads) k_level_down(TrieParams p, int d) {
  __shared__ uint32_t sm[32], wsum[32];
  __shared__ uint64_t s_off;
  __shared__ int s_last;
  const int tid = threadIdx.x, l = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  const uint64_t n = level_entries(p, d);
  const uint64_t noff = d == 1 ? 0 : p.st->node_off[d - 1] + p.st->cnt[d - 1];
  const bool ovf = p.st->ovf || noff + n > p.node_cap;
  const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint64_t b = (uint64_t)blockIdx.x * per, e = b + per < n ? b + per : n;
  uint32_t base = 0;
  if (!ovf) {
    uint32_t s = 0;
    for (int x = tid; x < (int)blockIdx.x; x += blockDim.x) s += p.partial[x];
    base = block_sum_u32(s, sm);
  }
  const uint64_t poff = d == 1 ? 0 : p.st->node_off[d - 1];
  for (uint64_t x0 = b; x0 < e; x0 += blockDim.x) {
    const uint64_t x = x0 + tid;
    const uint32_t f = x < e ? p.pres[x] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f != 0);
    __syncthreads();
    if (l == 0) wsum[w] = __popc(bal);
    __syncthreads();
    uint32_t before = base;
    for (int q = 0; q < w; ++q) before += wsum[q];
    before += __popc(bal & ((1u << l) - 1));
    if (f) {
      if (!ovf) {
        const uint32_t id = before;
        const uint64_t par = x / (uint64_t)p.U;
        p.npar[noff + id] = (uint32_t)par;
        p.ncode[noff + id] = (uint8_t)(x % (uint64_t)p.U);
        p.ncls[noff + id] = (uint16_t)(d == 1 ? p.root_cls[par] : p.ncls[poff + par]);
        p.cid[x] = id;
      }
      p.pres[x] = 0;
    }
    for (int q = 0; q < nw; ++q) base += wsum[q];
  }
  // last CTA: level total and plan
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&p.st->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) p.st->ticket = 0;
  if (ovf) {
    if (tid == 0) p.st->ovf = 1;
    return;
  }
  uint32_t s = 0;
  for (int x = tid; x < (int)gridDim.x; x += blockDim.x) s += __ldcg(p.partial + x);
  const uint32_t total = block_sum_u32(s, sm);
  // per class: node range (nodes are class-sorted), tiles, table sizes
  uint32_t* nb = p.nb + (size_t)d * p.n_cls;
  uint32_t* nK = p.nK + (size_t)d * p.n_cls;
  const uint16_t* cl = p.ncls + noff;  // written by the other CTAs: read through L2 (__ldcg)
  for (int c = tid; c < p.n_cls; c += blockDim.x) {
    uint32_t lo = 0, hi = total;  // lower_bound(c)
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldcg(cl + mid) < c) lo = mid + 1;
      else hi = mid;
    }
    uint32_t lo2 = lo, hi2 = total;  // upper_bound(c)
    while (lo2 < hi2) {
      const uint32_t mid = (lo2 + hi2) >> 1;
      if (__ldcg(cl + mid) <= c) lo2 = mid + 1;
      else hi2 = mid;
    }
    nb[c] = lo;
    nK[c] = lo2 - lo;
  }
  __syncthreads();
  if (tid == 0) {
    p.st->cnt[d] = total;
    p.st->node_off[d] = noff;
    uint32_t* tb = p.tbase + (size_t)d * (p.n_cls + 1);
    uint64_t* vb = p.vbase + (size_t)d * p.n_cls;
    uint64_t* bb = p.bbase + (size_t)d * p.n_cls;
    uint32_t tiles = 0;
    uint64_t vacc = 0, bacc = p.st->bp_bump;
    for (int c = 0; c < p.n_cls; ++c) {
      tb[c] = tiles;
      vb[c] = vacc;
      bb[c] = bacc;
      const uint32_t K = nK[c];
      if (!K) continue;
      const TrieStage ts = p.tstage[(size_t)c * (p.max_pp + 1) + d + 1];
      tiles += (K + ts.tn - 1) / ts.tn;
      if (d < p.cls[c].pp - 1) vacc += (uint64_t)K * ts.n;  // leaves keep argmins only
      bacc += (uint64_t)K * ts.n;
    }
    tb[p.n_cls] = tiles;
    p.st->ntiles[d] = tiles;
    p.st->bp_bump = bacc;
    if (vacc > p.vcap || bacc > p.bpcap) p.st->ovf = 1;
  }
}

__global__ void k_level_assign(TrieParams p, int d) {
  if (p.st->ovf) return;
  const uint64_t n = *p.n_sig;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = p.sig_key[i];
    const int pp = p.cls[trie_cls(p, key)].pp;
    if (pp - 1 < d) continue;
    const uint32_t node = p.cid[(uint64_t)p.nid[i] * p.U + trie_code(p, key, d - 1)];
    p.nid[i] = node;
    if (pp - 1 >= d + 1) p.pres[(uint64_t)node * p.U + trie_code(p, key, d)] = 1;
  }
}

// Stage j = d + 1 over the depth-d nodes, one tile per CTA iteration.
__global__ void __launch_bounds__(kTrieThreads, 4) k_trie_tiles(TrieParams p, int d) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_c;
  if (p.st->ovf) return;
  const int tid = threadIdx.x, nt = blockDim.x, L = p.L, LP = L + 1, j = d + 1;
  const uint32_t ntiles = p.st->ntiles[d];
  const uint32_t* tb = p.tbase + (size_t)d * (p.n_cls + 1);
  const uint64_t noff = p.st->node_off[d], poff = d >= 2 ? p.st->node_off[d - 1] : 0;
  const double* Vprev = p.varena[(d - 1) & 1];
  double* Vcur = p.varena[d & 1];
  unsigned long long mine = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (tid == 0) {
      int lo = 0, hi = p.n_cls - 1;  // last class with tbase <= t
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tb[mid] <= t) lo = mid;
        else hi = mid - 1;
      }
      s_c = lo;
    }
    __syncthreads();
    const int c = s_c;
    const ClassDev cl = p.cls[c];
    const TrieStage ts = p.tstage[(size_t)c * (p.max_pp + 1) + j];
    const TrieStage tp = p.tstage[(size_t)c * (p.max_pp + 1) + j - 1];
    const uint32_t nbc = p.nb[(size_t)d * p.n_cls + c], Kc = p.nK[(size_t)d * p.n_cls + c];
    const uint32_t n0 = nbc + (t - tb[c]) * ts.tn;
    const uint32_t nn = min(ts.tn, nbc + Kc - n0);
    const bool leaf = d == cl.pp - 1;
    // parents (consecutive depth-(d-1) nodes) and their stage-(j-1) tables
    const uint32_t pfirst = d >= 2 ? p.npar[noff + n0] : 0;
    const uint32_t plast = d >= 2 ? p.npar[noff + n0 + nn - 1] : 0;
    const int P = (int)(plast - pfirst) + 1;
    const int Pst = P | 1;  // odd stride (in doubles): rows start on distinct banks
    const int Np = (int)tp.n, Nj = (int)ts.n;
    double* sV = reinterpret_cast<double*>(smem_raw);
    double* sE = sV + (size_t)Np * Pst;
    double* sPf = sE + (size_t)p.n_codes * L;
    if (d >= 2) {
      const uint32_t pnb = p.nb[(size_t)(d - 1) * p.n_cls + c];
      const double* src = Vprev + p.vbase[(size_t)(d - 1) * p.n_cls + c] + (uint64_t)(pfirst - pnb) * Np;
      for (int x = tid; x < P * Np; x += nt) {
        const int pl = x / Np, xp = x - pl * Np;
        sV[xp * Pst + pl] = src[x];
      }
    } else {
      const double* src = p.v1g + p.v1off[c];
      for (int x = tid; x < Np; x += nt) sV[x * Pst] = src[x];
    }
    int* sNode = reinterpret_cast<int*>(sPf + LP);  // (code << 16) | parent slot
    const double* qt = p.qtab + (size_t)c * p.n_codes * L;
    for (int x = tid; x < p.n_codes * L; x += nt) sE[x] = qt[x];
    for (int x = tid; x < LP; x += nt) sPf[x] = p.prefix[(size_t)cl.pair * LP + x];
    for (int x = tid; x < (int)nn; x += nt) {
      const uint64_t node = noff + n0 + x;
      sNode[x] = ((int)p.ncode[node] << 16) | (d >= 2 ? (int)(p.npar[node] - pfirst) : 0);
    }
    __syncthreads();
    const double g1 = (double)(cl.gas - 1);
    const double* dom = p.domain + (size_t)cl.pair * p.nv_stride;
    const ProgDev pg = p.progs[p.class_prog[c]];
    const uint16_t* pr = p.preds + pg.pred_base;
    const int G = (int)((nn + kTrieNB - 1) / kTrieNB);
    const int items = Nj * G;
    const uint64_t vb = leaf ? 0 : p.vbase[(size_t)d * p.n_cls + c];
    uint8_t* bpo = p.bparena + p.bbase[(size_t)d * p.n_cls + c];
    for (int it = tid; it < items; it += nt) {
      const int x = it / G, g = it - x * G;
      const uint2 rec = p.cellrec[ts.cell0 + x];
      const int i = rec.x >> 16, m = rec.x & 0xffff;
      const uint16_t* q = pr + rec.y;
      const double dm = dom[m];
      const double Pi = sPf[i];
      int pl[kTrieNB];
      const double* E[kTrieNB];
      double best[kTrieNB];
      int bc[kTrieNB];
#pragma unroll
      for (int b = 0; b < kTrieNB; ++b) {
        const int ln = g * kTrieNB + b < (int)nn ? g * kTrieNB + b : g * kTrieNB;  // pad: repeat
        const int nd = sNode[ln];
        pl[b] = nd & 0xffff;
        E[b] = sE + (nd >> 16) * L;
        best[b] = CUDART_INF;
        bc[b] = -1;
      }
#pragma unroll 2
      for (int cut = j - 1; cut < i; ++cut) {  // pipeline_dp.cpp:114-131
        const double t2 = Pi - sPf[cut];
        const double term = t2 > dm ? g1 * (t2 - dm) : 0.0;
        const double* row = sV + (int)q[cut - (j - 1)] * Pst;
#pragma unroll
        for (int b = 0; b < kTrieNB; ++b) {
          const double gv = ((row[pl[b]] + term) + t2) + E[b][cut];
          if (gv < best[b]) {
            best[b] = gv;
            bc[b] = cut;
          }
        }
      }
#pragma unroll
      for (int b = 0; b < kTrieNB; ++b) {
        const int ln = g * kTrieNB + b;
        if (ln >= (int)nn) break;
        const uint64_t o = (uint64_t)(n0 - nbc + ln) * Nj + x;
        if (!leaf) Vcur[vb + o] = best[b];
        bpo[o] = (uint8_t)bc[b];
      }
    }
    mine += (unsigned long long)nn * ts.iters;
    __syncthreads();  // smem reuse by the next tile
  }
  if (p.exec && tid == 0 && mine) atomicAdd(&p.exec[1], mine);
}

// One thread per signature: backtrack (pipeline_dp.cpp:134-148) along its
// trie path and write its cuts.
__global__ void k_trie_back(TrieParams p) {
  if (p.st->ovf) return;
  const uint64_t n = *p.n_sig;
  const int L = p.L;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = p.sig_key[i];
    const int c = trie_cls(p, key);
    const int k = p.cls[c].pp;
    const ProgDev pg = p.progs[p.class_prog[c]];
    const uint16_t* pr = p.preds + pg.pred_base;
    uint8_t* co = p.repcuts + i * (p.max_pp + 1);
    co[k] = (uint8_t)L;
    uint32_t node = p.nid[i];  // leaf (depth k-1, local id)
    uint32_t x = 0;            // N_k = {(L, 0)}
    for (int j = k; j >= 2; --j) {
      const int d = j - 1;
      const TrieStage ts = p.tstage[(size_t)c * (p.max_pp + 1) + j];
      const uint32_t nbc = p.nb[(size_t)d * p.n_cls + c];
      const int cut = p.bparena[p.bbase[(size_t)d * p.n_cls + c] + (uint64_t)(node - nbc) * ts.n + x];
      co[j - 1] = (uint8_t)cut;
      const uint2 rec = p.cellrec[ts.cell0 + x];
      x = pr[rec.y + (cut - (j - 1))];
      if (d >= 2) node = p.npar[p.st->node_off[d] + node];
    }
    co[0] = 0;
  }
  if (p.exec && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&p.exec[0], (unsigned long long)n);  // one DP instance per signature
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
