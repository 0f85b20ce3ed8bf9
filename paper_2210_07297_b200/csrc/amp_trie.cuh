// amp_trie.cuh — the layer-partition DP shared across signature prefixes.
//
// Stage j of the DP (pipeline_dp.cpp:114-131) reads stage j-1 and the edge
// costs of boundary j-2 only, so the values and argmins of stage j are a
// function of the class and of the boundary codes c_0 .. c_{j-2}: every
// signature (class, c_0 .. c_{k-2}) with the same first j-1 codes has the
// same stage-j table.  After the signature sort (amp_dedup.cuh) the
// representatives are in key order, i.e. lexicographic in (class, c_0,
// c_1, ...), so the signatures sharing a prefix of length d are a run: the
// runs are the nodes of a trie, and stage j is solved once per node of
// depth j-1 instead of once per signature.  The operations per cell and cut
// are those of the per-candidate kernels (same operands, same order, same
// strict '<'), so every cut is bit-identical (tested against
// AMP_FLAG_NO_DEDUP).
//
//   K_flag(d)   head flag of each depth-d run        -> scan -> nid_d (1-based)
//   K_first     first representative of every node, per depth
//   K_size(d)   |N_{d+1}| of each depth-d node (0 when the class has pp <= d)
//               -> exclusive scan -> voff_d (values / backpointer offsets)
//   K_stage(j)  one thread per (node of depth j-1, cell of N_j): the cut loop
//               over the parent node's stage-(j-1) values (stage 1 from the
//               class table V1g); writes values (ping-pong) + u8 argmins
//   K_back      one thread per signature: walk its trie path, write its cuts
#pragma once

#include "amp_common.cuh"
#include "amp_dp_sparse.cuh"

namespace amp {

struct TrieParams {
  // signatures (run heads of the sorted keys)
  const uint64_t* n_rep;      // device count
  const uint64_t* rep_key;    // [n_rep]
  const uint32_t* rep_list;   // [n_rep] chunk item of each signature
  int32_t nq, cb;             // codes per key, bits per code
  int32_t L, max_pp;
  uint64_t stride;            // n_rep (row stride of the per-depth arrays)
  uint32_t* nid;              // [nq + 1][stride]  node id (1-based) at depth d
  uint32_t* first;            // [nq + 1][stride]  first signature of each node
  uint64_t* voff;             // [nq + 1][stride + 1] offsets of stage d+1 tables
  uint32_t* flags;            // [stride] scratch
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
  uint8_t* bp;                // all stages: bp[bbase_j + voff_{j-1}[node] + x]
  const uint64_t* bbase;      // [max_pp + 1] host-computed stage bases
  uint8_t* cutsb;             // [n_chunk][max_pp + 1]
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

// first signature of every depth-d node
__global__ void k_trie_first(TrieParams p, int d) {
  const uint64_t n = *p.n_rep;
  const uint32_t* nid = p.nid + (size_t)d * p.stride;
  uint32_t* first = p.first + (size_t)d * p.stride;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x)
    if (r == 0 || nid[r] != nid[r - 1]) first[nid[r] - 1] = (uint32_t)r;
}

// stage-(d+1) table size of every depth-d node; 0 beyond the depth's node
// count, for classes with pp <= d and for the failed / pp <= 2 run
__global__ void k_trie_size(TrieParams p, int d, uint64_t* size) {
  const uint64_t n = *p.n_rep;
  const uint32_t* nid = p.nid + (size_t)d * p.stride;
  const uint32_t* first = p.first + (size_t)d * p.stride;
  const uint32_t n_nodes = n ? nid[n - 1] : 0;
  const int j = d + 1;  // the stage these nodes solve
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= p.stride;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = 0;
    const uint64_t key = x < n_nodes ? p.rep_key[first[x]] : ~0ull;
    const int c = key == ~0ull ? 0 : key_cls(p, key);
    if (key != ~0ull && p.cls[c].pp >= j) {
      const ProgDev pg = p.progs[p.class_prog[c]];
      const uint32_t* ss = p.stage + pg.stage_base;
      s = ss[j] - ss[j - 1];
    }
    size[x] = s;
  }
}

// Stage j: one thread per (node of depth j-1, cell of N_j).
__global__ void __launch_bounds__(256) k_trie_stage(TrieParams p, int j, uint64_t total,
                                                    unsigned long long* exec) {
  __shared__ unsigned long long cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  unsigned long long mine = 0;
  const int d = j - 1, L = p.L, LP = L + 1;
  const uint64_t n = *p.n_rep;
  const uint32_t* nid = p.nid + (size_t)d * p.stride;
  const uint32_t* first = p.first + (size_t)d * p.stride;
  const uint64_t* voff = p.voff + (size_t)d * (p.stride + 1);
  const uint32_t n_nodes = n ? nid[n - 1] : 0;
  const double* Vprev = p.vals[(j - 1) & 1];
  double* Vcur = p.vals[j & 1];
  uint8_t* bpj = p.bp + p.bbase[j];
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    // node: last x with voff[x] <= t (voff is an exclusive scan of sizes)
    uint32_t lo = 0, hi = n_nodes - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (voff[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const uint32_t node = lo;
    const uint32_t x = (uint32_t)(t - voff[node]);
    const uint64_t key = p.rep_key[first[node]];
    const int c = key_cls(p, key);
    const ClassDev cl = p.cls[c];
    const ProgDev pg = p.progs[p.class_prog[c]];
    const uint32_t* ss = p.stage + pg.stage_base;
    const uint2 rec = p.cellrec[pg.cell_base + ss[j - 1] + x];
    const int i = rec.x >> 16, m = rec.x & 0xffff;
    const uint16_t* q = p.preds + pg.pred_base + rec.y;
    const double* Pf = p.prefix + (size_t)cl.pair * LP;
    const double dm = p.domain[(size_t)cl.pair * p.nv_stride + m];
    const double Pi = Pf[i];
    const double g1 = (double)(cl.gas - 1);
    const double* E = p.qtab + ((size_t)c * p.n_codes + key_code(p, key, j - 2)) * L;
    // the parent's stage-(j-1) values: the class's stage-1 table, or the
    // depth-(j-2) node this node extends
    const double* Vp;
    if (j == 2) {
      Vp = p.v1g + p.v1off[c];
    } else {
      const uint32_t pn = p.nid[(size_t)(d - 1) * p.stride + first[node]] - 1;
      Vp = Vprev + p.voff[(size_t)(d - 1) * (p.stride + 1) + pn];
    }
    double best = CUDART_INF;
    int bc = -1;
    for (int cut = j - 1; cut < i; ++cut) {  // pipeline_dp.cpp:114-131
      const double t2 = Pi - Pf[cut];
      const double term = t2 > dm ? g1 * (t2 - dm) : 0.0;
      const double g = ((Vp[q[cut - (j - 1)]] + term) + t2) + E[cut];
      if (g < best) {
        best = g;
        bc = cut;
      }
    }
    Vcur[voff[node] + x] = best;
    bpj[voff[node] + x] = (uint8_t)bc;
    mine += (unsigned long long)(i - (j - 1));
  }
  if (exec) {  // executed inner iterations (roofline accounting)
    atomicAdd(&cnt, mine);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(exec, cnt);
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
    uint8_t* co = p.cutsb + (uint64_t)p.rep_list[r] * (p.max_pp + 1);
    co[k] = (uint8_t)L;
    uint32_t x = ss[k - 1];  // N_k = {(L, 0)}
    for (int j = k; j >= 2; --j) {
      const int d = j - 1;
      const uint32_t node = p.nid[(size_t)d * p.stride + r] - 1;
      const uint64_t off = p.voff[(size_t)d * (p.stride + 1) + node];
      const int cut = p.bp[p.bbase[j] + off + (x - ss[j - 1])];
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
