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
// one-DP-per-candidate kernel and the oracle).
//
// Three kernels per chunk, every count on the device (no host round trip):
//   K_trie_build_sorted (cooperative, grid barriers between phases): the
//     chunk's distinct signature keys radix-sorted; in key order a signature
//     starts a node at every depth past its common prefix with the previous
//     key, so the depth-d node ids (lexicographic, class-contiguous, the
//     children of a parent adjacent) are prefix counts of those starts; the
//     node arrays, each class's node range per depth, the level plans (tiles,
//     value / argmin table bases by device bump allocation; exceeding a
//     capacity raises `ovf` and the signature-mode K_dp, amp_dp_multi.cuh,
//     solves the chunk instead) and the tile descriptors.  K_trie_build, the
//     level-by-level build of the same trie (a scan of child marks per
//     depth), is the comparison path (AMP_TRIE_LEVELS=1).
//   K_trie_dp (persistent, dataflow): CTAs take tiles in depth order from an
//     atomic counter (the next one while the current one is solved).  A tile
//     = (class, run of tn consecutive depth-d nodes, chunk of the cells of
//     N_{d+1}); it waits until the runs holding its parents are done, stages
//     their stage-d tables and the edge rows in shared memory, solves its
//     items, publishes its run.  The upper levels (few nodes, latency-bound)
//     thereby overlap the wide middle levels.
//   K_trie_back: one thread per signature backtracks (pipeline_dp.cpp:
//     134-148) along its trie path and writes its cuts.
#pragma once

#include "amp_common.cuh"
#include "amp_dp_sparse.cuh"

namespace amp {

constexpr int kTrieMaxD1 = 64;        // depths 0 .. nq (keys are <= 63 bits, >= 1 bit per code)
constexpr int kTrieMaxCls = 1024;     // classes of a trie context (plan arrays in smem)
#ifndef AMP_TRIE_MINB
#define AMP_TRIE_MINB 4       // K_trie_dp CTAs per SM
#define AMP_TRIE_SMEM_KB 46   // K_trie_dp smem per CTA
#endif
#ifndef AMP_TRIE_THREADS
#define AMP_TRIE_THREADS 256  // K_trie_dp block
#endif
constexpr int kTrieThreads = AMP_TRIE_THREADS;
constexpr int kTrieNB = 4;            // nodes per thread in wide stages (share the cell's work)
constexpr int kTrieSmem = AMP_TRIE_SMEM_KB * 1024;  // K_trie_dp smem per CTA
constexpr int kBuildThreads = 512;    // K_trie_build block
constexpr int kBuildReg = 4;          // signatures per thread K_trie_build keeps in registers

// Level state, in device memory (zeroed by the host before K_trie_build).
struct TrieState {
  uint32_t cnt[kTrieMaxD1];         // nodes per depth (depth 0: the heavy classes)
  uint64_t node_off[kTrieMaxD1];    // start of depth d's nodes in the node arrays
  uint32_t tile_off[kTrieMaxD1 + 1];  // first tile of depth d; [nq + 1]: all tiles
  unsigned long long v_bump, bp_bump, run_bump, tile_bump;
  uint32_t ovf;                     // capacity exceeded: signature-mode K_dp instead
  uint32_t next_tile;               // K_trie_dp dispenser
  uint32_t bar_count, bar_pad;      // K_trie_build grid barrier (arrivals)
  unsigned long long dtot[kTrieMaxD1][4];  // per-depth plan totals: tiles, values, argmins, runs
};

// Per (class, stage j) facts of the class's pruned program and its tile
// shape (host-built).
struct TrieStage {
  uint32_t cell0;   // first cell of N_j in cellrec (absolute)
  uint32_t n;       // |N_j|
  uint32_t iters;   // (cell, cut) pairs of stage j (unpadded)
  uint32_t tn;      // nodes per tile
  uint32_t wide;    // 1: groups of 4 nodes, per-node smem columns; 0: node per thread
};

// Value-table row stride (doubles) of a stage of n cells: whole 128-byte
// lines, so no L1 line spans two nodes' rows — a row is read (through L1,
// by cp.async) only after the run that wrote it is published, and no SM can
// hold a stale copy of it from an earlier read of a neighbouring row.
__host__ __device__ inline uint32_t vrow(uint32_t n) { return (n + 15u) & ~15u; }

__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// One K_trie_dp work item, with everything its prologue needs resolved by
// the build (one 64-byte load instead of a chain of dependent lookups).
struct alignas(16) TrieTile {
  uint32_t node;    // absolute index of the first node (node_off[d] + local id)
  uint32_t pub;     // done[] counter of the tile's node run
  uint16_t c;       // class
  uint8_t d, leaf;  // depth; 1: leaf depth (argmins only)
  uint16_t nn, x0, x1, pad;  // nodes, cell range [x0, x1) of N_{d+1}
  uint32_t pfirst, pn;  // parents: first (local id at depth d - 1), count
  uint32_t w0, w1;      // done[] counters of the parents' runs [w0, w1]
  uint32_t need;        // cell chunks per parent run
  int64_t vpar;         // value arena: row of parent P at vpar + P * vrow(N_d)
  uint64_t vout;        // value arena: the tile's first row
  uint64_t bout;        // argmin arena: the tile's first row
};

struct TrieParams {
  // signatures: the distinct keys of the chunk's hash table
  const unsigned long long* n_sig;  // device count
  uint32_t* uniq;                   // [n_sig] slots (the sorted build rewrites it: slot of signature i)
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
  uint8_t* pres;                    // child marks [cnt[d-1] * U] (kept clear between uses)
  uint32_t* cid;                    // their scan: child node id
  uint64_t pres_cap;
  uint32_t* partial;                // [gridDim of K_trie_build]
  uint32_t* npar;                   // node arrays (absolute index node_off[d] + id)
  uint16_t* ncls;
  uint8_t* ncode;
  uint64_t node_cap;
  // level plans [kTrieMaxD1][n_cls]
  uint32_t* nb;                     // first node of the class at depth d
  uint32_t* nK;                     // its node count
  uint32_t* nxc;                    // cell chunks per node run
  uint32_t* tbase;                  // [kTrieMaxD1][n_cls + 1] first tile (within the depth)
  uint64_t* vbase;                  // value table base (doubles, in varena)
  uint64_t* bbase;                  // argmin table base (bytes, in bparena)
  uint64_t* rbase;                  // first run counter
  const TrieStage* tstage;          // [n_cls][max_pp + 1]
  double* varena;
  uint64_t vcap;
  uint8_t* bparena;
  uint64_t bpcap;
  uint32_t* done;                   // per node run: finished cell chunks
  uint64_t run_cap;
  TrieTile* tiles;
  uint64_t tile_cap;
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
  // k_trie_build_sorted: radix-sort ping-pong buffers [n], per-CTA digit
  // histograms [grid][256] and per-depth start counts [grid][64]
  uint64_t* sk[2];
  uint32_t* sv[2];
  uint32_t* ghist;
  uint32_t* gpart;
  int32_t kbits, smem_bytes;        // significant key bits (class + codes); K_trie_dp dynamic smem
};

__device__ __forceinline__ int trie_cls(const TrieParams& p, uint64_t k) { return (int)(k >> (p.nq * p.cb)); }
__device__ __forceinline__ int trie_code(const TrieParams& p, uint64_t k, int q) {
  return (int)((k >> ((p.nq - 1 - q) * p.cb)) & (uint64_t)(p.U - 1));
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// Grid barrier of the cooperative K_trie_build (all CTAs co-resident): one
// monotonic arrival counter (zeroed per launch); CTA thread 0 adds its
// arrival with release semantics and polls until all CTAs of this phase
// arrived.
__device__ __forceinline__ void grid_barrier(TrieState* st, uint32_t& phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t target = ++phase * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&st->bar_count) : "memory");
    while (ld_acquire(&st->bar_count) < target) {
    }
    __threadfence();
  }
  __syncthreads();
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

// Exclusive prefix of n values in smem (in place) by one warp; returns the
// total (valid in that warp).
__device__ __forceinline__ unsigned long long warp_exscan(unsigned long long* a, int n) {
  const int l = threadIdx.x & 31;
  unsigned long long carry = 0;
  for (int b = 0; b < n; b += 32) {
    const unsigned long long v = b + l < n ? a[b + l] : 0;
    unsigned long long incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (l >= o) incl += y;
    }
    if (b + l < n) a[b + l] = carry + incl - v;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  return carry;
}

// CTA 0 of K_trie_build: the plan of depth d (all nodes of depth d written).
__device__ void plan_level(const TrieParams& p, int d, uint32_t total, uint64_t noff,
                           unsigned long long* sm4) {
  __shared__ unsigned long long s_tot[4];
  const int NC = p.n_cls, tid = threadIdx.x;
  unsigned long long* s_tiles = sm4;
  unsigned long long* s_v = sm4 + NC;
  unsigned long long* s_b = sm4 + 2 * NC;
  unsigned long long* s_r = sm4 + 3 * NC;
  const uint16_t* cl = p.ncls + noff;
  uint32_t* nb = p.nb + (size_t)d * NC;
  uint32_t* nK = p.nK + (size_t)d * NC;
  uint32_t* nx = p.nxc + (size_t)d * NC;
  (void)cl;
  (void)total;
  for (int c = tid; c < NC; c += blockDim.x) {
    // the scan left [first node, end) of the class at depth d in nb / nK
    // (both zero for a class without nodes)
    const uint32_t lo = __ldcg(nb + c), K = __ldcg(nK + c) - lo;
    nK[c] = K;
    uint32_t runs = 0, chunks = 1;
    unsigned long long vs = 0, bs = 0;
    if (K) {
      const TrieStage ts = p.tstage[(size_t)c * (p.max_pp + 1) + d + 1];
      runs = (K + ts.tn - 1) / ts.tn;
      // few node runs (the upper levels): cut the cells into chunks (>= 32
      // cells) so the level still spreads over the GPU
      if (ts.wide && runs < 64) chunks = min((64 + runs - 1) / runs, (ts.n + 31) / 32);
      if (d < p.cls[c].pp - 1) vs = (unsigned long long)K * vrow(ts.n);  // leaves keep argmins only
      bs = (unsigned long long)K * ts.n;
    }
    nx[c] = chunks;
    s_tiles[NC - 1 - c] = (unsigned long long)runs * chunks;  // (dispense order: last class first)
    s_v[c] = vs;
    s_b[c] = bs;
    s_r[c] = runs;
  }
  __syncthreads();
  const int w = tid >> 5;
  if (w < 4) {
    const unsigned long long t = warp_exscan(sm4 + (size_t)w * NC, NC);
    if ((tid & 31) == 0) s_tot[w] = t;
  }
  __syncthreads();
  TrieState* st = p.st;
  uint32_t* tb = p.tbase + (size_t)d * (NC + 1);
  uint64_t* vb = p.vbase + (size_t)d * NC;
  uint64_t* bb = p.bbase + (size_t)d * NC;
  uint64_t* rb = p.rbase + (size_t)d * NC;
  for (int c = tid; c < NC; c += blockDim.x) {
    tb[c] = (uint32_t)s_tiles[c];
    vb[c] = st->v_bump + s_v[c];
    bb[c] = st->bp_bump + s_b[c];
    rb[c] = st->run_bump + s_r[c];
  }
  __syncthreads();
  if (tid == 0) {
    tb[NC] = (uint32_t)s_tot[0];
    st->cnt[d] = total;
    st->node_off[d] = noff;
    st->tile_off[d] = (uint32_t)st->tile_bump;
    st->tile_bump += s_tot[0];
    st->v_bump += s_tot[1];
    st->bp_bump += s_tot[2];
    st->run_bump += s_tot[3];
    if (st->v_bump > p.vcap || st->bp_bump > p.bpcap || st->run_bump > p.run_cap ||
        st->tile_bump > p.tile_cap)
      st->ovf = 1;
  }
  __syncthreads();
}

// The tile list of all depths (after the level plans); run counters cleared.
__device__ void build_tile_list(const TrieParams& p, uint64_t gtid, uint64_t gstride) {
  TrieState* st = p.st;
  const uint32_t T = (uint32_t)st->tile_bump;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->tile_off[p.nq + 1] = T;
    st->next_tile = 0;
  }
  for (uint64_t r = gtid; r < st->run_bump; r += gstride) p.done[r] = 0;
  for (uint64_t t = gtid; t < T; t += gstride) {
    int d = 1;
    while (d < p.nq && st->tile_off[d + 1] <= t) ++d;
    const uint32_t tt = (uint32_t)t - st->tile_off[d];
    const uint32_t* tb = p.tbase + (size_t)d * (p.n_cls + 1);
    // within a depth the classes are dealt last class first (the plan()
    // list ends with the deepest pipelines, whose chain of levels is the
    // launch's critical path): tbase is by dispense position
    int lo = 0, hi = p.n_cls - 1;  // last position with tbase <= tt
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tb[mid] <= tt) lo = mid;
      else hi = mid - 1;
    }
    const int c = p.n_cls - 1 - lo;
    const TrieStage ts = p.tstage[(size_t)c * (p.max_pp + 1) + d + 1];
    const uint32_t chunks = p.nxc[(size_t)d * p.n_cls + c];
    const uint32_t lt = tt - tb[lo], run = lt / chunks, cc = lt - run * chunks;
    const uint32_t nbc = p.nb[(size_t)d * p.n_cls + c], K = p.nK[(size_t)d * p.n_cls + c];
    TrieTile tl;
    const uint32_t n0 = nbc + run * ts.tn;
    const uint64_t noff = st->node_off[d];
    const int NC = p.n_cls;
    tl.node = (uint32_t)(noff + n0);
    tl.pub = (uint32_t)(p.rbase[(size_t)d * NC + c] + run);
    tl.c = (uint16_t)c;
    tl.d = (uint8_t)d;
    tl.leaf = d == p.cls[c].pp - 1;
    tl.nn = (uint16_t)min(ts.tn, nbc + K - n0);
    const uint32_t xc = (ts.n + chunks - 1) / chunks;
    tl.x0 = (uint16_t)(cc * xc);
    tl.x1 = (uint16_t)min(ts.n, (cc + 1) * xc);
    tl.pad = 0;
    tl.vout = tl.leaf ? 0 : p.vbase[(size_t)d * NC + c] + (uint64_t)(n0 - nbc) * vrow(ts.n);
    tl.bout = p.bbase[(size_t)d * NC + c] + (uint64_t)(n0 - nbc) * ts.n;
    tl.pfirst = tl.pn = tl.w0 = tl.w1 = tl.need = 0;
    tl.vpar = 0;
    if (d >= 2) {  // (depth 1: the class's stage-1 table)
      const TrieStage tp = p.tstage[(size_t)c * (p.max_pp + 1) + d];
      const uint32_t pfirst = p.npar[noff + n0], plast = p.npar[noff + n0 + tl.nn - 1];
      const uint32_t pnb = p.nb[(size_t)(d - 1) * NC + c];
      const uint64_t rb = p.rbase[(size_t)(d - 1) * NC + c];
      tl.pfirst = pfirst;
      tl.pn = plast - pfirst + 1;
      tl.w0 = (uint32_t)(rb + (pfirst - pnb) / tp.tn);
      tl.w1 = (uint32_t)(rb + (plast - pnb) / tp.tn);
      tl.need = p.nxc[(size_t)(d - 1) * NC + c];
      tl.vpar = (int64_t)p.vbase[(size_t)(d - 1) * NC + c] - (int64_t)pnb * (int64_t)vrow(tp.n);
    }
    AMP_CHECK(t < p.tile_cap && tl.pub < p.run_cap && (d < 2 || tl.w1 < p.run_cap), "tile / run counters");
    AMP_CHECK(tl.bout + (uint64_t)tl.nn * ts.n <= p.bpcap, "tile argmin rows");
    AMP_CHECK(tl.leaf || tl.vout + (uint64_t)tl.nn * vrow(ts.n) <= p.vcap, "tile value rows");
    AMP_CHECK(tl.node + tl.nn <= p.node_cap, "tile nodes");
    p.tiles[t] = tl;
  }
}

// The trie of the chunk's signatures and the tile list of its DP, level by
// level (the comparison path, AMP_TRIE_LEVELS=1; the default is
// k_trie_build_sorted below).
__global__ void __launch_bounds__(kBuildThreads) k_trie_build(TrieParams p) {
  extern __shared__ unsigned long long build_sm[];  // [4][n_cls] (CTA 0's plans)
  __shared__ uint32_t sm[32], wsum[32];
  TrieState* st = p.st;
  const int tid = threadIdx.x, l = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + tid, gstride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n = *p.n_sig;
  uint32_t phase = 0;  // grid barriers passed
  // ---- signature list, roots, depth-1 marks --------------------------------
  // (a thread's first kBuildReg signatures keep key, depth and node in
  // registers over the levels; the rest go through sig_key / nid)
  uint64_t rkey[kBuildReg];
  uint32_t rnid[kBuildReg];
  int rdep[kBuildReg];
  for (uint64_t i = gtid, r = 0; i < n; i += gstride, ++r) {
    const uint32_t s = p.uniq[i];
    const unsigned long long k = p.tkey[s];
    const uint64_t key = p.key_shift >= 64 ? k : (k & ((1ull << p.key_shift) - 1));
    p.sig_key[i] = key;
    p.rep_item[i] = p.tval[s];
    p.tval[s] = (uint32_t)i;
    const int c = trie_cls(p, key);
    const int rt = p.root_rank[c];
    const int dep = p.cls[c].pp - 1;  // depth of the signature's leaf
    p.nid[i] = (uint32_t)rt;
    if (dep >= 1) p.pres[(uint64_t)rt * p.U + trie_code(p, key, 0)] = 1;
#pragma unroll
    for (int q = 0; q < kBuildReg; ++q)
      if (r == q) {
        rkey[q] = key;
        rnid[q] = (uint32_t)rt;
        rdep[q] = dep;
      }
  }
#pragma unroll
  for (int q = 0; q < kBuildReg; ++q)
    if (gtid + q * gstride >= n) rdep[q] = -1;
  grid_barrier(st, phase);
  uint32_t cnt_prev = (uint32_t)p.n_roots;       // nodes of depth d-1
  uint64_t off_prev = 0, noff = 0;               // node_off of depth d-1, d
  uint64_t marked = (uint64_t)p.n_roots * p.U;   // mark entries that may be set
  bool ovf = false;  // (every CTA takes the same decisions: the same inputs)
  for (int d = 1; d <= p.nq; ++d) {
    const uint64_t ne = marked;
    noff = d == 1 ? 0 : off_prev + cnt_prev;
    if (noff + ne > p.node_cap) {
      ovf = true;
      break;
    }
    // ---- scan of the marks: per-CTA sums -----------------------------------
    const uint64_t per = (ne + gridDim.x - 1) / gridDim.x;
    const uint64_t b = (uint64_t)blockIdx.x * per, e = b + per < ne ? b + per : ne;
    uint32_t s = 0;
    for (uint64_t x = b + tid; x < e; x += blockDim.x) s += __ldcg(p.pres + x);
    s = block_sum_u32(s, sm);
    if (tid == 0) p.partial[blockIdx.x] = s;
    grid_barrier(st, phase);
    // ---- node ids: exclusive scan, node arrays, clear the marks ------------
    uint32_t base = 0, total = 0;
    {
      uint32_t a = 0, t = 0;
      for (int x = tid; x < (int)gridDim.x; x += blockDim.x) {
        const uint32_t v = __ldcg(p.partial + x);
        t += v;
        if (x < (int)blockIdx.x) a += v;
      }
      base = block_sum_u32(a, sm);
      total = block_sum_u32(t, sm);
    }
    for (uint64_t x0 = b; x0 < e; x0 += blockDim.x) {
      const uint64_t x = x0 + tid;
      const uint32_t f = x < e ? __ldcg(p.pres + x) : 0;
      const unsigned bal = __ballot_sync(0xffffffffu, f != 0);
      __syncthreads();
      if (l == 0) wsum[w] = __popc(bal);
      __syncthreads();
      uint32_t before = base;
      for (int q = 0; q < w; ++q) before += wsum[q];
      before += __popc(bal & ((1u << l) - 1));
      if (x < e) {  // class node ranges at depth d: the prefix at a class's first / after its last parent
        const uint64_t par = x / (uint64_t)p.U;
        const uint32_t rem = (uint32_t)(x - par * p.U);
        if (rem == 0 || rem == (uint32_t)p.U - 1) {
          int c, cprev = -1, cnext = -1;
          if (d == 1) {
            c = p.root_cls[par];
          } else {
            const uint16_t* pc = p.ncls + off_prev;
            c = __ldcg(pc + par);
            if (rem == 0 && par > 0) cprev = __ldcg(pc + par - 1);
            if (rem != 0 && par + 1 < cnt_prev) cnext = __ldcg(pc + par + 1);
          }
          if (rem == 0 && cprev != c) p.nb[(size_t)d * p.n_cls + c] = before;
          if (rem == (uint32_t)p.U - 1 && cnext != c) p.nK[(size_t)d * p.n_cls + c] = before + f;
        }
      }
      if (f) {
        const uint64_t par = x / (uint64_t)p.U;
        p.npar[noff + before] = (uint32_t)par;
        p.ncode[noff + before] = (uint8_t)(x % (uint64_t)p.U);
        p.ncls[noff + before] = (uint16_t)(d == 1 ? p.root_cls[par] : __ldcg(p.ncls + off_prev + par));
        p.cid[x] = before;
        p.pres[x] = 0;
      }
      for (int q = 0; q < nw; ++q) base += wsum[q];
    }
    grid_barrier(st, phase);
    marked = 0;
    if (d < p.nq && (uint64_t)total * p.U > p.pres_cap) {
      ovf = true;
      break;
    }
    // ---- plan of depth d (CTA 0); each signature's node, depth-(d+1) marks
    if (blockIdx.x == 0) plan_level(p, d, total, noff, build_sm);
#pragma unroll
    for (int q = 0; q < kBuildReg; ++q) {
      if (rdep[q] < d) continue;
      const uint32_t node = __ldcg(p.cid + (uint64_t)rnid[q] * p.U + trie_code(p, rkey[q], d - 1));
      rnid[q] = node;
      if (rdep[q] >= d + 1) p.pres[(uint64_t)node * p.U + trie_code(p, rkey[q], d)] = 1;
    }
    for (uint64_t i = gtid + kBuildReg * gstride; i < n; i += gstride) {
      const uint64_t key = p.sig_key[i];
      const int pp = p.cls[trie_cls(p, key)].pp;
      if (pp - 1 < d) continue;
      const uint32_t node = __ldcg(p.cid + (uint64_t)p.nid[i] * p.U + trie_code(p, key, d - 1));
      p.nid[i] = node;
      if (pp - 1 >= d + 1) p.pres[(uint64_t)node * p.U + trie_code(p, key, d)] = 1;
    }
    if (d < p.nq) marked = (uint64_t)total * p.U;
    grid_barrier(st, phase);
    if (ld_acquire(&st->ovf) != 0) {  // a plan capacity was exceeded
      ovf = true;
      break;
    }
    off_prev = noff;
    cnt_prev = total;
  }
  if (ovf) {  // clear the marks left behind; the signature-mode K_dp takes over
    for (uint64_t x = gtid; x < marked; x += gstride) p.pres[x] = 0;
    if (blockIdx.x == 0 && tid == 0) st->ovf = 1;
    return;
  }
#pragma unroll
  for (int q = 0; q < kBuildReg; ++q)
    if (rdep[q] >= 0) p.nid[gtid + q * gstride] = rnid[q];
  build_tile_list(p, gtid, gstride);
}

// k_trie_build_sorted, the plan of depth d relative to the depth's own
// bases (the depths are planned in parallel, one CTA each): per class the
// node runs, cell chunks, tiles and table sizes; the per-depth totals go to
// st->dtot[d].
__device__ void plan_depth(const TrieParams& p, int d, unsigned long long* sm4) {
  const int NC = p.n_cls, tid = threadIdx.x;
  unsigned long long* s_tiles = sm4;
  unsigned long long* s_v = sm4 + NC;
  unsigned long long* s_b = sm4 + 2 * NC;
  unsigned long long* s_r = sm4 + 3 * NC;
  uint32_t* nb = p.nb + (size_t)d * NC;
  uint32_t* nK = p.nK + (size_t)d * NC;
  uint32_t* nx = p.nxc + (size_t)d * NC;
  for (int c = tid; c < NC; c += blockDim.x) {
    const uint32_t lo = __ldcg(nb + c), K = __ldcg(nK + c) - lo;  // [first node, end) -> count
    nK[c] = K;
    uint32_t runs = 0, chunks = 1;
    unsigned long long vs = 0, bs = 0;
    if (K) {
      const TrieStage ts = p.tstage[(size_t)c * (p.max_pp + 1) + d + 1];
      runs = (K + ts.tn - 1) / ts.tn;
      if (ts.wide && runs < 64) chunks = min((64 + runs - 1) / runs, (ts.n + 31) / 32);
      if (d < p.cls[c].pp - 1) vs = (unsigned long long)K * vrow(ts.n);  // leaves keep argmins only
      bs = (unsigned long long)K * ts.n;
    }
    nx[c] = chunks;
    s_tiles[NC - 1 - c] = (unsigned long long)runs * chunks;  // (dispense order: last class first)
    s_v[c] = vs;
    s_b[c] = bs;
    s_r[c] = runs;
  }
  __syncthreads();
  const int w = tid >> 5;
  if (w < 4) {
    const unsigned long long t = warp_exscan(sm4 + (size_t)w * NC, NC);
    if ((tid & 31) == 0) p.st->dtot[d][w] = t;
  }
  __syncthreads();
  uint32_t* tb = p.tbase + (size_t)d * (NC + 1);
  uint64_t* vb = p.vbase + (size_t)d * NC;
  uint64_t* bb = p.bbase + (size_t)d * NC;
  uint64_t* rb = p.rbase + (size_t)d * NC;
  for (int c = tid; c < NC; c += blockDim.x) {
    tb[c] = (uint32_t)s_tiles[c];
    vb[c] = s_v[c];
    bb[c] = s_b[c];
    rb[c] = s_r[c];
  }
  if (tid == 0) tb[NC] = (uint32_t)p.st->dtot[d][0];
  __syncthreads();
}

// The trie of the chunk's signatures from their sorted keys (one pass for
// all depths) and the tile list of its DP.  Node ids are those of the level
// build (k_trie_build): the depth-d nodes are the distinct (class, c_0 ..
// c_{d-1}) prefixes in lexicographic order, so in key order a signature
// starts a new node at every depth past the length of its common prefix
// with the previous signature (a different class: every depth), and its
// depth-d node is the count of such starts so far, minus one.
//   1. LSD radix sort of the signature keys (8-bit digits; per pass a digit
//      histogram per CTA, one grid barrier, the scatter ranked stably by
//      warp match + per-warp counts in smem, one grid barrier);
//   2. per-CTA start counts per depth, one grid barrier, then in key order:
//      node ids by ballot prefixes per depth, the node arrays, the class
//      node ranges, each signature's leaf node, the slot -> signature map;
//   3. the level plans (one CTA per depth, in parallel), their offsets
//      across depths, the tile list.
__global__ void __launch_bounds__(kBuildThreads) k_trie_build_sorted(TrieParams p) {
  extern __shared__ unsigned long long build_sm[];  // [4][n_cls] (plans)
  constexpr int NW = kBuildThreads / 32;
  __shared__ uint32_t s_hist[256], s_base[256];
  __shared__ uint16_t s_wc[NW][256];
  __shared__ uint32_t s_wd[NW][kTrieMaxD1];  // per-warp start counts, then their exclusive prefix
  __shared__ uint32_t s_run[kTrieMaxD1];     // starts before the current chunk (per depth)
  __shared__ uint64_t s_noff[kTrieMaxD1 + 1];
  __shared__ int s_ovf;
  TrieState* st = p.st;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, G = gridDim.x, bid = blockIdx.x;
  const uint64_t gtid = (uint64_t)bid * blockDim.x + tid, gstride = (uint64_t)G * blockDim.x;
  const uint64_t n = *p.n_sig;
  const int nq = p.nq, cb = p.cb;
  const uint64_t TS = (n + G - 1) / G, b0 = min((uint64_t)bid * TS, n), b1 = min(b0 + TS, n);
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t phase = 0;
  // ---- keys of the chunk's distinct signatures ------------------------------
  for (uint64_t i = gtid; i < n; i += gstride) {
    const uint32_t sl = p.uniq[i];
    const unsigned long long k = p.tkey[sl];
    p.sk[0][i] = p.key_shift >= 64 ? k : (k & ((1ull << p.key_shift) - 1));
    p.sv[0][i] = sl;
  }
  grid_barrier(st, phase);
  // ---- 1. LSD radix sort, 8-bit digits ---------------------------------------
  int cur = 0;
  for (int sh = 0; sh < p.kbits; sh += 8, cur ^= 1) {
    const uint64_t* sk = p.sk[cur];
    const uint32_t* sv = p.sv[cur];
    for (int x = tid; x < 256; x += blockDim.x) s_hist[x] = 0;
    __syncthreads();
    for (uint64_t i = b0 + tid; i < b1; i += blockDim.x) atomicAdd(&s_hist[(sk[i] >> sh) & 255], 1u);
    __syncthreads();
    for (int x = tid; x < 256; x += blockDim.x) p.ghist[(size_t)bid * 256 + x] = s_hist[x];
    grid_barrier(st, phase);
    // this CTA's first position of every digit: all CTAs' counts of smaller
    // digits plus the earlier CTAs' counts of the digit
    {  // (thread = digit, the two halves of the block over the two halves of the CTAs)
      const int dg = tid & 255, half = tid >> 8, bh = (G + 1) >> 1;
      const int bb0 = half ? bh : 0, bb1 = half ? G : bh;
      uint32_t tot = 0, pre = 0;
#pragma unroll 8
      for (int b = bb0; b < bb1; ++b) {
        const uint32_t v = __ldcg(p.ghist + (size_t)b * 256 + dg);
        tot += v;
        pre += b < bid ? v : 0u;
      }
      if (half) {
        // (s_wc as u32 scratch for the upper half's sums; cleared before the scatter)
        reinterpret_cast<uint32_t*>(&s_wc[0][0])[dg] = tot;
        reinterpret_cast<uint32_t*>(&s_wc[0][0])[256 + dg] = pre;
      }
      __syncthreads();
      if (!half) {
        s_hist[dg] = tot + reinterpret_cast<uint32_t*>(&s_wc[0][0])[dg];
        s_base[dg] = pre + reinterpret_cast<uint32_t*>(&s_wc[0][0])[256 + dg];
      }
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the digit totals
      uint32_t carry = 0;
      for (int b = 0; b < 256; b += 32) {
        const uint32_t v = s_hist[b + lane];
        uint32_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        s_base[b + lane] += carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    // stable scatter, blockDim items at a time in order
    uint64_t* dk = p.sk[cur ^ 1];
    uint32_t* dv = p.sv[cur ^ 1];
    for (uint64_t c0 = b0; c0 < b1; c0 += blockDim.x) {
      for (int x = tid; x < NW * 256; x += blockDim.x) (&s_wc[0][0])[x] = 0;
      __syncthreads();
      const uint64_t i = c0 + tid;
      const bool live = i < b1;
      uint64_t key = 0;
      uint32_t val = 0;
      int dig = 256;  // (dead lanes: a digit no live lane has)
      if (live) {
        key = sk[i];
        val = sv[i];
        dig = (int)((key >> sh) & 255);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, dig);
      const int rank = __popc(peers & lt_mask);
      if (live && rank == 0) s_wc[w][dig] = (uint16_t)__popc(peers);
      __syncthreads();
      if (live) {
        uint32_t pos = s_base[dig] + rank;
        for (int q = 0; q < w; ++q) pos += s_wc[q][dig];
        AMP_CHECK(pos < n, "radix scatter");
        dk[pos] = key;
        dv[pos] = val;
      }
      __syncthreads();
      if (tid < 256) {
        uint32_t t = 0;
        for (int q = 0; q < NW; ++q) t += s_wc[q][tid];
        s_base[tid] += t;
      }
      __syncthreads();
    }
    grid_barrier(st, phase);
  }
  const uint64_t* K = p.sk[cur];
  const uint32_t* V = p.sv[cur];
  const int cshift = nq * cb;
  const uint64_t cmask = cshift >= 64 ? ~0ull : ((1ull << cshift) - 1);
  // common-prefix length (codes) with the previous key; 0 at a class change
  auto lcp_of = [&](uint64_t i, uint64_t key) -> int {
    if (i == 0) return 0;
    const uint64_t prev = K[i - 1];
    if ((prev >> cshift) != (key >> cshift)) return 0;
    const uint64_t x = (prev ^ key) & cmask;  // != 0: keys are distinct
    return (__clzll((long long)x) - (64 - cshift)) / cb;
  };
  // ---- the signature list in key order (also for the capacity fallback) ---
  for (uint64_t i = b0 + tid; i < b1; i += blockDim.x) {
    const uint32_t sl = V[i];
    p.uniq[i] = sl;  // (signature -> slot, read by k_run_pipe)
    p.sig_key[i] = K[i];
    p.rep_item[i] = p.tval[sl];
    p.tval[sl] = (uint32_t)i;
  }
  // ---- 2. node starts per depth: per-CTA counts ------------------------------
  for (int x = tid; x < kTrieMaxD1; x += blockDim.x) s_run[x] = 0;
  __syncthreads();
  for (uint64_t i = b0 + tid; i < b1; i += blockDim.x) {
    const uint64_t key = K[i];
    const int dep = p.cls[key >> cshift].pp - 1;
    for (int d = lcp_of(i, key) + 1; d <= dep; ++d) atomicAdd(&s_run[d], 1u);
  }
  __syncthreads();
  for (int x = tid; x < kTrieMaxD1; x += blockDim.x) p.gpart[(size_t)bid * kTrieMaxD1 + x] = s_run[x];
  grid_barrier(st, phase);
  if (tid < kTrieMaxD1) {
    uint32_t tot = 0, pre = 0;
    for (int b = 0; b < G; ++b) {
      const uint32_t v = __ldcg(p.gpart + (size_t)b * kTrieMaxD1 + tid);
      tot += v;
      if (b < bid) pre += v;
    }
    s_run[tid] = pre;
    s_wd[0][tid] = tot;  // (depth totals, consumed below)
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t off = 0;
    for (int d = 1; d <= nq; ++d) {
      s_noff[d] = off;
      off += s_wd[0][d];
    }
    s_noff[nq + 1] = off;
    s_ovf = off > p.node_cap;
    if (bid == 0) {
      for (int d = 1; d <= nq; ++d) {
        st->cnt[d] = s_wd[0][d];
        st->node_off[d] = s_noff[d];
      }
      if (s_ovf) st->ovf = 1;
    }
  }
  __syncthreads();
  if (s_ovf) return;  // (uniform: every CTA read the same totals)
  for (uint64_t c0 = b0; c0 < b1; c0 += blockDim.x) {
    const uint64_t i = c0 + tid;
    const bool live = i < b1;
    uint64_t key = 0;
    int lcp = 0, dep = -1, c = 0;
    if (live) {
      key = K[i];
      c = (int)(key >> cshift);
      dep = p.cls[c].pp - 1;
      lcp = lcp_of(i, key);
    }
    for (int d = 1; d <= nq; ++d) {  // per-warp start counts
      const unsigned b = __ballot_sync(0xffffffffu, live && d > lcp && d <= dep);
      if (lane == 0) s_wd[w][d] = __popc(b);
    }
    __syncthreads();
    if (tid >= 1 && tid <= nq) {  // exclusive prefix over the warps, per depth
      uint32_t a = 0;
      for (int q = 0; q < NW; ++q) {
        const uint32_t v = s_wd[q][tid];
        s_wd[q][tid] = a;
        a += v;
      }
      s_base[tid] = a;  // (this chunk's starts at depth tid)
    }
    __syncthreads();
    const bool first = live && (i == 0 || (K[i - 1] >> cshift) != (uint64_t)c);
    const bool last = live && (i + 1 == n || (K[i + 1] >> cshift) != (uint64_t)c);
    uint32_t par = live ? (uint32_t)p.root_rank[c] : 0u;
    for (int d = 1; d <= nq; ++d) {  // (uniform trip count: the ballots)
      const bool f = live && d > lcp && d <= dep;
      const unsigned b = __ballot_sync(0xffffffffu, f);
      if (live && d <= dep) {
        // inclusive count of the starts at depth d up to this signature
        const uint32_t node = s_run[d] + s_wd[w][d] + __popc(b & lt_mask) + (f ? 1u : 0u) - 1u;
        if (f) {  // this signature starts the node
          const uint64_t at = s_noff[d] + node;
          AMP_CHECK(at < p.node_cap, "node arrays");
          p.npar[at] = par;
          p.ncode[at] = (uint8_t)((key >> ((nq - d) * cb)) & (uint64_t)(p.U - 1));
          p.ncls[at] = (uint16_t)c;
        }
        if (first) p.nb[(size_t)d * p.n_cls + c] = node;
        if (last) p.nK[(size_t)d * p.n_cls + c] = node + 1;
        par = node;
      }
    }
    if (live) p.nid[i] = par;  // leaf node
    __syncthreads();
    if (tid >= 1 && tid <= nq) s_run[tid] += s_base[tid];
    __syncthreads();
  }
  grid_barrier(st, phase);
  // ---- 3. level plans (CTA d-1 plans depth d), offsets across depths ---------
  for (int d = bid + 1; d <= nq; d += G) plan_depth(p, d, build_sm);
  grid_barrier(st, phase);
  for (int d = bid + 1; d <= nq; d += G) {
    unsigned long long off[4] = {0, 0, 0, 0};
    for (int e = 1; e < d; ++e)
      for (int q = 0; q < 4; ++q) off[q] += __ldcg(&st->dtot[e][q]);
    const int NC = p.n_cls;
    uint64_t* vb = p.vbase + (size_t)d * NC;
    uint64_t* bb = p.bbase + (size_t)d * NC;
    uint64_t* rb = p.rbase + (size_t)d * NC;
    for (int c = tid; c < NC; c += blockDim.x) {
      vb[c] += off[1];
      bb[c] += off[2];
      rb[c] += off[3];
    }
    if (tid == 0) {
      st->tile_off[d] = (uint32_t)off[0];
      if (d == nq) {
        st->tile_bump = off[0] + __ldcg(&st->dtot[d][0]);
        st->v_bump = off[1] + __ldcg(&st->dtot[d][1]);
        st->bp_bump = off[2] + __ldcg(&st->dtot[d][2]);
        st->run_bump = off[3] + __ldcg(&st->dtot[d][3]);
        if (st->v_bump > p.vcap || st->bp_bump > p.bpcap || st->run_bump > p.run_cap ||
            st->tile_bump > p.tile_cap)
          st->ovf = 1;
      }
    }
  }
  grid_barrier(st, phase);
  if (ld_acquire(&st->ovf) != 0) return;
  build_tile_list(p, gtid, gstride);
}

// Wide stages (many cells): the (cell x, group g of 4 nodes) items of one
// tile.  sV holds, per predecessor cell x' of N_{j-1}, the parent value of
// every node of the tile (row x', column = node; SINGLE: the one parent's
// value), sE the edge cost of every node per cut (row cut - (j-1)); rows are
// TNst doubles (even: a group's 4 nodes are two 16-byte loads).  Per cut the
// predecessor index, t2 and the tolerance term are shared by the group's 4
// nodes; each node adds its parent value and its edge
// (pipeline_dp.cpp:118-127: same operands, same order, strict '<': the
// lowest cut wins ties).
template <bool SINGLE>
__device__ __forceinline__ void tile_wide(const TrieParams& p, const double* __restrict__ sV,
                                          const double* __restrict__ sE, const double* __restrict__ sPf,
                                          int TNst, int G, int x0, int x1, int Nj, int VS, int j, int nn,
                                          const TrieStage& ts, const uint16_t* __restrict__ pr,
                                          const double* __restrict__ dom, double g1, bool leaf,
                                          double* __restrict__ vout, uint8_t* __restrict__ bpo,
                                          unsigned long long& mine) {
  const int items = (x1 - x0) * G;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int xl = it / G, g = it - xl * G, x = x0 + xl;
    const uint2 rec = p.cellrec[ts.cell0 + x];
    const int i = rec.x >> 16, m = rec.x & 0xffff;
    const uint16_t* q = pr + rec.y - (j - 1);
    const double dm = dom[m];
    const double Pi = sPf[i];
    const double* vcol = sV + (SINGLE ? 0 : 4 * g);
    const double* ecol = sE + 4 * g - (j - 1) * TNst;
    mine += (unsigned long long)(i - (j - 1)) * (unsigned long long)min(4, nn - 4 * g);
    double b0 = CUDART_INF, b1 = CUDART_INF, b2 = CUDART_INF, b3 = CUDART_INF;
    int c0 = -1, c1 = -1, c2 = -1, c3 = -1;
#pragma unroll 2
    for (int cut = j - 1; cut < i; ++cut) {  // pipeline_dp.cpp:114-131
      const double t2 = Pi - sPf[cut];
      const double term = t2 > dm ? g1 * (t2 - dm) : 0.0;
      double v0, v1, v2, v3;
      if (SINGLE) {
        v0 = v1 = v2 = v3 = vcol[q[cut]];
      } else {
        const int qq = q[cut];
        const double2 va = *reinterpret_cast<const double2*>(vcol + qq * TNst);
        const double2 vb = *reinterpret_cast<const double2*>(vcol + qq * TNst + 2);
        v0 = va.x;
        v1 = va.y;
        v2 = vb.x;
        v3 = vb.y;
      }
      const double2 ea = *reinterpret_cast<const double2*>(ecol + cut * TNst);
      const double2 eb = *reinterpret_cast<const double2*>(ecol + cut * TNst + 2);
      const double h0 = ((v0 + term) + t2) + ea.x;
      const double h1 = ((v1 + term) + t2) + ea.y;
      const double h2 = ((v2 + term) + t2) + eb.x;
      const double h3 = ((v3 + term) + t2) + eb.y;
      if (h0 < b0) { b0 = h0; c0 = cut; }
      if (h1 < b1) { b1 = h1; c1 = cut; }
      if (h2 < b2) { b2 = h2; c2 = cut; }
      if (h3 < b3) { b3 = h3; c3 = cut; }
    }
    const double bs[4] = {b0, b1, b2, b3};
    const int cs[4] = {c0, c1, c2, c3};
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int ln = 4 * g + b;
      if (ln >= nn) break;
      AMP_CHECK(bpo + (uint64_t)ln * Nj + x < p.bparena + p.bpcap, "wide argmin");
      AMP_CHECK(leaf || vout + (uint64_t)ln * VS + x < p.varena + p.vcap, "wide value");
      if (!leaf) vout[(uint64_t)ln * VS + x] = bs[b];
      bpo[(uint64_t)ln * Nj + x] = (uint8_t)cs[b];
    }
  }
}

// Narrow stages (few cells, many nodes): one (cell x, node) item per
// thread.  sV holds the tile's parents' tables once each (row x', column =
// parent, odd stride), sE the class's edge rows per code (row code).
__device__ __forceinline__ void tile_narrow(const TrieParams& p, const double* __restrict__ sV,
                                            const double* __restrict__ sE, const double* __restrict__ sPf,
                                            const int* __restrict__ sNode, int Pst, int Nj, int VS, int j, int nn,
                                            const TrieStage& ts, const uint16_t* __restrict__ pr,
                                            const double* __restrict__ dom, double g1, bool leaf,
                                            double* __restrict__ vout, uint8_t* __restrict__ bpo,
                                            unsigned long long& mine) {
  const int L = p.L, items = Nj * nn;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int x = it / nn, ln = it - x * nn;
    const uint2 rec = p.cellrec[ts.cell0 + x];
    const int i = rec.x >> 16, m = rec.x & 0xffff;
    const uint16_t* q = pr + rec.y - (j - 1);
    const double dm = dom[m];
    const double Pi = sPf[i];
    const int nd = sNode[ln];
    const double* vcol = sV + (nd & 0xffff);
    const double* E = sE + (nd >> 16) * L;
    mine += (unsigned long long)(i - (j - 1));
    double best = CUDART_INF;
    int bc = -1;
#pragma unroll 2
    for (int cut = j - 1; cut < i; ++cut) {  // pipeline_dp.cpp:114-131
      const double t2 = Pi - sPf[cut];
      const double term = t2 > dm ? g1 * (t2 - dm) : 0.0;
      const double h = ((vcol[(int)q[cut] * Pst] + term) + t2) + E[cut];
      if (h < best) {
        best = h;
        bc = cut;
      }
    }
    AMP_CHECK(bpo + (uint64_t)ln * Nj + x < p.bparena + p.bpcap, "narrow argmin");
    AMP_CHECK(leaf || vout + (uint64_t)ln * VS + x < p.varena + p.vcap, "narrow value");
    if (!leaf) vout[(uint64_t)ln * VS + x] = best;
    bpo[(uint64_t)ln * Nj + x] = (uint8_t)bc;
  }
}

// All stages of the chunk's trie: persistent CTAs take tiles in depth order;
// a tile waits for the node runs holding its parents (their stage tables),
// stages them and the edge rows in shared memory, solves its items and
// publishes its run.  Parent tables are read through L2 (__ldcg): they were
// written by other SMs during this launch.
__global__ void __launch_bounds__(kTrieThreads, AMP_TRIE_MINB) k_trie_dp(TrieParams p) {
  extern __shared__ __align__(16) double smem_d[];
  __shared__ uint32_t s_t;
  if (p.st->ovf) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int L = p.L, LP = L + 1, P1 = p.max_pp + 1;
  const uint32_t T = p.st->tile_off[p.nq + 1];
  unsigned long long mine = 0;
  // the next tile is taken while this one is solved (its index is read at
  // the publish barrier); a CTA never waits on its own prefetched tile, and
  // every tile it waits on has a smaller index than its current one
  if (tid == 0) s_t = atomicAdd(&p.st->next_tile, 1u);
  __syncthreads();
  uint32_t t = s_t;
  for (;;) {
    if (t >= T) break;
    uint32_t tnext = 0;
    if (tid == 0) tnext = atomicAdd(&p.st->next_tile, 1u);
    const TrieTile tl = p.tiles[t];
    const int c = tl.c, d = tl.d, j = d + 1, nn = tl.nn;
    const bool leaf = tl.leaf;
    const bool single = d < 2;  // depth-1 nodes: one parent, the class's stage-1 table
    if (!single) {  // wait for the parents' runs (all their cell chunks)
      if (warp == 0)
        for (uint32_t r = tl.w0 + lane; r <= tl.w1; r += 32)
          while (ld_acquire(p.done + r) < tl.need) __nanosleep(128);
    }
    const ClassDev cl = p.cls[c];
    const TrieStage ts = p.tstage[(size_t)c * P1 + j];
    const int Np = (int)p.tstage[(size_t)c * P1 + j - 1].n, Nj = (int)ts.n, VS = (int)vrow(ts.n),
              VSp = (int)vrow((uint32_t)Np);
    const double* qt = p.qtab + (size_t)c * p.n_codes * L;
    const ProgDev pg = p.progs[p.class_prog[c]];
    const double* dom = p.domain + (size_t)cl.pair * p.nv_stride;
    double* vout = p.varena + tl.vout;
    uint8_t* bpo = p.bparena + tl.bout;
    const double* vpar = p.varena + tl.vpar;
    if (!single) __syncthreads();
    const double g1 = (double)(cl.gas - 1);
    if (ts.wide) {
      const int G = (nn + 3) >> 2, TW = 4 * G, TNst = TW + 2, ER = L - (j - 1);
      double* sV = smem_d;
      double* sE = sV + (single ? ((Np + 1) & ~1) : Np * TNst);
      double* sPf = sE + ER * TNst;
      AMP_CHECK((size_t)(sPf + LP - smem_d) * sizeof(double) <= (size_t)p.smem_bytes, "wide tile smem");
      if (single) {
        const double* src = p.v1g + p.v1off[c];
        for (int x = tid; x < Np; x += blockDim.x) sV[x] = src[x];
      } else {
        for (int ln = warp; ln < TW; ln += nw) {
          const int lr = ln < nn ? ln : 0;  // padding columns repeat node 0
          const double* src = vpar + (uint64_t)p.npar[tl.node + lr] * VSp;
          AMP_CHECK(src >= p.varena && src + Np <= p.varena + p.vcap, "wide parent row");
          for (int x = lane; x < Np; x += 32) cp_async8(sV + x * TNst + ln, src + x);
        }
      }
      for (int ln = warp; ln < TW; ln += nw) {
        const int lr = ln < nn ? ln : 0;
        const double* er = qt + (size_t)p.ncode[tl.node + lr] * L + (j - 1);
        for (int r = lane; r < ER; r += 32) sE[r * TNst + ln] = er[r];
      }
      for (int x = tid; x < LP; x += blockDim.x) sPf[x] = p.prefix[(size_t)cl.pair * LP + x];
      cp_async_wait_all();
      __syncthreads();
      if (single)
        tile_wide<true>(p, sV, sE, sPf, TNst, G, tl.x0, tl.x1, Nj, VS, j, nn, ts, p.preds + pg.pred_base, dom,
                        g1, leaf, vout, bpo, mine);
      else
        tile_wide<false>(p, sV, sE, sPf, TNst, G, tl.x0, tl.x1, Nj, VS, j, nn, ts, p.preds + pg.pred_base, dom,
                         g1, leaf, vout, bpo, mine);
    } else {
      const int P = single ? 1 : (int)tl.pn;
      const int Pst = P | 1;  // odd stride: rows start on distinct banks
      double* sV = smem_d;
      double* sE = sV + (size_t)Np * Pst;
      double* sPf = sE + (size_t)p.n_codes * L;
      int* sNode = reinterpret_cast<int*>(sPf + LP);  // (code << 16) | parent column
      AMP_CHECK((size_t)((char*)(sNode + nn) - (char*)smem_d) <= (size_t)p.smem_bytes, "narrow tile smem");
      if (single) {
        const double* src = p.v1g + p.v1off[c];
        for (int x = tid; x < Np; x += blockDim.x) sV[x * Pst] = src[x];
      } else {
        const double* src = vpar + (uint64_t)tl.pfirst * VSp;
        AMP_CHECK(single || (src >= p.varena && src + (uint64_t)(P - 1) * VSp + Np <= p.varena + p.vcap),
                  "narrow parent rows");
        for (int pl = warp; pl < P; pl += nw)
          for (int x = lane; x < Np; x += 32) cp_async8(sV + x * Pst + pl, src + (size_t)pl * VSp + x);
      }
      for (int x = tid; x < p.n_codes * L; x += blockDim.x) sE[x] = qt[x];
      for (int x = tid; x < LP; x += blockDim.x) sPf[x] = p.prefix[(size_t)cl.pair * LP + x];
      for (int x = tid; x < nn; x += blockDim.x) {
        const uint64_t node = (uint64_t)tl.node + x;
        sNode[x] = ((int)p.ncode[node] << 16) | (single ? 0 : (int)(p.npar[node] - tl.pfirst));
      }
      cp_async_wait_all();
      __syncthreads();
      tile_narrow(p, sV, sE, sPf, sNode, Pst, Nj, VS, j, nn, ts, p.preds + pg.pred_base, dom, g1, leaf, vout,
                  bpo, mine);
    }
    // publish: the CTA's stores (ordered before thread 0 by the barrier),
    // then the run's chunk count with release semantics
    if (tid == 0) s_t = tnext;
    __syncthreads();
    if (tid == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.done + tl.pub) : "memory");
    t = s_t;
  }
  if (p.exec) {  // executed inner iterations (roofline accounting), one atomic per warp
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0 && mine) atomicAdd(&p.exec[1], mine);
  }
}

// Shared memory (doubles) of a K_trie_dp tile at stage j (host mirror of the
// carve-ups above): wide, n groups of 4 nodes; narrow, n nodes (and at most
// n parents).
__host__ __device__ inline size_t trie_tile_doubles(bool wide, int j, int n, int Np, int L, int n_codes) {
  if (wide) {
    const size_t TNst = 4 * (size_t)n + 2;
    return (j == 2 ? ((size_t)Np + 1) & ~size_t(1) : (size_t)Np * TNst) + (size_t)(L - (j - 1)) * TNst +
           (size_t)L + 1;
  }
  const size_t Pst = (j == 2 ? 1 : (size_t)n) | 1;
  return (size_t)Np * Pst + (size_t)n_codes * L + (size_t)L + 1 + ((size_t)n + 1) / 2;
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
      AMP_CHECK(p.bbase[(size_t)d * p.n_cls + c] + (uint64_t)(node - nbc) * ts.n + x < p.bpcap, "backtrack argmin");
      const int cut = p.bparena[p.bbase[(size_t)d * p.n_cls + c] + (uint64_t)(node - nbc) * ts.n + x];
      co[j - 1] = (uint8_t)cut;
      const uint2 rec = p.cellrec[ts.cell0 + x];
      x = pr[rec.y + (cut - (j - 1))];
      if (d >= 2) node = p.npar[p.st->node_off[d] + node];
    }
    co[0] = 0;
  }
  if (p.exec && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&p.exec[0], (unsigned long long)n);
}

// Signature list only (trie off: the signature-mode K_dp solves the DP).
__global__ void k_sig_list(TrieParams p) {
  const uint64_t n = *p.n_sig;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = p.uniq[i];
    const unsigned long long k = p.tkey[s];
    p.sig_key[i] = p.key_shift >= 64 ? k : (k & ((1ull << p.key_shift) - 1));
    p.rep_item[i] = p.tval[s];
    p.tval[s] = (uint32_t)i;
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
