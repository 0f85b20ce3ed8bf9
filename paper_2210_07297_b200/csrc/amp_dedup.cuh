// amp_dedup.cuh — exact DP memoisation by signature.
//
// optimal_assignment (pipeline_dp.cpp:70-149) is a pure function of the
// class (pp, dp, tmp, mbs: layer times, gas, k) and the edge function
// e(cut, q) = act[cut-1]*mbs / bw[q] (optimizer.cpp:130-139).  With coded
// bandwidths (K_place) the edge function is fixed by the per-boundary codes,
// so candidates with the same signature key = class << (nq * cb) | codes
// have bit-identical cuts.  Per chunk the heavy items insert their keys into
// a hash table (fused into K_place_t, or k_hash_insert); its distinct keys
// become the signature list (amp_trie.cuh K_sig_init) whose DP is solved
// once; K_est reads each item's cuts at its signature.  Failed and pp <= 2
// items carry the all-ones key (never a real signature: keys use at most 63
// bits) and are not inserted.
#pragma once

#include "amp_common.cuh"

namespace amp {

// ---- signature hash table --------------------------------------------------
//
// Each heavy item inserts its key into an open-addressing table (linear
// probing, load <= 1/2): an item reads the slot first and only the first
// writer of a key CASes it in, so the many items of a hot signature cost one
// L2 read each.  The first writer appends the slot to the list of distinct
// keys (the signature list, in insertion order: the trie orders nothing by
// sorting).  Which item becomes a signature's representative does not
// matter: all its items have identical DP inputs.
constexpr uint64_t kHashEmpty = ~0ull;

struct HashParams {
  const CandWork* work;
  const ClassDev* cls;
  const uint8_t* bwcb;
  uint64_t n;              // heavy items
  int32_t max_pp, code_bits;
  int32_t wide, pad1;      // hashed keys (sig_key_wide)
  uint64_t mask;           // table size - 1
  uint64_t max_probe;      // probe bound (hash_insert_warp)
  uint64_t epoch;          // this run's tag (> 0)
  int32_t epoch_shift, pad0;  // key bits (tag above them), 64: no tag
  const uint64_t* sigkey;  // [n] keys written by K_place, or NULL (computed here)
  unsigned long long* tkey;  // [T] keys (kHashEmpty = free)
  uint32_t* tval;          // [T] first item, then run index
  uint32_t* slot_of;       // [n] slot of every item (~0u: no signature)
  uint32_t* uniq;          // [n] slots of the distinct keys
  unsigned long long* n_uniq;
  uint32_t* rep_of;        // [n] signature of every item (k_hash_scatter)
};

__device__ __forceinline__ uint64_t sig_key(const CandWork& w, const ClassDev* cls,
                                            const uint8_t* codes, int max_pp, int cb) {
  if (w.fail_code != 0) return kHashEmpty;
  const ClassDev cl = cls[w.cls];
  if (cl.pp < 3) return kHashEmpty;
  uint64_t key = (uint64_t)w.cls;
  for (int q = 0; q < max_pp - 1; ++q) key = (key << cb) | (q < cl.pp - 1 ? (uint64_t)codes[q] : 0ull);
  return key;
}

// Hashed key (the exact key would exceed 63 bits: |D| = 1024 with pp up to
// 64): a 64-bit mix of the class and the codes.  Equal signatures get equal
// keys; distinct ones may collide, which k_hash_verify detects exactly (the
// memoisation is then dropped for the chunk, see memo_bad).
__device__ __forceinline__ uint64_t sig_key_wide(const CandWork& w, const ClassDev* cls,
                                                 const uint8_t* codes) {
  if (w.fail_code != 0) return kHashEmpty;
  const ClassDev cl = cls[w.cls];
  if (cl.pp < 3) return kHashEmpty;
  uint64_t h = splitmix64((uint64_t)w.cls);
  const int nq = cl.pp - 1;
  for (int q0 = 0; q0 < nq; q0 += 8) {
    uint64_t word = 0;
    for (int q = q0; q < nq && q < q0 + 8; ++q) word |= (uint64_t)codes[q] << ((q - q0) * 8);
    h = splitmix64(h ^ word);
  }
  return h == kHashEmpty ? h - 1 : h;
}

// (the tests keep fewer hash bits to force collisions)
__device__ __forceinline__ uint64_t wide_bits(uint64_t k, int bits) {
  return (bits >= 64 || k == kHashEmpty) ? k : (k & ((1ull << bits) - 1));
}

// Table entries carry the run's epoch above the key bits (epoch_shift), so
// a slot of an older epoch reads as free and the table is never cleared
// between chunks (epoch_shift = 64: no tag, the table is cleared instead).
__device__ __forceinline__ bool slot_free(unsigned long long k, uint64_t epoch, int sh) {
  return sh >= 64 ? k == kHashEmpty : (k >> sh) != epoch;
}

// Lanes of a warp holding the same key (neighbouring placements of a class
// often share a signature) elect one prober (__match_any_sync): a hot
// signature's slot is read once per warp, not once per item, so the L2
// line holding it does not serialise the whole grid.  The loop trip count is
// uniform per warp for the warp-wide match / shuffle.
// Warp-cooperative insert (all 32 lanes call it): lanes with equal keys
// elect one prober; returns the key's slot (~0u for kHashEmpty).  The table
// is sized for every heavy item at load <= 1/2, so a probe always ends; the
// max_probe bound (= the table size) only guards the loop (n_uniq[1]).
__device__ __forceinline__ uint32_t hash_insert_warp(uint64_t key, uint64_t u, int lane,
                                                     unsigned long long* tkey, uint32_t* tval,
                                                     uint32_t* uniq, unsigned long long* n_uniq,
                                                     uint64_t mask, uint64_t tag, uint64_t epoch,
                                                     int sh, uint64_t max_probe) {
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int leader = __ffs(peers) - 1;
  uint32_t slot = ~0u;
  if (lane == leader && key != kHashEmpty) {
    const unsigned long long want = key | tag;
    uint64_t h = splitmix64(key) & mask;
    for (uint64_t probe = 0;; ++probe) {
      if (probe == max_probe) {
        atomicOr(&n_uniq[1], 1ull);
        break;
      }
      unsigned long long k = *(volatile unsigned long long*)&tkey[h];
      if (k == want) break;
      if (slot_free(k, epoch, sh)) {
        const unsigned long long old = atomicCAS(&tkey[h], k, want);
        if (old == k) {  // first writer of this key in this epoch
          tval[h] = (uint32_t)u;
          uniq[atomicAdd(n_uniq, 1ull)] = (uint32_t)h;
          break;
        }
        if (old == want) break;
        k = old;  // lost to another key: probe on
      }
      h = (h + 1) & mask;
    }
    slot = (uint32_t)h;
  }
  return __shfl_sync(0xffffffffu, slot, leader);
}

__global__ void k_hash_insert(HashParams p) {
  const int sh = p.epoch_shift, lane = threadIdx.x & 31;
  const uint64_t tag = sh >= 64 ? 0 : (p.epoch << sh);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < p.n;
       base += stride) {
    const uint64_t u = base + lane;
    const bool live = u < p.n;
    const uint64_t key = !live ? kHashEmpty
                         : p.sigkey ? p.sigkey[u]
                         : p.wide   ? wide_bits(sig_key_wide(p.work[u], p.cls, p.bwcb + u * p.max_pp), p.wide)
                                    : sig_key(p.work[u], p.cls, p.bwcb + u * p.max_pp, p.max_pp,
                                              p.code_bits);
    const uint32_t slot = hash_insert_warp(key, u, lane, p.tkey, p.tval, p.uniq, p.n_uniq, p.mask,
                                           tag, p.epoch, sh, p.max_probe);
    if (live) p.slot_of[u] = slot;
  }
}

__global__ void k_hash_scatter(HashParams p) {
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < p.n;
       base += stride) {
    const uint64_t u = base + lane;
    const bool live = u < p.n;
    const uint32_t s = live ? p.slot_of[u] : ~0u;
    const unsigned peers = __match_any_sync(0xffffffffu, s);  // one table read per distinct slot
    const int leader = __ffs(peers) - 1;
    uint32_t r = 0u;
    if (lane == leader && s != ~0u) r = p.tval[s];
    r = __shfl_sync(0xffffffffu, r, leader);
    if (live) p.rep_of[u] = r;
  }
}

// Hashed keys: every item's class and codes against its signature
// representative's (rep_of after k_hash_scatter, rep_list from K_sig_list);
// any difference is a collision and sets *bad.
__global__ void k_hash_verify(HashParams p, const uint32_t* rep_list, uint32_t* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < p.n; u += stride) {
    if (p.slot_of[u] == ~0u) continue;
    const uint64_t r = rep_list[p.rep_of[u]];
    if (r == u) continue;
    const CandWork& a = p.work[u];
    const CandWork& b = p.work[r];
    bool same = a.cls == b.cls && b.fail_code == 0;
    const int nq = p.cls[a.cls].pp - 1;
    const uint8_t* ca = p.bwcb + u * p.max_pp;
    const uint8_t* cb = p.bwcb + r * p.max_pp;
    for (int q = 0; same && q < nq; ++q) same = ca[q] == cb[q];
    if (!same) atomicOr(bad, 1u);
  }
}

}  // namespace amp
