// amp_dedup.cuh — exact DP memoisation by signature.
//
// optimal_assignment (pipeline_dp.cpp:70-149) is a pure function of the
// class (pp, dp, tmp, mbs: layer times, gas, k) and the edge function
// e(cut, q) = act[cut-1]*mbs / bw[q] (optimizer.cpp:130-139).  With coded
// bandwidths (K_place) the edge function is fixed by the per-boundary codes,
// so candidates with the same (class, code vector) have bit-identical cuts.
// Per chunk:
//   K_key    key[u] = class << (nq * cb) | codes, value u   (heavy items)
//   radix sort (cub::DeviceRadixSort) of (key, u)
//   K_heads  head flag of every run of equal keys
//   scan     run id of every sorted position (cub::DeviceScan)
//   K_reps   run heads -> rep_list[run] = u;  then rep_of[u] = rep_list[run]
// K_dp solves only rep_list[0 .. n_rep) (class-contiguous: the class is in
// the key's high bits), K_est reads each candidate's cuts at rep_of[u].
// Failed and pp <= 2 items get the all-ones key (never a real signature:
// keys use at most 63 bits); K_dp skips them as before.
#pragma once

#include "amp_common.cuh"

namespace amp {

struct DedupParams {
  const CandWork* work;
  const ClassDev* cls;
  const uint8_t* bwcb;  // [n][max_pp] boundary codes
  uint64_t n;           // heavy prefix of the chunk
  int32_t max_pp, code_bits, pad0, pad1;
  uint64_t* keys;       // [n]
  uint32_t* vals;       // [n]
  const uint64_t* skeys;  // sorted
  const uint32_t* svals;
  uint32_t* flags;      // [n] head flags -> (scan) run ids (inclusive)
  const uint32_t* runid;
  uint32_t* rep_list;   // [n] representative item of each run
  uint32_t* rep_of;     // [n] signature run of every item
  uint64_t* n_rep;      // device count of runs
  uint64_t* rep_key;    // [n] key of each run (NULL: not needed)
};

__global__ void k_dedup_keys(DedupParams p) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < p.n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const CandWork& w = p.work[u];
    uint64_t key = ~0ull;
    if (w.fail_code == 0) {
      const ClassDev cl = p.cls[w.cls];
      if (cl.pp >= 3) {
        key = (uint64_t)w.cls;
        const uint8_t* c = p.bwcb + u * p.max_pp;
        for (int q = 0; q < p.max_pp - 1; ++q)
          key = (key << p.code_bits) | (q < cl.pp - 1 ? (uint64_t)c[q] : 0ull);
      }
    }
    p.keys[u] = key;
    p.vals[u] = (uint32_t)u;
  }
}

__global__ void k_dedup_heads(DedupParams p) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < p.n;
       s += (uint64_t)gridDim.x * blockDim.x)
    p.flags[s] = (s == 0 || p.skeys[s] != p.skeys[s - 1]) ? 1u : 0u;
}

__global__ void k_dedup_reps(DedupParams p) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < p.n;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const bool head = s == 0 || p.skeys[s] != p.skeys[s - 1];
    if (head) {
      p.rep_list[p.runid[s] - 1] = p.svals[s];
      if (p.rep_key) p.rep_key[p.runid[s] - 1] = p.skeys[s];
    }
    if (s + 1 == p.n) *p.n_rep = p.runid[s];
  }
}

__global__ void k_dedup_scatter(DedupParams p) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < p.n;
       s += (uint64_t)gridDim.x * blockDim.x)
    p.rep_of[p.svals[s]] = p.runid[s] - 1;  // the signature's run (index into repcuts)
}

}  // namespace amp

namespace amp {

// ---- hash-based signature runs (replaces the full radix sort) -------------
//
// Each heavy item inserts its key into an open-addressing table (linear
// probing, load <= 1/2): an item reads the slot first and only the first
// writer of a key CASes it in, so the many items of a hot signature cost one
// L2 read each.  The first writer appends the slot to the list of distinct
// keys.  Only those (a few hundred thousand) are then sorted: the run order
// (class, c_0, c_1, ...) that K_dp / the trie need.  Which item becomes a
// signature's representative does not matter: all its items have identical
// DP inputs.
constexpr uint64_t kHashEmpty = ~0ull;

struct HashParams {
  const CandWork* work;
  const ClassDev* cls;
  const uint8_t* bwcb;
  uint64_t n;              // heavy items
  int32_t max_pp, code_bits;
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
  // after the host sorted the distinct keys
  const uint64_t* skeys;   // [n_uniq] sorted keys
  const uint32_t* sslots;  // [n_uniq] their slots
  uint64_t* rep_key;       // [n_uniq] (NULL: not needed)
  uint32_t* rep_list;      // [n_uniq] representative item of each run
  uint32_t* rep_of;        // [n] run of every item
  uint64_t* n_rep;         // device count of runs
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
// elect one prober; returns the key's slot (~0u for kHashEmpty).
// The table may be sized from the previous chunk's distinct-key count: a
// probe sequence longer than max_probe (such a table far above half full)
// gives up and raises n_uniq[1]; the host then redoes the chunk's inserts
// with a table sized for every item (max_probe = its size: never hit).
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
                                    : sig_key(p.work[u], p.cls, p.bwcb + u * p.max_pp, p.max_pp,
                                              p.code_bits);
    const uint32_t slot = hash_insert_warp(key, u, lane, p.tkey, p.tval, p.uniq, p.n_uniq, p.mask,
                                           tag, p.epoch, sh, p.max_probe);
    if (live) p.slot_of[u] = slot;
  }
}

__global__ void k_hash_gather(HashParams p, uint64_t* keys, uint32_t* slots) {
  const uint64_t n = *p.n_uniq;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = p.uniq[i];
    const unsigned long long k = p.tkey[s];
    keys[i] = p.epoch_shift >= 64 ? k : (k & ((1ull << p.epoch_shift) - 1));  // drop the tag
    slots[i] = s;
  }
}

__global__ void k_hash_runs(HashParams p) {
  const uint64_t n = *p.n_uniq;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = p.sslots[r];
    p.rep_list[r] = p.tval[s];
    if (p.rep_key) p.rep_key[r] = p.skeys[r];
    p.tval[s] = (uint32_t)r;  // slot -> run
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.n_rep = n;
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

}  // namespace amp
