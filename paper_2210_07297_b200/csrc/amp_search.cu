// amp_search.cu — host side of the C ABI declared in include/amp_search.h.
//
// Owns the device tables, launches K0 (pair tables) at create time and
// K1+K2 (evaluate) + K3 (merge) per run.  No CPU evaluation path exists:
// every candidate is evaluated by the sm_100a kernels; the host only
// enumerates classes (integers), encodes the profile map into a dense cube,
// and schedules work.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_set>
#include <vector>

#include "amp_common.cuh"
#include "amp_kernels.cuh"
#include "amp_pipeline.cuh"
#include "amp_dp_multi.cuh"
#include "amp_dedup.cuh"
#include "amp_thread.cuh"
#include "amp_trie.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

using namespace amp;

namespace {

thread_local std::string g_last_error;

// AMP_TIMING=1: print host-side phase times of amp_search_create to stderr.
struct PhaseTimer {
  bool on = std::getenv("AMP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[amp create] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Device buffers come from the device's stream-ordered memory pool, kept
// warm across contexts (release threshold = max), so a create/run/destroy
// cycle does not pay cudaMalloc/cudaFree.  Allocation, free and every use
// (uploads, memsets, kernels) are ordered on the stream of the API call in
// flight (g_alloc_stream: the context's stream), so no allocation needs a
// host synchronisation; an API call synchronises once before it returns.
thread_local cudaStream_t g_alloc_stream = nullptr;

void warm_pool(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done.push_back(device);
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes && p) return cudaSuccess;
    release();
    s = g_alloc_stream;
    cudaError_t e = cudaMallocAsync(&p, n ? n : 16, s);
    if (e == cudaSuccess) bytes = n;
    else p = nullptr;
    return e;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// Sets the allocation stream for the duration of an API call.
struct AllocStream {
  cudaStream_t prev;
  explicit AllocStream(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
  ~AllocStream() { g_alloc_stream = prev; }
};

// Per-device hand-over between contexts (the common create / run / destroy
// cycle of plan() and of the e2e path): a destroyed context leaves its
// (idle) stream, its signature hash table with its epoch state, and its trie
// mark array (kept clear by every run) to the next context created on the
// device, which then needs no stream creation and no table clearing.
struct Recycled {
  bool used = false;
  cudaStream_t stream = nullptr;
  void* tkey = nullptr;
  size_t tkey_bytes = 0;
  uint64_t T = 0, epoch = 0;
  int esh = -1;
  void* pres = nullptr;
  size_t pres_bytes = 0;
};
std::mutex g_rec_mu;

// NCCL communicators of a device set, handed from a destroyed multi-GPU
// context to the next one on the same devices (ncclCommInitAll and the
// connection setup of a communicator's first collective cost 0.1-1 s; a
// plan() creates a context per call).  A set is owned by one context at a
// time (checked out at create, returned at destroy).
std::mutex g_comm_mu;
std::map<std::vector<int>, std::vector<std::vector<ncclComm_t>>> g_comm_pool;
std::map<int, Recycled> g_rec;

std::vector<int> divisors(int n) {
  std::vector<int> out;
  for (int d = 1; d * d <= n; ++d)
    if (n % d == 0) {
      out.push_back(d);
      if (d != n / d) out.push_back(n / d);
    }
  std::sort(out.begin(), out.end());
  return out;
}

}  // namespace

struct amp_ctx {
  int device = 0;
  std::string err;
  int L = 0, D = 0, gbs = 0;
  uint64_t P = 1, seed = 0;
  int max_ctas_cfg = 0;
  int has_ceiling = 0;
  double ceiling = 0.0, bpp = 2.0;
  std::vector<ClassDev> classes;
  std::vector<PairDev> pairs;
  std::vector<double> class_inner;  // DP inner iterations per candidate
  std::vector<double> class_lt;     // of which m < seg(cut, i)
  std::vector<double> class_cells;
  int max_pp = 1, max_M = 1, nv_stride = 1, npow2 = 2;
  size_t bp_stride = 0, slice_stride = 0;
  int slice_in_smem = 1;
  int w_in_smem = 1;
  const void* eval_fn = nullptr;
  int eval_threads = kEvalThreads;
  size_t smem_bytes = 0;
  int n_ctas = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  DevBuf param, act, bw, base_order, times, prefix, domain, seg, pairs_d, cls_d;
  DevBuf bp, slice, wtab, cta_topk, topk, taken, segs, counter, index_list;
  DevBuf o_all, o_cuts, o_stage, o_edge, o_place, o_sim, simbuf;
  // pruned DP programs
  bool sparse = false, progs_ok = false;
  int mode = 0;
  std::vector<int32_t> class_prog;
  std::vector<ProgDev> progs_h;
  std::vector<double> prog_inner;  // inner iterations per program
  int max_cells = 1, max_prog_cells = 1;
  int max_n1 = 1, max_v = 1, max_rest = 1;
  int multi_b = 0;                 // K_dp multi: candidates per group (0: per-candidate k_dp)
  std::vector<double> prog_inner_raw;  // unpadded inner iterations per program
  // gangs: DP instances of programs >= gang_min inner iterations solved by
  // several CTAs (k_gang_plan + the gang phase of k_dp<kSparseG>)
  bool gang_on = false;
  double gang_min = 5e5, gang_unit = 4e6;  // (C4: DP 12.8 -> 3.4 ms; smaller parts lose to the per-stage barrier)
  int gang_max = 32;
  DevBuf gang_hdr, gang_slot, gang_off, gang_sync;
  size_t v_stride = 0;
  DevBuf progs_d, stage_d, class_prog_d, cells, cellpred, preds, vbuf;
  DevBuf c_work, c_place, c_bwq, c_cuts, c_bwc, c_placep;  // pipeline chunk buffers
  // bandwidth codes (ranks of the distinct link bandwidths) and per-class
  // edge-cost tables; n_codes = 0 when disabled
  int n_codes = 0;
  bool bw_positive = false;  // smallest distinct bandwidth > 0
  DevBuf bwcode, bwval, qtab, cellrec, cut2tab, rsum_t, rsum_p;
  DevBuf node_of, nodebw;  // node-determined bandwidths (n_nodes > 0)
  std::vector<int32_t> row_shape;  // code-table row -> shape key pp * 1024 + dp * 32 + tmp
  DevBuf row_shape_d, ctab;        // the code table (k_code_table), built for ctab_P placements
  uint64_t ctab_P = 0;
  int n_nodes = 0;
  DevBuf perm_tab;         // placements of p in [0, perm_n) (|D| = 16), built on first use
  uint64_t perm_n = 0;
  // multi-GPU context (config n_gpus > 1): this context drives the first
  // device, subs[r - 1] device + r; comms[r] is rank r's NCCL communicator
  std::vector<amp_ctx*> subs;
  std::vector<ncclComm_t> comms;
  std::vector<int> comm_devs;  // the devices of comms (the pool key)
  DevBuf gathered, mtopk;
  uint64_t n_heavy = 0;  // items of pp >= 3 classes in the current run's dispatch order
  // DP memoisation by signature (amp_dedup.cuh)
  bool dedup = false;
  bool wide = false;   // hashed signature keys (exact key > 63 bits), verified per chunk
  int wide_bits = 64;  // hash bits kept (AMP_WIDE_HASH_BITS: forced collisions in the tests)
  int code_bits = 0, key_bits = 0;
  DevBuf dd_rep_list, dd_rep_of, dd_bad;
  DevBuf dd_runpipe;  // per-run pipeline time of dp == 1 classes (k_run_pipe)
  DevBuf dd_counters, prog_inner_d, dd_repcuts;
  DevBuf dd_tkey, dd_tval, dd_slot, dd_uniq, dd_nuniq, dd_sigkey;  // hash dedup
  uint64_t hash_epoch = 0, hash_T = 0;
  int hash_esh = -1;  // epoch shift the table's tags were written with
  // DP shared across signature prefixes (amp_trie.cuh)
  bool trie = false;
  int trie_nq = 0, trie_U = 0;
  int tr_smem = 0;  // K_trie_dp dynamic smem per CTA
  int tr_build_grid = 0, tr_dp_grid = 0;
  std::vector<uint32_t> stage_h;  // host copy of the program stage starts
  std::vector<uint64_t> prog_stage_inner;  // [prog][L+1] unpadded (cell, cut) pairs of stage j
  std::vector<int32_t> root_cls_h;         // heavy classes (trie roots) in class order
  DevBuf tr_ghist, tr_gpart, tr_sortk, tr_sortv;  // k_trie_build_sorted scratch
  bool tr_sorted = true;                            // sorted-key trie build (AMP_TRIE_LEVELS=1: level build)
  DevBuf v1off_d, v1g_d, dd_rep_key, dd_nid, tr_state, tr_pres, tr_cid, tr_partial, tr_npar,
      tr_ncls, tr_ncode, tr_nb, tr_nK, tr_vbase, tr_bbase, tr_rbase, tr_tbase, tr_nxc, tr_tstage, tr_v0, tr_bp,
      tr_done, tr_tiles,
      tr_rank, tr_rcls;
  uint64_t tr_pres_cap = 0, tr_node_cap = 0, tr_vcap = 0, tr_bpcap = 0;
  std::vector<cudaEvent_t> tev;  // {before, after} every K_trie_dp launch of the last run
  int tev_used = 0;
  DevBuf ovf_log;                // trie capacity flag of every chunk of the last run
  int ovf_used = 0;
  uint64_t chunk = 1;
  int est_ctas = 1, sms = 148, launches = 0;
  // per-chunk kernel events {before K_place, after K_place, after K_dp,
  // after K_est}; resolved into stats.{place,dp,est}_ms
  std::vector<cudaEvent_t> kev;
  int kev_used = 0;
  bool kev_pending = false;
  bool stats_exec_pending = false;  // exec counters of a memoised run to read back
  amp_stats stats{};
  // light-tail overlap: K_est of the pp <= 2 items on a second stream while
  // the heavy items go through K_place -> K_dp -> K_est
  cudaStream_t aux = nullptr;
  cudaEvent_t aux_start = nullptr, aux_done = nullptr;
  int n_topk_lists = 0;  // CTA lists of the last launch_evaluate (main + aux)
};

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
      return e_ == cudaErrorMemoryAllocation ? AMP_E_OOM                              \
             : (e_ == cudaErrorNoKernelImageForDevice || e_ == cudaErrorInvalidDeviceFunction \
                    ? AMP_E_NOT_BUILT                                                 \
                    : AMP_E_CUDA);                                                    \
    }                                                                                 \
  } while (0)

// AMP_DEBUG_SYNC=1: synchronise after every kernel of a run and name the
// kernel that faulted (debugging aid; off in normal runs).
static const bool g_debug_sync = std::getenv("AMP_DEBUG_SYNC") != nullptr;
#define DBG_SYNC(name)                                                                   \
  do {                                                                                   \
    if (g_debug_sync) {                                                                  \
      cudaError_t e_ = cudaStreamSynchronize(ctx->stream);                               \
      if (e_ == cudaSuccess) e_ = cudaGetLastError();                                    \
      if (e_ != cudaSuccess) {                                                           \
        ctx->err = std::string(name) + ": " + cudaGetErrorString(e_);                    \
        return AMP_E_CUDA;                                                               \
      }                                                                                  \
    }                                                                                    \
  } while (0)

namespace {

int fail(amp_ctx* ctx, int code, const std::string& msg) {
  ctx->err = msg;
  return code;
}

template <class T>
cudaError_t upload(DevBuf& b, const T* src, size_t n) {
  cudaError_t e = b.ensure(sizeof(T) * n);
  if (e != cudaSuccess) return e;
  // (stream-ordered after the allocation; a pageable source is staged
  // before the call returns, a pinned one is read before the API call's
  // final synchronisation)
  if (n) e = cudaMemcpyAsync(b.p, src, sizeof(T) * n, cudaMemcpyHostToDevice, g_alloc_stream);
  return e;
}

// K0b driver: programs for every distinct (pair, k) of the feasible classes.
// Pass 1 counts |N_j| and predecessor entries per stage; the host lays out
// the arrays; pass 2 writes them.  Sets ctx->progs_ok = false (dense DP)
// when some |N_j| exceeds the u16 index range.
int build_programs(amp_ctx* ctx, const std::vector<uint16_t>& seg_h) {
  (void)seg_h;
  const int L = ctx->L, LP = L + 1;
  std::map<std::pair<int, int>, int> prog_of;
  std::vector<int32_t> pk, ppair;
  ctx->class_prog.assign(ctx->classes.size(), 0);
  for (size_t c = 0; c < ctx->classes.size(); ++c) {
    const ClassDev& cl = ctx->classes[c];
    if (cl.pp > L || ctx->pairs[cl.pair].fail_code) continue;
    auto key = std::make_pair(cl.pair, cl.pp);
    auto it = prog_of.find(key);
    if (it == prog_of.end()) {
      it = prog_of.emplace(key, (int)pk.size()).first;
      pk.push_back(cl.pp);
      ppair.push_back(cl.pair);
    }
    ctx->class_prog[c] = it->second;
  }
  const int n = (int)pk.size();
  ctx->progs_ok = true;
  ctx->prog_inner.assign(n, 0.0);
  if (n == 0) {
    CK(upload(ctx->class_prog_d, ctx->class_prog.data(), ctx->class_prog.size()));
    return AMP_OK;
  }
  DevBuf d_k, d_pair, d_bm, d_bmoff, d_sizes, d_preds_n, d_inner_n, d_items;
  CK(upload(d_k, pk.data(), pk.size()));
  CK(upload(d_pair, ppair.data(), ppair.size()));
  // stage bitmaps of every program ([k][(L+1) * W] u32 each)
  std::vector<uint64_t> bmoff(n);
  uint64_t bm_total = 0;
  for (int g = 0; g < n; ++g) {
    bmoff[g] = bm_total;
    bm_total += (uint64_t)pk[g] * LP * ((ctx->pairs[ppair[g]].M + 31) / 32);
  }
  const int W = (ctx->max_M + 31) / 32;
  const size_t nw = (size_t)LP * W;
  const size_t smem_c = sizeof(uint32_t) * 2 * nw + sizeof(uint16_t) * ((LP * LP + 1) & ~1) + sizeof(int) * 3 * LP;
  const size_t smem_e = sizeof(uint32_t) * (4 * nw + 2 * kEmitSlice) + sizeof(uint64_t) * LP + sizeof(uint16_t) * LP * LP;
  if (smem_c > 227 * 1024 || smem_e > 227 * 1024 || bm_total > (4ull << 30)) {
    ctx->progs_ok = false;
    return AMP_OK;
  }
  CK(d_bm.ensure(sizeof(uint32_t) * bm_total));
  CK(upload(d_bmoff, bmoff.data(), bmoff.size()));
  CK(d_sizes.ensure(sizeof(uint32_t) * (size_t)n * LP));
  CK(d_preds_n.ensure(sizeof(uint64_t) * (size_t)n * LP));
  CK(d_inner_n.ensure(sizeof(uint64_t) * (size_t)n * LP));
  CK(cudaMemsetAsync(d_sizes.p, 0, sizeof(uint32_t) * (size_t)n * LP, ctx->stream));
  CK(cudaMemsetAsync(d_preds_n.p, 0, sizeof(uint64_t) * (size_t)n * LP, ctx->stream));
  CK(cudaMemsetAsync(d_inner_n.p, 0, sizeof(uint64_t) * (size_t)n * LP, ctx->stream));
  ProgBuildParams bp{};
  bp.L = L;
  bp.n_progs = n;
  bp.prog_k = d_k.as<int32_t>();
  bp.prog_pair = d_pair.as<int32_t>();
  bp.pairs = ctx->pairs_d.as<PairDev>();
  bp.seg = ctx->seg.as<uint16_t>();
  bp.bm = d_bm.as<uint32_t>();
  bp.bm_off = d_bmoff.as<uint64_t>();
  bp.stage_sizes = d_sizes.as<uint32_t>();
  bp.stage_preds = d_preds_n.as<uint64_t>();
  bp.stage_inner = d_inner_n.as<uint64_t>();
  PhaseTimer tm;
  CK(cudaFuncSetAttribute(k_prog_closure, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c));
  k_prog_closure<<<n, 512, smem_c, ctx->stream>>>(bp);
  CK(cudaGetLastError());
  std::vector<uint32_t> sizes((size_t)n * LP);
  std::vector<uint64_t> pn((size_t)n * LP), pin((size_t)n * LP);
  CK(cudaMemcpyAsync(sizes.data(), d_sizes.p, sizeof(uint32_t) * sizes.size(),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(pn.data(), d_preds_n.p, sizeof(uint64_t) * pn.size(), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaMemcpyAsync(pin.data(), d_inner_n.p, sizeof(uint64_t) * pin.size(),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  tm.mark("K0b closure");
  ctx->prog_inner_raw.assign(n, 0.0);
  ctx->prog_stage_inner = pin;
  // layout
  std::vector<ProgDev> progs(n);
  std::vector<uint32_t> stage;
  std::vector<uint64_t> pstart((size_t)n * LP, 0);
  std::vector<uint4> items;  // emit work: {g, j, first cell, end cell}
  uint64_t cell_total = 0, pred_total = 0;
  int max_cells = 1;
  uint64_t max_prog_cells = 1;
  for (int g = 0; g < n; ++g) {
    const int k = pk[g];
    ProgDev& d = progs[g];
    d.k = k;
    d.pair = ppair[g];
    d.cell_base = (uint32_t)cell_total;
    d.stage_base = (uint32_t)stage.size();
    d.pred_base = pred_total;
    uint32_t acc = 0, mx = 0;
    for (int j = 1; j <= k; ++j) {
      stage.push_back(acc);
      const uint32_t sz = sizes[(size_t)g * LP + j];
      for (uint32_t x = 0; x < sz; x += kEmitSlice)
        items.push_back(make_uint4((uint32_t)g, (uint32_t)j, x, std::min(sz, x + kEmitSlice)));
      acc += sz;
      mx = std::max(mx, sz);
    }
    stage.push_back(acc);
    uint64_t pacc = 0, iacc = 0;
    uint32_t mxv = 1;
    for (int j = 2; j <= k; ++j) {
      pstart[(size_t)g * LP + j] = pacc;
      pacc += pn[(size_t)g * LP + j];
      iacc += pin[(size_t)g * LP + j];
      mxv = std::max(mxv, sizes[(size_t)g * LP + j]);
    }
    ctx->prog_inner_raw[g] = (double)iacc;
    ctx->max_n1 = std::max<int>(ctx->max_n1, (int)sizes[(size_t)g * LP + 1]);
    if (k >= 2) {
      ctx->max_v = std::max<int>(ctx->max_v, (int)mxv);
      ctx->max_rest = std::max<int>(ctx->max_rest, (int)(acc - sizes[(size_t)g * LP + 1]));
    }
    d.n_cells = acc;
    d.max_cells = mx;
    d.n_preds = pacc;
    d.ok = mx < 65536;  // u16 indices plus the sentinel slot |N_j|
    if (!d.ok) ctx->progs_ok = false;
    cell_total += acc;
    pred_total += pacc;
    max_cells = std::max<int>(max_cells, (int)mx);
    max_prog_cells = std::max<uint64_t>(max_prog_cells, acc);
    ctx->prog_inner[g] = (double)pacc;
  }
  if (!ctx->progs_ok || cell_total >= (1ull << 32)) {
    ctx->progs_ok = false;
    return AMP_OK;
  }
  ctx->max_cells = max_cells;
  ctx->max_prog_cells = (int)max_prog_cells;
  CK(upload(ctx->progs_d, progs.data(), progs.size()));
  CK(upload(ctx->stage_d, stage.data(), stage.size()));
  ctx->stage_h = stage;
  CK(upload(ctx->class_prog_d, ctx->class_prog.data(), ctx->class_prog.size()));
  DevBuf d_pst;
  CK(upload(d_pst, pstart.data(), pstart.size()));
  CK(upload(d_items, items.data(), items.size()));
  CK(ctx->cells.ensure(sizeof(uint32_t) * cell_total));
  CK(ctx->cellpred.ensure(sizeof(uint32_t) * cell_total));
  CK(ctx->preds.ensure(sizeof(uint16_t) * (pred_total + 8)));
  bp.progs = ctx->progs_d.as<ProgDev>();
  bp.cells = ctx->cells.as<uint32_t>();
  bp.cellpred = ctx->cellpred.as<uint32_t>();
  bp.preds = ctx->preds.as<uint16_t>();
  bp.stage = ctx->stage_d.as<uint32_t>();
  bp.pred_start = d_pst.as<uint64_t>();
  bp.items = d_items.as<uint4>();
  tm.mark("K0b layout+alloc");
  CK(cudaFuncSetAttribute(k_prog_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e));
  if (!items.empty()) k_prog_emit<<<(unsigned)items.size(), 512, smem_e, ctx->stream>>>(bp);
  CK(cudaGetLastError());
  if (tm.on) CK(cudaStreamSynchronize(ctx->stream));
  tm.mark("K0b emit");
  if (tm.on)
    std::fprintf(stderr, "[amp create] K0b: %d programs, cells %llu, preds %llu, max |N_j| %d, %zu emit CTAs\n", n,
                 (unsigned long long)cell_total, (unsigned long long)pred_total, max_cells, items.size());
  ctx->progs_h = progs;
  return AMP_OK;
}

bool is_heavy(const amp_ctx* ctx, uint64_t c);

// Dynamic smem of k_dp_multi<b> (mirror of its carve-up).
size_t multi_smem_bytes(const amp_ctx* ctx, int b) {
  const int L = ctx->L;
  size_t d = sizeof(double) * (2 * (size_t)(ctx->max_v + 1) * b + 2 * (size_t)(L + 3) * b +
                               (ctx->max_n1 + 1) + ctx->max_M + (L + 4));
  return d + 2 * (size_t)b * ctx->max_rest + 16;  // two backpointer buffers
}

int setup(amp_ctx* ctx, const amp_problem* p, const amp_search_config* cfg) {
  if (!p) return fail(ctx, AMP_E_INVALID, "problem is NULL");
  const int L = p->n_layers, D = p->n_devices;
  if (L < 1) return fail(ctx, AMP_E_INVALID, "model must have at least one layer");
  if (L > kMaxLayers)
    return fail(ctx, AMP_E_UNSUPPORTED, "n_layers > " + std::to_string(kMaxLayers));
  if (D < 1) return fail(ctx, AMP_E_INVALID, "cluster must have at least one device");
  if (D > 4096) return fail(ctx, AMP_E_UNSUPPORTED, "n_devices > 4096");
  if (p->gbs < 1) return fail(ctx, AMP_E_INVALID, "gbs must be >= 1");
  if (!p->param_count || !p->node_id || !p->bandwidth || (L > 1 && !p->activation_volumes))
    return fail(ctx, AMP_E_INVALID, "missing model/cluster array");
  if (p->n_profile_entries < 0 ||
      (p->n_profile_entries > 0 &&
       (!p->profile_layer || !p->profile_tmp || !p->profile_mbs || !p->profile_seconds)))
    return fail(ctx, AMP_E_INVALID, "missing profile arrays");
  const uint64_t P = cfg ? cfg->placements_per_class : 1;
  if (P < 1) return fail(ctx, AMP_E_INVALID, "placements_per_class must be >= 1");
  ctx->L = L;
  ctx->D = D;
  ctx->gbs = p->gbs;
  ctx->P = P;
  ctx->seed = cfg ? cfg->seed : 0;
  ctx->device = cfg ? cfg->device : 0;
  ctx->max_ctas_cfg = cfg ? cfg->max_ctas : 0;
  ctx->has_ceiling = p->has_max_params_per_device;
  ctx->ceiling = p->max_params_per_device;
  ctx->bpp = p->bytes_per_param;

  PhaseTimer tm;
  CK(cudaSetDevice(ctx->device));
  // cudaGetDeviceProperties costs milliseconds; cache it per device
  static std::mutex prop_mu;
  static std::map<int, cudaDeviceProp> prop_cache;
  cudaDeviceProp prop;
  {
    std::lock_guard<std::mutex> lk(prop_mu);
    auto it = prop_cache.find(ctx->device);
    if (it == prop_cache.end()) {
      CK(cudaGetDeviceProperties(&prop, ctx->device));
      prop_cache.emplace(ctx->device, prop);
    } else {
      prop = it->second;
    }
  }
  tm.mark("device+props");
  if (prop.major != 10)
    return fail(ctx, AMP_E_NOT_BUILT,
                "device is sm_" + std::to_string(prop.major * 10 + prop.minor) +
                    "; this build contains sm_100a kernels only");
  warm_pool(ctx->device);
  {
    std::lock_guard<std::mutex> lk(g_rec_mu);
    Recycled& r = g_rec[ctx->device];
    if (r.used && std::getenv("AMP_NO_RECYCLE") == nullptr) {
      ctx->stream = r.stream;
      ctx->dd_tkey.p = r.tkey;
      ctx->dd_tkey.bytes = r.tkey_bytes;
      ctx->dd_tkey.s = r.stream;
      ctx->hash_T = r.T;
      ctx->hash_epoch = r.epoch;
      ctx->hash_esh = r.esh;
      ctx->tr_pres.p = r.pres;
      ctx->tr_pres.bytes = r.pres_bytes;
      ctx->tr_pres.s = r.stream;
      r = Recycled{};
    }
  }
  if (!ctx->stream) CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  g_alloc_stream = ctx->stream;
  CK(cudaEventCreate(&ctx->ev0));
  CK(cudaEventCreate(&ctx->ev1));
  CK(cudaEventCreate(&ctx->ev2));

  tm.mark("stream/events");
  // ---- classes: the plan() candidate list (optimizer.cpp:202-207) -------
  std::map<std::pair<int, int>, int> pair_of;
  std::vector<int> pair_tmp, pair_mbs;
  for (int pp : divisors(D))
    for (int dp : divisors(D / pp)) {
      const int tmp = D / (pp * dp);
      if (p->gbs % dp != 0) continue;
      for (int mbs : divisors(p->gbs / dp)) {
        auto key = std::make_pair(tmp, mbs);
        auto it = pair_of.find(key);
        int pr;
        if (it == pair_of.end()) {
          pr = static_cast<int>(pair_tmp.size());
          pair_of.emplace(key, pr);
          pair_tmp.push_back(tmp);
          pair_mbs.push_back(mbs);
        } else {
          pr = it->second;
        }
        ClassDev c{};
        c.pp = pp;
        c.dp = dp;
        c.tmp = tmp;
        c.mbs = mbs;
        c.gas = p->gbs / (dp * mbs);
        c.pair = pr;
        ctx->classes.push_back(c);
        if (pp <= L) ctx->max_pp = std::max(ctx->max_pp, pp);  // (pp > L fails before any stage)
      }
    }
  if (ctx->classes.empty()) return fail(ctx, AMP_E_INVALID, "no candidates");
  const int n_pairs = static_cast<int>(pair_tmp.size());

  // ---- profile cube: ProfileTable map -> dense [pair][layer] -----------
  std::vector<double> cube((size_t)n_pairs * L, 0.0);
  std::vector<uint8_t> hit((size_t)n_pairs * L, 0);
  for (int64_t e = 0; e < p->n_profile_entries; ++e) {  // later entries overwrite
    const int l = p->profile_layer[e];
    if (l < 0 || l >= L) continue;
    auto it = pair_of.find({p->profile_tmp[e], p->profile_mbs[e]});
    if (it == pair_of.end()) continue;
    cube[(size_t)it->second * L + l] = p->profile_seconds[e];
    hit[(size_t)it->second * L + l] = 1;
  }
  std::vector<double> flops(L, 0.0);
  std::vector<uint8_t> flops_ok(L, 0);
  for (int l = 0; l < L; ++l) {
    flops_ok[l] = p->flops_present ? p->flops_present[l] : 0;
    if (flops_ok[l] && p->flops_per_sample) flops[l] = p->flops_per_sample[l];
  }
  std::vector<double> act(std::max(1, L - 1), 0.0);
  for (int l = 0; l + 1 < L; ++l) act[l] = p->activation_volumes[l];
  std::vector<double> bw((size_t)D * D);
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j)
      bw[(size_t)i * D + j] = i == j ? INFINITY : p->bandwidth[(size_t)i * D + j];
  // heuristic_placement device order (placement.cpp:37-49)
  std::vector<int> order(D);
  for (int i = 0; i < D; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return p->node_id[a] != p->node_id[b] ? p->node_id[a] < p->node_id[b] : a < b;
  });

  // ---- bandwidth codes: rank of each link among the distinct bandwidths --
  // (used by K_place and the K_dp edge tables; disabled with NaN links or
  // more than 255 distinct values)
  {
    // distinct values: a hash set (|D|^2 entries, few distinct), then sort
    std::vector<double> vals;
    bool nan = false;
    {
      // (runs of equal links are the common case: compare with the previous
      // link before the set lookup)
      std::unordered_set<uint64_t> seen;
      uint64_t last_bits = 0;
      bool have_last = false;
      for (double v : bw) {
        if (std::isnan(v)) {
          nan = true;
          break;
        }
        uint64_t bits;
        std::memcpy(&bits, &v, sizeof bits);
        if (v == 0.0) bits = 0;  // +0 / -0 are one value
        if (have_last && bits == last_bits) continue;
        last_bits = bits;
        have_last = true;
        if (seen.insert(bits).second) vals.push_back(v == 0.0 ? 0.0 : v);
        if (vals.size() > 255) break;  // codes disabled anyway
      }
    }
    std::sort(vals.begin(), vals.end());
    ctx->n_codes = 0;
    if (!nan && vals.size() <= 255 && std::getenv("AMP_NO_CODES") == nullptr) {
      std::vector<uint8_t> code((size_t)D * D);
      double last = NAN;
      uint8_t last_c = 0;
      for (size_t x = 0; x < code.size(); ++x) {  // (runs of equal values are common)
        if (!(bw[x] == last)) {
          last = bw[x];
          last_c = (uint8_t)(std::lower_bound(vals.begin(), vals.end(), bw[x]) - vals.begin());
        }
        code[x] = last_c;
      }
      const int U = (int)vals.size();
      // qtab[cls][code][c] = act[c-1] * mbs / vals[code] (optimizer.cpp:130-139)
      const size_t qn = ctx->classes.size() * (size_t)U * L;
      if (qn * sizeof(double) <= ((size_t)256 << 20)) {
        std::vector<double> q(qn, 0.0);
        for (size_t c = 0; c < ctx->classes.size(); ++c)
          for (int u = 0; u < U; ++u)
            for (int cut = 1; cut < L; ++cut)
              q[(c * U + u) * L + cut] = act[cut - 1] * ctx->classes[c].mbs / vals[u];
        CK(upload(ctx->bwcode, code.data(), code.size()));
        CK(upload(ctx->bwval, vals.data(), vals.size()));
        CK(upload(ctx->qtab, q.data(), q.size()));
        ctx->n_codes = U;
        ctx->bw_positive = vals[0] > 0;
      }
    }
  }
  // ---- node-determined bandwidths (every link a function of its two
  //      nodes, symmetric, no NaN): the node-pair all-reduce minimum ------
  {
    std::vector<int> nodes(p->node_id, p->node_id + D);
    std::sort(nodes.begin(), nodes.end());
    nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
    const int NN = (int)nodes.size();
    std::vector<int32_t> nof(D);
    for (int a = 0; a < D; ++a)
      nof[a] = (int32_t)(std::lower_bound(nodes.begin(), nodes.end(), p->node_id[a]) - nodes.begin());
    bool ok = D > 32 && NN <= 4096 && std::getenv("AMP_NO_NODEBW") == nullptr;
    std::vector<double> nb(ok ? (size_t)NN * NN : 0, NAN);
    std::vector<uint8_t> set(ok ? (size_t)NN * NN : 0, 0);
    for (int a = 0; a < D && ok; ++a) {
      const double* row = bw.data() + (size_t)a * D;
      double* nrow = nb.data() + (size_t)nof[a] * NN;
      uint8_t* srow = set.data() + (size_t)nof[a] * NN;
      for (int b = 0; b < D; ++b) {
        if (a == b) continue;
        const double v = row[b];
        const int x = nof[b];
        if (srow[x]) {
          if (!(nrow[x] == v)) ok = false;  // (NaN != NaN: rejected too)
        } else if (std::isnan(v)) {
          ok = false;
        } else {
          nrow[x] = v;
          srow[x] = 1;
        }
      }
    }
    for (int n1 = 0; n1 < NN && ok; ++n1)
      for (int n2 = n1 + 1; n2 < NN && ok; ++n2)
        if (set[(size_t)n1 * NN + n2] && !(nb[(size_t)n1 * NN + n2] == nb[(size_t)n2 * NN + n1])) ok = false;
    ctx->n_nodes = ok ? NN : 0;
    if (ok) {
      for (size_t x = 0; x < nb.size(); ++x)
        if (!set[x]) nb[x] = INFINITY;  // (a node with one device: never read)
      CK(upload(ctx->node_of, nof.data(), nof.size()));
      CK(upload(ctx->nodebw, nb.data(), nb.size()));
    }
  }
  CK(upload(ctx->param, p->param_count, L));
  CK(upload(ctx->act, act.data(), act.size()));
  CK(upload(ctx->bw, bw.data(), bw.size()));
  CK(upload(ctx->base_order, order.data(), order.size()));
  // code-table rows: the distinct full 16-device shapes (K_place / K_est
  // shape kernels read the placement's link codes by (shape, placement))
  ctx->row_shape.clear();
  for (ClassDev& c : ctx->classes) {
    c.crow = -1;
    if (D != 16 || c.pp * c.dp * c.tmp != 16) continue;
    const int key = c.pp * 1024 + c.dp * 32 + c.tmp;
    auto it = std::find(ctx->row_shape.begin(), ctx->row_shape.end(), key);
    c.crow = (int32_t)(it - ctx->row_shape.begin());
    if (it == ctx->row_shape.end()) ctx->row_shape.push_back(key);
  }
  if (!ctx->row_shape.empty()) CK(upload(ctx->row_shape_d, ctx->row_shape.data(), ctx->row_shape.size()));
  CK(upload(ctx->cls_d, ctx->classes.data(), ctx->classes.size()));

  tm.mark("encode+uploads");
  // ---- K0: pair tables on the device ----------------------------------
  const int nv = 1 + L * (L + 1) / 2;
  int npow2 = 2;
  while (npow2 < nv) npow2 <<= 1;
  ctx->npow2 = npow2;
  ctx->nv_stride = nv;
  DevBuf d_cube, d_hit, d_flops, d_flops_ok, d_ptmp, d_pmbs;
  CK(upload(d_cube, cube.data(), cube.size()));
  CK(upload(d_hit, hit.data(), hit.size()));
  CK(upload(d_flops, flops.data(), flops.size()));
  CK(upload(d_flops_ok, flops_ok.data(), flops_ok.size()));
  CK(upload(d_ptmp, pair_tmp.data(), pair_tmp.size()));
  CK(upload(d_pmbs, pair_mbs.data(), pair_mbs.size()));
  CK(ctx->pairs_d.ensure(sizeof(PairDev) * n_pairs));
  CK(ctx->times.ensure(sizeof(double) * n_pairs * L));
  CK(ctx->prefix.ensure(sizeof(double) * n_pairs * (L + 1)));
  CK(ctx->domain.ensure(sizeof(double) * (size_t)n_pairs * nv));
  CK(ctx->seg.ensure(sizeof(uint16_t) * (size_t)n_pairs * (L + 1) * (L + 1)));
  TableParams tp{};
  tp.L = L;
  tp.n_pairs = n_pairs;
  tp.npow2 = npow2;
  tp.fallback_enabled = p->fallback_enabled;
  tp.pair_tmp = d_ptmp.as<int32_t>();
  tp.pair_mbs = d_pmbs.as<int32_t>();
  tp.cube = d_cube.as<double>();
  tp.cube_hit = d_hit.as<uint8_t>();
  tp.flops = d_flops.as<double>();
  tp.flops_ok = d_flops_ok.as<uint8_t>();
  tp.act = ctx->act.as<double>();
  tp.device_flops = p->fallback_device_flops;
  tp.tmp_bandwidth = p->fallback_tmp_bandwidth;
  tp.pairs = ctx->pairs_d.as<PairDev>();
  tp.times = ctx->times.as<double>();
  tp.prefix = ctx->prefix.as<double>();
  tp.domain = ctx->domain.as<double>();
  tp.seg = ctx->seg.as<uint16_t>();
  tp.nv_stride = nv;
  const size_t k0_smem = sizeof(double) * (npow2 + L + 1);
  CK(cudaFuncSetAttribute(k_pair_tables, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)k0_smem));
  k_pair_tables<<<n_pairs, 512, k0_smem, ctx->stream>>>(tp);
  CK(cudaGetLastError());
  ctx->pairs.resize(n_pairs);
  std::vector<uint16_t> seg_h((size_t)n_pairs * (L + 1) * (L + 1));
  CK(cudaMemcpyAsync(ctx->pairs.data(), ctx->pairs_d.p, sizeof(PairDev) * n_pairs,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(seg_h.data(), ctx->seg.p, sizeof(uint16_t) * seg_h.size(),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));

  tm.mark("K0 pair tables");
  // ---- per-class work accounting (scheduling + roofline) ---------------
  ctx->class_inner.assign(ctx->classes.size(), 0.0);
  ctx->class_lt.assign(ctx->classes.size(), 0.0);
  ctx->class_cells.assign(ctx->classes.size(), 0.0);
  size_t bp_stride = 16;
  for (size_t c = 0; c < ctx->classes.size(); ++c) {
    const ClassDev& cl = ctx->classes[c];
    const PairDev& pr = ctx->pairs[cl.pair];
    if (cl.pp > L || pr.fail_code) continue;
    const int M = pr.M;
    ctx->max_M = std::max(ctx->max_M, M);
    bp_stride = std::max(bp_stride, (size_t)(cl.pp + 1) * (L + 1) * M);
    double inner = 0, lt = 0;
    const uint16_t* sg = seg_h.data() + (size_t)cl.pair * (L + 1) * (L + 1);
    for (int cut = 1; cut < L; ++cut) {
      const int w = std::min(cl.pp, cut + 1) - 1;  // stages j in [2, min(k, cut+1)]
      if (w <= 0) continue;
      for (int i = cut + 1; i <= L; ++i) {
        inner += (double)w * M;
        lt += (double)w * sg[cut * (L + 1) + i];
      }
    }
    ctx->class_inner[c] = inner;
    ctx->class_lt[c] = lt;
    double cells = (double)L * M;
    for (int j = 2; j <= cl.pp; ++j) cells += (double)(L - j + 1) * M;
    ctx->class_cells[c] = cells;
  }
  ctx->bp_stride = (bp_stride + 255) & ~size_t(255);

  const int LP = L + 1;
  tm.mark("class accounting");
  // ---- K0b: pruned-DP programs, one per distinct (pair, k) ---------------
  bool sparse = !(cfg && (cfg->flags & AMP_FLAG_DENSE_DP));
  if (sparse) {
    int rc = build_programs(ctx, seg_h);
    if (rc != AMP_OK) return rc;
    sparse = ctx->progs_ok;
  }
  ctx->sparse = sparse;
  if (sparse)  // scheduling/roofline weights: executed predecessor entries
    for (size_t c = 0; c < ctx->classes.size(); ++c)
      if (ctx->class_inner[c] > 0) {
        ctx->class_inner[c] = ctx->prog_inner_raw[ctx->class_prog[c]];
        ctx->class_lt[c] = 0;
      }

  tm.mark("K0b programs");
  // ---- evaluate kernel launch shape -------------------------------------
  // K_dp smem (mirror of the carve-up in amp_pipeline.cuh k_dp)
  size_t small = 16 + sizeof(double) * ctx->max_M + sizeof(double) * LP +
                 4 * sizeof(double) * L + sizeof(CandWork) * kDpBatch +
                 sizeof(int) * (ctx->max_pp + 2);
  small = (small + 15) & ~size_t(15);
  const size_t w_b = sizeof(WEnt) * (size_t)LP * L;
  int mode;
  if (sparse) {
    // value arrays (2 stages) + backpointers of one candidate
    const size_t v_b = sizeof(double) * 2 * (size_t)ctx->max_cells +
                       (((size_t)ctx->max_prog_cells + 15) & ~size_t(15));
    const bool v_smem = small + v_b <= 64 * 1024;
    mode = v_smem ? kSparseS : kSparseG;
    if (mode == kSparseG && std::getenv("AMP_NO_GANG") == nullptr) {
      // (C4: a few instances hold most of the DP — pp = 64 programs of
      // ~1e7 iterations — and would each bound the launch on one SM)
      if (const char* e = std::getenv("AMP_GANG_MIN")) ctx->gang_min = std::atof(e);
      if (const char* e = std::getenv("AMP_GANG_UNIT")) ctx->gang_unit = std::atof(e);
      if (const char* e = std::getenv("AMP_GANG_MAX")) ctx->gang_max = std::max(2, std::atoi(e));
      for (double x : ctx->prog_inner_raw) ctx->gang_on = ctx->gang_on || x >= ctx->gang_min;
    }
    ctx->smem_bytes = small + (v_smem ? v_b : 0);
    ctx->eval_threads = v_smem ? 128 : 1024;
    ctx->bp_stride = v_smem ? 0 : (((size_t)ctx->max_prog_cells + 255) & ~size_t(255));
    ctx->v_stride = v_smem ? 0 : 2 * (size_t)ctx->max_cells;
    ctx->slice_in_smem = ctx->w_in_smem = 1;
  } else {
    // smem = [C slice (L+1) x max_M] [W table (L+1) x L x 32 B] + small
    // arrays + seg table; keep whichever big one fits (slice first).
    small += sizeof(uint16_t) * LP * LP;
    const size_t slice_b = sizeof(double) * (size_t)LP * ctx->max_M;
    const size_t smem_limit = 200 * 1024;
    ctx->slice_in_smem = small + slice_b <= smem_limit;
    ctx->w_in_smem = small + w_b + (ctx->slice_in_smem ? slice_b : 0) <= smem_limit;
    ctx->smem_bytes = small + (ctx->slice_in_smem ? slice_b : 0) + (ctx->w_in_smem ? w_b : 0);
    mode = ctx->slice_in_smem ? (ctx->w_in_smem ? kDenseSS : kDenseSG)
                              : (ctx->w_in_smem ? kDenseGS : kDenseGG);
    // one thread per domain column (threads beyond M idle in the DP sweep)
    ctx->eval_threads = std::min(kEvalThreads, std::max(128, (ctx->max_M + 31) / 32 * 32));
    ctx->v_stride = 0;
  }
  // K_dp multi (amp_dp_multi.cuh): B candidates of one class per group when
  // B value arrays + backpointers fit two CTAs per SM.  AMP_DP_B=0 selects
  // the per-candidate kernel (comparison runs).
  ctx->multi_b = 0;
  if (sparse) {
    const char* eb = std::getenv("AMP_DP_B");
    const int want = eb ? std::atoi(eb) : 4;
    for (int b : {8, 4, 2}) {
      if (b > want) continue;
      const size_t sb = multi_smem_bytes(ctx, b);
      if (sb <= (b <= 2 ? 75 : (b >= 8 ? 226 : 113)) * 1024) {
        ctx->multi_b = b;
        ctx->smem_bytes = sb;
        ctx->eval_threads = b >= 8 ? 512 : 256;
        ctx->bp_stride = 0;
        ctx->v_stride = 0;
        break;
      }
    }
  }
  if (ctx->smem_bytes > 227 * 1024) return fail(ctx, AMP_E_UNSUPPORTED, "shared memory budget");
  static const void* const kModes[] = {(const void*)k_dp<kDenseSS>, (const void*)k_dp<kDenseSG>,
                                       (const void*)k_dp<kDenseGS>, (const void*)k_dp<kDenseGG>,
                                       (const void*)k_dp<kSparseS>, (const void*)k_dp<kSparseG>};
  ctx->mode = mode;
  ctx->eval_fn = kModes[mode];
  if (ctx->multi_b) {  // {cell, cellpred} records of every program
    uint64_t cell_total = 0;
    for (const ProgDev& d : ctx->progs_h) cell_total = std::max<uint64_t>(cell_total, d.cell_base + d.n_cells);
    CK(ctx->cellrec.ensure(sizeof(uint2) * (cell_total + 1)));
    if (cell_total) {
      k_pack_cells<<<(int)std::min<uint64_t>((cell_total + 255) / 256, 4096), 256, 0, ctx->stream>>>(
          ctx->cells.as<uint32_t>(), ctx->cellpred.as<uint32_t>(), ctx->cellrec.as<uint2>(), cell_total);
      CK(cudaGetLastError());
    }
  }
  // ---- DP memoisation by signature: key = class | codes ------
  ctx->dedup = false;
  if (ctx->sparse && ctx->n_codes > 0 && !(cfg && (cfg->flags & AMP_FLAG_NO_DEDUP)) &&
      std::getenv("AMP_NO_DEDUP") == nullptr) {
    int cb = 1;
    while ((1 << cb) < ctx->n_codes) ++cb;
    int clsb = 1;
    while ((1ull << clsb) < ctx->classes.size()) ++clsb;
    const int kb = clsb + (ctx->max_pp - 1) * cb;
    // keys wider than 63 bits (|D| = 1024: pp up to 64) are hashed and every
    // item verified against its representative (AMP_WIDE_MEMO=1 forces the
    // hashed keys, AMP_NO_WIDE_MEMO=1 disables them)
    const bool wide = kb > 63 || std::getenv("AMP_WIDE_MEMO") != nullptr;
    if (!wide || std::getenv("AMP_NO_WIDE_MEMO") == nullptr) {
      ctx->dedup = true;
      ctx->wide = wide;
      if (const char* wb = std::getenv("AMP_WIDE_HASH_BITS")) ctx->wide_bits = std::max(1, std::min(64, std::atoi(wb)));
      ctx->code_bits = cb;
      ctx->key_bits = wide ? 64 : kb;
      std::vector<double> pin(ctx->prog_inner_raw.begin(), ctx->prog_inner_raw.end());
      if (pin.empty()) pin.push_back(0.0);
      CK(upload(ctx->prog_inner_d, pin.data(), pin.size()));
      CK(ctx->dd_counters.ensure(2 * sizeof(unsigned long long)));
    }
  }
  // ---- stage-time / parameter range sums (thread K_est), once ------------
  if ((size_t)(L + 1) * (L + 1) * (n_pairs + 1) * sizeof(double) <= ((size_t)256 << 20)) {
    CK(ctx->rsum_t.ensure(sizeof(double) * (size_t)n_pairs * (L + 1) * (L + 1)));
    CK(ctx->rsum_p.ensure(sizeof(double) * (size_t)(L + 1) * (L + 1)));
    k_range_sums<<<n_pairs + 1, 128, 0, ctx->stream>>>(ctx->times.as<double>(), ctx->param.as<double>(),
                                                      L, n_pairs, ctx->rsum_t.as<double>(),
                                                      ctx->rsum_p.as<double>());
    CK(cudaGetLastError());
  }
  // ---- 2-stage DP table (pp == 2 classes x boundary codes), once ----------
  if (ctx->n_codes > 0) {
    EvalParams tp{};
    tp.L = L;
    tp.cls = ctx->cls_d.as<ClassDev>();
    tp.prefix = ctx->prefix.as<double>();
    tp.domain = ctx->domain.as<double>();
    tp.seg = ctx->seg.as<uint16_t>();
    tp.nv_stride = ctx->nv_stride;
    tp.qtab = ctx->qtab.as<double>();
    tp.n_codes = ctx->n_codes;
    tp.n_cls_total = (int)ctx->classes.size();
    const size_t nt = ctx->classes.size() * (size_t)ctx->n_codes;
    CK(ctx->cut2tab.ensure(nt + 16));
    k_cut2_table<<<(int)((nt + 127) / 128), 128, 0, ctx->stream>>>(tp, ctx->cut2tab.as<uint8_t>());
    CK(cudaGetLastError());
  }
  // ---- prefix-shared DP (amp_trie.cuh): static per-class stage facts ------
  ctx->trie = ctx->dedup && ctx->multi_b && !ctx->wide && (1 << ctx->code_bits) <= 16 && std::getenv("AMP_NO_TRIE") == nullptr;
  if (ctx->trie) {
    const int NC = (int)ctx->classes.size(), P1 = ctx->max_pp + 1;
    std::vector<TrieStage> ts((size_t)NC * P1, TrieStage{0, 0, 0, 1, 0});
    std::vector<int32_t> rank(NC, -1), heavy;
    std::vector<uint64_t> v1off(NC, 0);
    uint64_t acc = 0;
    int nq = 1;
    for (int c = 0; c < NC; ++c) {
      if (!is_heavy(ctx, c)) continue;
      const int g = ctx->class_prog[c];
      const ProgDev& pg = ctx->progs_h[g];
      const uint32_t* sh = ctx->stage_h.data() + pg.stage_base;
      rank[c] = (int32_t)heavy.size();
      heavy.push_back(c);
      v1off[c] = acc;
      acc += sh[1] - sh[0];
      nq = std::max(nq, ctx->classes[c].pp - 1);
      for (int j = 1; j <= ctx->classes[c].pp; ++j) {
        TrieStage& t = ts[(size_t)c * P1 + j];
        t.cell0 = pg.cell_base + sh[j - 1];
        t.n = sh[j] - sh[j - 1];
        t.iters = (uint32_t)ctx->prog_stage_inner[(size_t)g * LP + j];
      }
    }
    // tile shapes (K_trie_dp, one smem budget for all stages): wide stages
    // (>= 32 cells) take groups of 4 nodes with per-node smem columns when
    // one group fits kTrieSmem, else a node per thread over the parents'
    // tables; the budget grows (fewer CTAs / SM) only if a one-node tile
    // does not fit.  Each class then takes as many nodes as fit (wide: up to
    // 4 groups; narrow: ~2 items per thread).
    size_t B = kTrieSmem;
    for (int c : heavy)
      for (int j = 2; j <= ctx->classes[c].pp; ++j) {
        TrieStage& t = ts[(size_t)c * P1 + j];
        const int Np = (int)ts[(size_t)c * P1 + j - 1].n;
        t.wide = t.n >= 32 && sizeof(double) * trie_tile_doubles(true, j, 1, Np, L, ctx->n_codes) <= kTrieSmem;
        B = std::max(B, sizeof(double) * trie_tile_doubles(t.wide, j, 1, Np, L, ctx->n_codes));
      }
    if (B > 227 * 1024 || (int)ctx->classes.size() > kTrieMaxCls) ctx->trie = false;
    ctx->tr_smem = (int)B;
    for (int c : heavy)
      for (int j = 2; j <= ctx->classes[c].pp; ++j) {
        TrieStage& t = ts[(size_t)c * P1 + j];
        const int Np = (int)ts[(size_t)c * P1 + j - 1].n;
        int n = t.wide ? 4 : std::min(4096, std::max(1, (2 * kTrieThreads + (int)t.n - 1) / (int)t.n));
        while (n > 1 && sizeof(double) * trie_tile_doubles(t.wide, j, n, Np, L, ctx->n_codes) > B) --n;
        t.tn = (uint32_t)(t.wide ? kTrieNB * n : n);
      }
    if (ctx->trie && heavy.empty()) ctx->trie = false;
    if (ctx->trie) {
      ctx->trie_nq = nq;
      ctx->trie_U = 1 << ctx->code_bits;
      ctx->root_cls_h = heavy;
      CK(upload(ctx->tr_tstage, ts.data(), ts.size()));
      CK(upload(ctx->tr_rank, rank.data(), rank.size()));
      CK(upload(ctx->tr_rcls, heavy.data(), heavy.size()));
      CK(ctx->tr_state.ensure(sizeof(TrieState)));
      CK(ctx->tr_nb.ensure(sizeof(uint32_t) * kTrieMaxD1 * NC));
      CK(ctx->tr_nK.ensure(sizeof(uint32_t) * kTrieMaxD1 * NC));
      CK(ctx->tr_vbase.ensure(sizeof(uint64_t) * kTrieMaxD1 * NC));
      CK(ctx->tr_bbase.ensure(sizeof(uint64_t) * kTrieMaxD1 * NC));
      CK(ctx->tr_rbase.ensure(sizeof(uint64_t) * kTrieMaxD1 * NC));
      CK(ctx->tr_tbase.ensure(sizeof(uint32_t) * kTrieMaxD1 * (NC + 1)));
      CK(ctx->tr_nxc.ensure(sizeof(uint32_t) * kTrieMaxD1 * NC));
      CK(upload(ctx->v1off_d, v1off.data(), v1off.size()));
      CK(ctx->v1g_d.ensure(sizeof(double) * (acc + 1)));
      DevBuf d_heavy;
      CK(upload(d_heavy, heavy.data(), heavy.size()));
      k_trie_v1<<<(int)heavy.size(), 256, 0, ctx->stream>>>(
          ctx->cls_d.as<ClassDev>(), ctx->class_prog_d.as<int32_t>(), ctx->progs_d.as<ProgDev>(),
          ctx->stage_d.as<uint32_t>(), ctx->cells.as<uint32_t>(), ctx->prefix.as<double>(),
          ctx->domain.as<double>(), ctx->nv_stride, L, d_heavy.as<int32_t>(), (int)heavy.size(),
          ctx->v1off_d.as<uint64_t>(), ctx->v1g_d.as<double>());
      CK(cudaGetLastError());
      CK(cudaFuncSetAttribute(k_trie_dp, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->tr_smem));
      const int bsm = (int)(4 * sizeof(unsigned long long) * NC);
      CK(cudaFuncSetAttribute(k_trie_build, cudaFuncAttributeMaxDynamicSharedMemorySize, bsm));
      CK(cudaFuncSetAttribute(k_trie_build_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize, bsm));
      int ob = 0, od = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob, k_trie_build, kBuildThreads, bsm));
      int ob2 = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob2, k_trie_build_sorted, kBuildThreads, bsm));
      ob = std::min(ob, ob2);
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&od, k_trie_dp, kTrieThreads, ctx->tr_smem));
      if (ob < 1 || od < 1) return fail(ctx, AMP_E_UNSUPPORTED, "trie kernels do not fit on an SM");
      ctx->tr_build_grid = std::min(ob, 2) * prop.multiProcessorCount;
      ctx->tr_dp_grid = od * prop.multiProcessorCount;
      CK(ctx->tr_partial.ensure(sizeof(uint32_t) * ctx->tr_build_grid));
      CK(ctx->tr_ghist.ensure(sizeof(uint32_t) * 256 * ctx->tr_build_grid));
      CK(ctx->tr_gpart.ensure(sizeof(uint32_t) * kTrieMaxD1 * ctx->tr_build_grid));
      ctx->tr_sorted = std::getenv("AMP_TRIE_LEVELS") == nullptr;
    }
  }
  if (ctx->multi_b == 2) ctx->eval_fn = (const void*)k_dp_multi<2>;
  if (ctx->multi_b == 4) ctx->eval_fn = (const void*)k_dp_multi<4>;
  if (ctx->multi_b == 8) ctx->eval_fn = (const void*)k_dp_multi<8>;
  CK(cudaFuncSetAttribute(ctx->eval_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)ctx->smem_bytes));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ctx->eval_fn, ctx->eval_threads,
                                                   ctx->smem_bytes));
  if (occ < 1) return fail(ctx, AMP_E_UNSUPPORTED, "evaluate kernel does not fit on an SM");
  int n_ctas = occ * prop.multiProcessorCount;
  ctx->slice_stride = (sparse || ctx->slice_in_smem) ? 0 : (size_t)LP * ctx->max_M;
  // keep per-CTA scratch (backpointers + global slice/table/values) within 16 GiB
  const size_t per_cta = ctx->bp_stride + sizeof(double) * (ctx->slice_stride + ctx->v_stride) +
                         ((sparse || ctx->w_in_smem) ? 0 : w_b);
  const size_t cap = (size_t)16 << 30;
  if (per_cta && (size_t)n_ctas * per_cta > cap) n_ctas = std::max<size_t>(1, cap / per_cta);
  if (ctx->max_ctas_cfg > 0) n_ctas = std::min(n_ctas, ctx->max_ctas_cfg);
  ctx->n_ctas = n_ctas;
  ctx->sms = prop.multiProcessorCount;
  const char* ec = std::getenv("AMP_EST_CTAS_PER_SM");
  ctx->est_ctas = prop.multiProcessorCount * (ec ? std::atoi(ec) : 4);  // 8-warp estimate CTAs per SM (64 regs)
  // chunk size: keep the per-chunk buffers within ~256 MB
  const size_t per_item = sizeof(CandWork) + sizeof(int32_t) * D + sizeof(double) * ctx->max_pp +
                          (ctx->max_pp + 1);
  // (+ the dedup buffers, ~40 B/item) — up to 64 M items (~20 GB of the
  // 180 GB HBM) per chunk, so a 100 M step is two passes: fewer launch tails
  // and dedup over most of the step; AMP_CHUNK overrides (multi-chunk tests)
  const uint64_t chunk_cap = std::getenv("AMP_CHUNK") ? std::strtoull(std::getenv("AMP_CHUNK"), nullptr, 10)
                                                : (64ull << 20);
  ctx->chunk = std::max<uint64_t>(1024, std::min<uint64_t>(chunk_cap, (24ull << 30) / per_item));
  CK(ctx->bp.ensure(ctx->bp_stride * n_ctas + 16));
  if (ctx->slice_stride) CK(ctx->slice.ensure(sizeof(double) * ctx->slice_stride * n_ctas));
  if (!sparse && !ctx->w_in_smem) CK(ctx->wtab.ensure(w_b * n_ctas));
  if (ctx->v_stride) CK(ctx->vbuf.ensure(sizeof(double) * ctx->v_stride * n_ctas));
  CK(ctx->counter.ensure(sizeof(unsigned long long)));
  CK(cudaStreamSynchronize(ctx->stream));  // (the caller's arrays are read before create returns)
  tm.mark("launch shape+scratch");
  return AMP_OK;
}

// Work list: the classes intersecting [begin, end), heaviest first.
// Classes whose candidates go through K_dp (pp <= 2 is solved in K_est).
bool is_heavy(const amp_ctx* ctx, uint64_t c) {
  return ctx->classes[c].pp >= 3 && ctx->class_inner[c] > 0;
}

std::vector<Segment> make_segments(const amp_ctx* ctx, uint64_t begin, uint64_t end) {
  std::vector<std::pair<double, Segment>> v;
  const uint64_t P = ctx->P;
  for (uint64_t c = begin / P; c < ctx->classes.size() && c * P < end; ++c) {
    const uint64_t lo = std::max(begin, c * P), hi = std::min(end, (c + 1) * P);
    if (hi <= lo) continue;
    Segment s{};
    s.first = lo;
    s.count = hi - lo;
    s.out = lo - begin;
    s.p0 = lo - c * P;
    s.cls = (int64_t)c;
    // pp >= 3 classes (the only ones K_dp solves) lead the dispatch order
    const double w = ctx->class_inner[c] + (is_heavy(ctx, c) ? 1e30 : 0.0);
    v.emplace_back(w, s);
  }
  std::stable_sort(v.begin(), v.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<Segment> out;
  uint64_t off = 0;
  for (auto& e : v) {
    e.second.offset = off;
    off += e.second.count;
    out.push_back(e.second);
  }
  return out;
}

// Sum the per-chunk kernel events of the last launch_evaluate (blocks
// until they completed).
void resolve_kernel_times(amp_ctx* ctx) {
  if (!ctx->kev_pending) return;
  double pl = 0, dpm = 0, es = 0;
  for (int c = 0; c + 3 < ctx->kev_used; c += 4) {
    cudaEventSynchronize(ctx->kev[c + 3]);
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, ctx->kev[c], ctx->kev[c + 1]);
    cudaEventElapsedTime(&b, ctx->kev[c + 1], ctx->kev[c + 2]);
    cudaEventElapsedTime(&d, ctx->kev[c + 2], ctx->kev[c + 3]);
    pl += a;
    dpm += b;
    es += d;
  }
  ctx->stats.place_ms = pl;
  ctx->stats.dp_ms = dpm;
  ctx->stats.est_ms = es;
  double st_ms = 0;
  for (int c = 0; c + 1 < ctx->tev_used; c += 2) {
    float a = 0;
    cudaEventElapsedTime(&a, ctx->tev[c], ctx->tev[c + 1]);
    st_ms += a;
  }
  ctx->stats.dp_stage_ms = st_ms;
  ctx->stats.dp_stage_launches = ctx->tev_used / 2;
  ctx->stats.dp_fallback = 0;
  if (ctx->ovf_used > 0) {
    std::vector<uint32_t> o(ctx->ovf_used);
    if (cudaMemcpy(o.data(), ctx->ovf_log.p, sizeof(uint32_t) * o.size(), cudaMemcpyDeviceToHost) ==
        cudaSuccess)
      for (uint32_t v : o) ctx->stats.dp_fallback += v ? 1 : 0;
  }
  ctx->kev_pending = false;
  if (ctx->stats_exec_pending) {  // memoised run: executed DP instances / iterations
    unsigned long long c[2] = {0, 0};
    if (cudaMemcpy(c, ctx->dd_counters.p, sizeof c, cudaMemcpyDeviceToHost) == cudaSuccess) {
      ctx->stats.dp_items = c[0];
      ctx->stats.dp_instances = c[0];
      ctx->stats.dp_inner = (double)c[1];
      ctx->stats.fp64_ops = 7.0 * (double)c[1];
    }
    ctx->stats_exec_pending = false;
  }
}

void account(amp_ctx* ctx, uint64_t begin, uint64_t end, const uint64_t* list, int32_t n,
             const std::vector<Segment>* segs = nullptr) {
  amp_stats& s = ctx->stats;
  s.dp_inner = s.dp_inner_lt = s.dp_cells = 0;
  s.candidates = 0;
  s.dp_instances = 0;
  auto add = [&](uint64_t c, double cnt) {
    s.dp_inner += ctx->class_inner[c] * cnt;
    s.dp_inner_lt += ctx->class_lt[c] * cnt;
    s.dp_cells += ctx->class_cells[c] * cnt;
    if (ctx->class_cells[c] > 0) s.dp_instances += (uint64_t)cnt;
  };
  if (segs) {
    for (const Segment& sg : *segs) {
      add((uint64_t)sg.cls, (double)sg.count);
      s.candidates += sg.count;
    }
  } else if (list) {
    for (int32_t i = 0; i < n; ++i) add(list[i] / ctx->P, 1.0);
    s.candidates = (uint64_t)n;
  } else {
    const uint64_t P = ctx->P;
    for (uint64_t c = begin / P; c < ctx->classes.size() && c * P < end; ++c) {
      const uint64_t lo = std::max(begin, c * P), hi = std::min(end, (c + 1) * P);
      if (hi > lo) add(c, (double)(hi - lo));
    }
    s.candidates = end - begin;
  }
  // FP64 ops of the executed recurrence.  Dense split form:
  // m >= seg: 2 DADD + DSETP; m < seg: DADD, DMUL, 3 DADD, DSETP.  Pruned
  // form: the SURVEY §8(d) count of 7 FP64 ops per inner iteration (t2-dom,
  // max, DMUL, 3 DADD, DSETP) over the executed (unpadded) iterations.
  const double ge = s.dp_inner - s.dp_inner_lt;
  s.fp64_ops = ctx->sparse ? 7.0 * s.dp_inner : 3.0 * ge + 6.0 * s.dp_inner_lt;
  s.bytes = 0;
}

// DP of the chunk's distinct signatures, after the hash insert: the
// signature list (K_sig_init), then the prefix-shared trie DP (amp_trie.cuh)
// or — trie off, or its device capacity exceeded — the signature-mode K_dp
// (k_dp_multi over the keys).  Every count stays on the device: no host
// synchronisation.  Writes the cuts of signature i at ep.repcuts[i].
int run_sig_dp(amp_ctx* ctx, EvalParams& ep, const HashParams& hp) {
  const uint64_t C = std::max<uint64_t>(ep.n_dp, 1);  // signatures <= heavy items
  const int L = ctx->L, NC = (int)ctx->classes.size();
  CK(ctx->dd_rep_key.ensure(sizeof(uint64_t) * C));
  CK(ctx->dd_rep_list.ensure(sizeof(uint32_t) * C));
  CK(ctx->dd_repcuts.ensure((size_t)C * (ctx->max_pp + 1)));
  TrieParams tp{};
  tp.n_sig = hp.n_uniq;
  tp.uniq = hp.uniq;
  tp.tkey = hp.tkey;
  tp.tval = hp.tval;
  tp.key_shift = hp.epoch_shift;
  tp.nq = ctx->max_pp - 1;
  tp.cb = ctx->code_bits;
  tp.U = 1 << ctx->code_bits;
  tp.L = L;
  tp.max_pp = ctx->max_pp;
  tp.n_cls = NC;
  tp.n_roots = (int)ctx->root_cls_h.size();
  tp.sig_key = ctx->dd_rep_key.as<uint64_t>();
  tp.rep_item = ctx->dd_rep_list.as<uint32_t>();
  tp.cls = ctx->cls_d.as<ClassDev>();
  tp.repcuts = ctx->dd_repcuts.as<uint8_t>();
  tp.exec = ep.exec_counters;
  const int g = (int)std::min<uint64_t>((C + 255) / 256, (uint64_t)ctx->sms * 8);
  if (ctx->trie) {
    // capacities of the device-side trie (exceeding one raises ovf and the
    // signature-mode K_dp solves the chunk): nodes per level <= signatures
    // <= heavy items, and <= roots * U^d; parents of depth 1 are the roots
    const uint64_t U = tp.U;
    uint64_t node_b = 0, lvl_b = (uint64_t)tp.n_roots, w = (uint64_t)tp.n_roots;
    for (int d = 1; d <= ctx->trie_nq; ++d) {
      w = std::min<uint64_t>(w * U, C);
      node_b += w;
      lvl_b = std::max(lvl_b, w);
    }
    const uint64_t node_cap = std::min<uint64_t>(node_b, 32ull << 20);
    const uint64_t pres_cap = std::min<uint64_t>(lvl_b, 32ull << 20) * U;
    if (ctx->tr_pres.bytes < pres_cap + 16) {  // marks start clear (and are kept clear); read as 16-byte vectors
      CK(ctx->tr_pres.ensure(pres_cap + 16));
      CK(cudaMemsetAsync(ctx->tr_pres.p, 0, pres_cap + 16, ctx->stream));
    }
    CK(ctx->tr_cid.ensure(sizeof(uint32_t) * pres_cap));
    CK(ctx->tr_npar.ensure(sizeof(uint32_t) * node_cap));
    CK(ctx->tr_ncls.ensure(sizeof(uint16_t) * node_cap));
    CK(ctx->tr_ncode.ensure(node_cap));
    // value tables of every depth (256 M doubles; AMP_TRIE_VCAP shrinks them
    // to exercise the capacity fallback in the tests), argmins, run counters
    const char* vc = std::getenv("AMP_TRIE_VCAP");
    const uint64_t vcap = vc ? std::strtoull(vc, nullptr, 10) : (256ull << 20), bpcap = 1ull << 30;
    const uint64_t run_cap = node_cap, tile_cap = node_cap + (4ull << 20);
    CK(ctx->tr_v0.ensure(sizeof(double) * std::max<uint64_t>(vcap, 1)));
    CK(ctx->tr_bp.ensure(bpcap));
    CK(ctx->tr_done.ensure(sizeof(uint32_t) * run_cap));
    CK(ctx->tr_tiles.ensure(sizeof(TrieTile) * tile_cap));
    CK(ctx->dd_nid.ensure(sizeof(uint32_t) * C));
    tp.nid = ctx->dd_nid.as<uint32_t>();
    tp.root_rank = ctx->tr_rank.as<int32_t>();
    tp.root_cls = ctx->tr_rcls.as<int32_t>();
    tp.st = ctx->tr_state.as<TrieState>();
    tp.pres = ctx->tr_pres.as<uint8_t>();
    tp.cid = ctx->tr_cid.as<uint32_t>();
    tp.pres_cap = pres_cap;
    tp.partial = ctx->tr_partial.as<uint32_t>();
    tp.smem_bytes = ctx->tr_smem;
    if (ctx->tr_sorted) {
      CK(ctx->tr_sortk.ensure(sizeof(uint64_t) * 2 * C));
      CK(ctx->tr_sortv.ensure(sizeof(uint32_t) * 2 * C));
      tp.sk[0] = ctx->tr_sortk.as<uint64_t>();
      tp.sk[1] = tp.sk[0] + C;
      tp.sv[0] = ctx->tr_sortv.as<uint32_t>();
      tp.sv[1] = tp.sv[0] + C;
      tp.ghist = ctx->tr_ghist.as<uint32_t>();
      tp.gpart = ctx->tr_gpart.as<uint32_t>();
      int clsb = 0;
      while ((1 << clsb) < NC) ++clsb;
      tp.kbits = tp.nq * tp.cb + clsb;
    }
    tp.npar = ctx->tr_npar.as<uint32_t>();
    tp.ncls = ctx->tr_ncls.as<uint16_t>();
    tp.ncode = ctx->tr_ncode.as<uint8_t>();
    tp.node_cap = node_cap;
    tp.nb = ctx->tr_nb.as<uint32_t>();
    tp.nK = ctx->tr_nK.as<uint32_t>();
    tp.nxc = ctx->tr_nxc.as<uint32_t>();
    tp.tbase = ctx->tr_tbase.as<uint32_t>();
    tp.vbase = ctx->tr_vbase.as<uint64_t>();
    tp.bbase = ctx->tr_bbase.as<uint64_t>();
    tp.rbase = ctx->tr_rbase.as<uint64_t>();
    tp.tstage = ctx->tr_tstage.as<TrieStage>();
    tp.varena = ctx->tr_v0.as<double>();
    tp.vcap = vcap;
    tp.bparena = ctx->tr_bp.as<uint8_t>();
    tp.bpcap = bpcap;
    tp.done = ctx->tr_done.as<uint32_t>();
    tp.run_cap = run_cap;
    tp.tiles = ctx->tr_tiles.as<TrieTile>();
    tp.tile_cap = tile_cap;
    tp.cellrec = ctx->cellrec.as<uint2>();
    tp.preds = ctx->preds.as<uint16_t>();
    tp.progs = ctx->progs_d.as<ProgDev>();
    tp.class_prog = ctx->class_prog_d.as<int32_t>();
    tp.prefix = ctx->prefix.as<double>();
    tp.domain = ctx->domain.as<double>();
    tp.nv_stride = ctx->nv_stride;
    tp.n_codes = ctx->n_codes;
    tp.qtab = ctx->qtab.as<double>();
    tp.v1g = ctx->v1g_d.as<double>();
    tp.v1off = ctx->v1off_d.as<uint64_t>();
    CK(cudaMemsetAsync(ctx->tr_state.p, 0, sizeof(TrieState), ctx->stream));
    CK(cudaMemsetAsync(ctx->tr_nb.p, 0, sizeof(uint32_t) * kTrieMaxD1 * NC, ctx->stream));
    CK(cudaMemsetAsync(ctx->tr_nK.p, 0, sizeof(uint32_t) * kTrieMaxD1 * NC, ctx->stream));
    void* args[] = {&tp};
    CK(cudaLaunchCooperativeKernel(ctx->tr_sorted ? (const void*)k_trie_build_sorted : (const void*)k_trie_build,
                                   dim3(ctx->tr_build_grid), dim3(kBuildThreads),
                                   args, 4 * sizeof(unsigned long long) * NC, ctx->stream));
    DBG_SYNC("k_trie_build");
    while ((int)ctx->tev.size() < ctx->tev_used + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ctx->tev.push_back(e);
    }
    CK(cudaEventRecord(ctx->tev[ctx->tev_used++], ctx->stream));
    k_trie_dp<<<ctx->tr_dp_grid, kTrieThreads, ctx->tr_smem, ctx->stream>>>(tp);
    CK(cudaEventRecord(ctx->tev[ctx->tev_used++], ctx->stream));
    CK(cudaGetLastError());
    DBG_SYNC("k_trie_dp");
    k_trie_back<<<g, 256, 0, ctx->stream>>>(tp);
    CK(cudaGetLastError());
    DBG_SYNC("k_trie_back");
    ctx->launches += 3;
    if ((size_t)(ctx->ovf_used + 1) * sizeof(uint32_t) > ctx->ovf_log.bytes) {
      // (grows between runs only: a run's chunk count is bounded by the first)
      CK(ctx->ovf_log.ensure(sizeof(uint32_t) * std::max(64, 2 * (ctx->ovf_used + 1))));
    }
    CK(cudaMemcpyAsync(ctx->ovf_log.as<uint32_t>() + ctx->ovf_used,
                       reinterpret_cast<const char*>(tp.st) + offsetof(TrieState, ovf), sizeof(uint32_t),
                       cudaMemcpyDeviceToDevice, ctx->stream));
    ++ctx->ovf_used;
  } else {
    k_sig_list<<<g, 256, 0, ctx->stream>>>(tp);
    CK(cudaGetLastError());
    DBG_SYNC("k_sig_list");
    ctx->launches += 1;
  }
  // signature-mode K_dp: the whole DP when the trie is off; with the trie
  // only if its capacity was exceeded on the device (it exits otherwise)
  EvalParams es = ep;
  // (hashed keys, or the per-candidate K_dp of programs too large for
  // k_dp_multi: class and codes of each signature's representative item)
  const bool by_rep = ctx->wide || !ctx->multi_b;
  es.sig_keys = by_rep ? nullptr : ctx->dd_rep_key.as<uint64_t>();
  es.sig_guard = ctx->trie ? reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(tp.st) +
                                                               offsetof(TrieState, ovf))
                          : nullptr;
  es.n_rep = reinterpret_cast<const uint64_t*>(hp.n_uniq);
  es.rep_list = by_rep ? ctx->dd_rep_list.as<uint32_t>() : nullptr;
  es.repcuts = ctx->dd_repcuts.as<uint8_t>();
  es.sig_code_bits = ctx->code_bits;
  if (ctx->gang_on && ctx->eval_fn == (const void*)k_dp<kSparseG>) {
    CK(ctx->gang_hdr.ensure(4 * sizeof(uint32_t)));
    CK(ctx->gang_slot.ensure(sizeof(uint32_t) * C));
    CK(ctx->gang_off.ensure(sizeof(uint32_t) * (C + 1)));
    CK(ctx->gang_sync.ensure(2 * sizeof(uint32_t) * C));
    es.gang_hdr = ctx->gang_hdr.as<uint32_t>();
    es.gang_slot = ctx->gang_slot.as<uint32_t>();
    es.gang_off = ctx->gang_off.as<uint32_t>();
    es.gang_sync = ctx->gang_sync.as<uint32_t>();
    es.gang_min = ctx->gang_min;
    es.gang_unit = ctx->gang_unit;
    es.gang_max = std::min(ctx->gang_max, ctx->n_ctas);  // a gang's parts must be co-resident
    k_gang_plan<<<1, 1024, 0, ctx->stream>>>(es);
    CK(cudaGetLastError());
    DBG_SYNC("k_gang_plan");
    ctx->launches += 1;
  }
  void* args[] = {&es};
  if (es.gang_hdr)  // a gang's parts wait on each other: co-residency guaranteed by a cooperative launch
    CK(cudaLaunchCooperativeKernel(ctx->eval_fn, dim3(ctx->n_ctas), dim3(ctx->eval_threads), args,
                                   ctx->smem_bytes, ctx->stream));
  else
    CK(cudaLaunchKernel(ctx->eval_fn, dim3(ctx->n_ctas), dim3(ctx->eval_threads), args, ctx->smem_bytes,
                        ctx->stream));
  CK(cudaGetLastError());
  DBG_SYNC("k_dp_multi (signatures)");
  ctx->launches += 1;
  return AMP_OK;
}

// Launch K1+K2 over either a segment list or an explicit index list.
// Evaluate n_work items (segment list or explicit index list) as a pipeline
// of chunks: K_place -> K_dp -> K_est per chunk (amp_pipeline.cuh).  CTA
// top-k lists of K_est persist across chunks in ctx->cta_topk.
int launch_evaluate(amp_ctx* ctx, const std::vector<Segment>* segs, const uint64_t* d_list,
                    uint64_t n_work, int32_t k, bool want_all, bool want_details,
                    bool want_place, const uint8_t* d_given_cuts = nullptr,
                    bool want_sim = false, const int32_t* d_given_place = nullptr) {
  EvalParams ep{};
  ep.L = ctx->L;
  ep.D = ctx->D;
  ep.gbs = ctx->gbs;
  ep.max_pp = ctx->max_pp;
  ep.P = ctx->P;
  ep.seed = ctx->seed;
  ep.param = ctx->param.as<double>();
  ep.act = ctx->act.as<double>();
  ep.bw = ctx->bw.as<double>();
  ep.base_order = ctx->base_order.as<int32_t>();
  ep.has_ceiling = ctx->has_ceiling;
  ep.n_pairs = static_cast<int32_t>(ctx->pairs.size());
  ep.ceiling = ctx->ceiling;
  ep.bpp = ctx->bpp;
  ep.cls = ctx->cls_d.as<ClassDev>();
  ep.pairs = ctx->pairs_d.as<PairDev>();
  ep.times = ctx->times.as<double>();
  ep.prefix = ctx->prefix.as<double>();
  ep.domain = ctx->domain.as<double>();
  ep.seg = ctx->seg.as<uint16_t>();
  ep.nv_stride = ctx->nv_stride;
  ep.slice_in_smem = ctx->slice_in_smem;
  ep.w_in_smem = ctx->w_in_smem;
  ep.wtab = ctx->wtab.as<WEnt>();
  if (segs) {
    CK(upload(ctx->segs, segs->data(), segs->size()));
    ep.segs = ctx->segs.as<Segment>();
    ep.n_segs = static_cast<int32_t>(segs->size());
  }
  ep.n_work = n_work;
  ep.index_list = d_list;
  ep.given_place = d_given_place;
  ep.counter = ctx->counter.as<unsigned long long>();
  ep.bp = ctx->bp.as<uint8_t>();
  ep.bp_stride = ctx->bp_stride;
  ep.slice = ctx->slice.as<double>();
  ep.slice_stride = ctx->slice_stride;
  if (want_all) {
    CK(ctx->o_all.ensure(sizeof(amp_record) * n_work));
    ep.all = ctx->o_all.as<amp_record>();
  }
  if (want_details) {
    CK(ctx->o_cuts.ensure(sizeof(int32_t) * n_work * (ctx->max_pp + 1)));
    CK(ctx->o_stage.ensure(sizeof(double) * n_work * ctx->max_pp));
    CK(ctx->o_edge.ensure(sizeof(double) * n_work * ctx->max_pp));
    ep.all_cuts = ctx->o_cuts.as<int32_t>();
    ep.all_stage = ctx->o_stage.as<double>();
    ep.all_edge = ctx->o_edge.as<double>();
  }
  if (want_place) {
    CK(ctx->o_place.ensure(sizeof(int32_t) * n_work * ctx->D));
    ep.all_place = ctx->o_place.as<int32_t>();
  }
  if (want_sim) {
    CK(ctx->o_sim.ensure(sizeof(double) * n_work));
    ep.all_sim = ctx->o_sim.as<double>();
    if (ctx->max_pp > 32) {  // per-warp ready-time array of the pp > 32 path
      CK(ctx->simbuf.ensure(sizeof(double) * (size_t)ctx->est_ctas * kEstWarps * ctx->gbs));
      ep.simbuf = ctx->simbuf.as<double>();
    }
  }
  const int kk = std::max(1, k);
  CK(ctx->cta_topk.ensure(sizeof(amp_record) * (size_t)kk * ctx->est_ctas));
  ep.cta_topk = ctx->cta_topk.as<amp_record>();
  ep.k = kk;
  ep.max_M = ctx->max_M;
  ep.progs = ctx->progs_d.as<ProgDev>();
  ep.class_prog = ctx->class_prog_d.as<int32_t>();
  ep.cells = ctx->cells.as<uint32_t>();
  ep.cellpred = ctx->cellpred.as<uint32_t>();
  ep.preds = ctx->preds.as<uint16_t>();
  ep.stage = ctx->stage_d.as<uint32_t>();
  ep.vbuf = ctx->vbuf.as<double>();
  ep.max_cells = ctx->max_cells;
  ep.max_prog_cells = ctx->max_prog_cells;
  ep.max_n1 = ctx->max_n1;
  ep.max_v = ctx->max_v;
  ep.max_rest = ctx->max_rest;
  // chunk buffers (grown on demand up to ctx->chunk items)
  const uint64_t C = std::min<uint64_t>(ctx->chunk, std::max<uint64_t>(n_work, 1));
  CK(ctx->c_work.ensure(sizeof(CandWork) * C));
  CK(ctx->c_place.ensure(sizeof(int32_t) * C * ctx->D));
  CK(ctx->c_bwq.ensure(sizeof(double) * C * ctx->max_pp));
  CK(ctx->c_cuts.ensure((size_t)C * (ctx->max_pp + 1)));
  ep.work = ctx->c_work.as<CandWork>();
  ep.placeb = ctx->c_place.as<int32_t>();
  ep.bwqb = ctx->c_bwq.as<double>();
  ep.cutsb = ctx->c_cuts.as<uint8_t>();
  CK(ctx->c_bwc.ensure((size_t)C * ctx->max_pp));
  ep.bwcb = ctx->c_bwc.as<uint8_t>();
  ep.n_codes = ctx->n_codes;
  ep.bwcode = ctx->n_codes ? ctx->bwcode.as<uint8_t>() : nullptr;
  ep.bwval = ctx->bwval.as<double>();
  ep.qtab = ctx->n_codes ? ctx->qtab.as<double>() : nullptr;
  ep.cellrec = ctx->cellrec.as<uint2>();
  ep.cut2tab = ctx->n_codes ? ctx->cut2tab.as<uint8_t>() : nullptr;
  ep.rsum_t = ctx->rsum_t.as<double>();
  ep.bw_positive = ctx->n_codes > 0 && ctx->bw_positive;
  ep.rsum_p = ctx->rsum_p.as<double>();
  ep.n_cls_total = (int)ctx->classes.size();
  if (ctx->dedup && !d_given_cuts) {
    CK(ctx->dd_rep_of.ensure(sizeof(uint32_t) * C));
    CK(cudaMemsetAsync(ctx->dd_counters.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
    ep.exec_counters = ctx->dd_counters.as<unsigned long long>();
    ep.prog_inner = ctx->prog_inner_d.as<double>();
  }
  ctx->stats_exec_pending = ctx->dedup && !d_given_cuts;
  // items of pp >= 3 classes lead the dispatch order of a segment list
  uint64_t n_heavy = n_work;
  if (segs) {
    n_heavy = 0;
    for (const Segment& sg : *segs) {
      if (!is_heavy(ctx, (uint64_t)sg.cls)) break;
      n_heavy += sg.count;
    }
  }
  const int D = ctx->D, mp = ctx->max_pp;
  const size_t place_smem = (D <= 32 ? (sizeof(double) + 1) * D * D : 0) + sizeof(int) * 32 * 8;
  if (ctx->n_nodes > 0) {
    ep.node_of = ctx->node_of.as<int32_t>();
    ep.nodebw = ctx->nodebw.as<double>();
    ep.n_nodes = ctx->n_nodes;
    ep.node_words = (ctx->n_nodes + 31) / 32;
  }
  size_t est_smem = (ep.nodebw ? sizeof(unsigned) * 2 * ep.node_words * kEstWarps : 0) +
                    (D <= 32 ? sizeof(double) * D * D : 0) +
                    sizeof(double) * 2 * mp * kEstWarps + sizeof(int) * (mp + 2) * kEstWarps;
  est_smem = ((est_smem + 15) & ~size_t(15)) + sizeof(EstWarp) * kEstWarps +
             (kk <= 32 ? sizeof(amp_record) * kk : 0);
  if (est_smem > 48 * 1024)
    CK(cudaFuncSetAttribute(k_est, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)est_smem));
  ctx->stats.dp_items = 0;
  ctx->stats.dp_launches = 0;
  ctx->tev_used = 0;
  ctx->ovf_used = 0;
  ctx->stats.dp_group = ctx->multi_b;
  // thread-per-candidate K_place / K_est (amp_thread.cuh): |D| <= 16 with
  // coded bandwidths; AMP_NO_THREAD=1 keeps the warp kernels
  const bool thread_mode = ctx->D <= kThreadMaxD && ctx->n_codes > 0 && ctx->max_pp <= kThreadMaxD &&
                           std::getenv("AMP_NO_THREAD") == nullptr;
  // thread-mode traffic trims: packed placements (8 B instead of |D| ints)
  // when K_est_t reads them; bandwidth values only for kernels without the
  // edge tables
  const bool est_thread = thread_mode && !want_sim && kk <= 32;
  ep.need_place_rows = !est_thread;
  // K_est_t places the pp <= 2 tail of a segment list itself (never in K_dp)
  ep.fuse_light = est_thread && segs != nullptr && d_given_cuts == nullptr &&
                  std::getenv("AMP_NO_FUSE") == nullptr;
  ep.need_bwq = !(thread_mode && ctx->multi_b);
  ep.placep = nullptr;
  ep.sigkey = nullptr;
  if (thread_mode) {
    CK(ctx->c_placep.ensure(sizeof(uint64_t) * C));
    ep.placep = ctx->c_placep.as<uint64_t>();
    if (ctx->dedup && !ctx->wide && !d_given_cuts) {  // K_place_t writes the DP signature keys
      CK(ctx->dd_sigkey.ensure(sizeof(uint64_t) * C));
      ep.sigkey = ctx->dd_sigkey.as<uint64_t>();
      ep.sig_code_bits = ctx->code_bits;
    }
  }
  // the placement table: the shuffle of placement p is the same for every
  // class, so it is computed once per context (P placements) and read by
  // K_place_t / K_est_t (AMP_NO_PERM_TAB=1: every candidate shuffles)
  ep.perm_tab = nullptr;
  ep.perm_n = 0;
  if (thread_mode && ctx->D == 16 && !d_given_place && ctx->P > 1 && ctx->P <= (64ull << 20) &&
      std::getenv("AMP_NO_PERM_TAB") == nullptr) {
    if (ctx->perm_n != ctx->P) {
      CK(ctx->perm_tab.ensure(sizeof(uint64_t) * ctx->P));
      const int gp = (int)std::min<uint64_t>((ctx->P + 255) / 256, (uint64_t)ctx->sms * 8);
      k_perm_table<<<gp, 256, 0, ctx->stream>>>(ep, ctx->perm_tab.as<uint64_t>(), ctx->P);
      CK(cudaGetLastError());
      DBG_SYNC("k_perm_table");
      ctx->launches += 1;
      ctx->perm_n = ctx->P;
    }
    ep.perm_tab = ctx->perm_tab.as<uint64_t>();
    ep.perm_n = ctx->perm_n;
  }
  // unrolled shape kernels in K_est_t: |D| == 16, every class a full
  // pp * dp * tmp == 16 shape, positive coded bandwidths, the range / 2-stage
  // tables, records only (AMP_NO_SHAPE=1 keeps the generic body)
  bool shape16 = thread_mode && ctx->D == 16 && ep.bw_positive && std::getenv("AMP_NO_SHAPE") == nullptr &&
                 (ctx->P == 1 || ep.perm_tab != nullptr) && !d_given_place;
  for (const auto& c : ctx->classes) shape16 = shape16 && c.pp * c.dp * c.tmp == 16;
  ep.est_fast = shape16 && est_thread && ep.cut2tab && ep.rsum_t && !ep.all_cuts && !ep.all_stage &&
                !ep.all_edge && !ep.all_place && !d_given_cuts && !ctx->wide;
  // the code table of every (shape, placement): the shape kernels need it;
  // codes < 16 (4 bits each), at most 4 GB (else the generic bodies run)
  ep.ctab = nullptr;
  if (ep.est_fast) {
    const uint64_t tb = sizeof(ulonglong2) * (uint64_t)ctx->row_shape.size() * ctx->P;
    if (ctx->n_codes <= 16 && tb <= (4ull << 30) && !ctx->row_shape.empty() &&
        std::getenv("AMP_NO_CTAB") == nullptr) {
      if (ctx->ctab_P != ctx->P) {
        CK(ctx->ctab.ensure(tb));
        const uint64_t n = (uint64_t)ctx->row_shape.size() * ctx->P;
        const int gc = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sms * 8);
        k_code_table<<<gc, 256, 0, ctx->stream>>>(ep, ctx->row_shape_d.as<int32_t>(), (int)ctx->row_shape.size(),
                                                   ctx->ctab.as<ulonglong2>());
        CK(cudaGetLastError());
        DBG_SYNC("k_code_table");
        ctx->launches += 1;
        ctx->ctab_P = ctx->P;
      }
      ep.ctab = ctx->ctab.as<ulonglong2>();
      ep.placep = nullptr;  // (K_est reads the codes, not the placement)
    } else {
      ep.est_fast = false;
    }
  }
  // the boundary codes are read by K_dp without the trie, the sort dedup
  // path and K_est's pp == 2 items placed by K_place; with the hash dedup on
  // K_place's signature keys, the trie and the fused light path, nothing
  ep.need_bwcb = !(ep.sigkey && ctx->dedup && ep.fuse_light);
  // ---- light tail on the aux stream -------------------------------------
  // The pp <= 2 items [n_heavy, n_work) of a segment run need no K_place /
  // K_dp (K_est places them itself), so their K_est runs on a second stream
  // with its own CTA lists (after the main ones in cta_topk, merged with
  // them) and a smaller grid, overlapping the heavy items' latency-bound
  // K_dp.  Opt-in (AMP_OVERLAP=1): measured on the bench sweep it does not
  // pay — K_place slows 2.1 -> 4.9 ms sharing the SMs, step 8.13 -> 8.32 ms.
  const char* ax = std::getenv("AMP_AUX_CTAS_PER_SM");
  const int aux_ctas = std::min(kMergeMaxLists - ctx->est_ctas, ctx->sms * (ax ? std::atoi(ax) : 2));
  const bool overlap = ep.est_fast && ep.fuse_light && segs && n_heavy > 0 && n_heavy < n_work &&
                       aux_ctas >= 1 && std::getenv("AMP_OVERLAP") != nullptr;
  const uint64_t n_main = overlap ? n_heavy : n_work;
  const int n_aux_chunks = overlap ? (int)((n_work - n_heavy + C - 1) / C) : 0;
  ctx->n_topk_lists = ctx->est_ctas + (overlap ? aux_ctas : 0);
  if (overlap) {
    CK(ctx->cta_topk.ensure(sizeof(amp_record) * (size_t)kk * ctx->n_topk_lists));
    ep.cta_topk = ctx->cta_topk.as<amp_record>();
    if (!ctx->aux) {
      CK(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->aux_start, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->aux_done, cudaEventDisableTiming));
    }
  }
  const int n_chunks = (int)((n_main + C - 1) / C) + n_aux_chunks;
  while ((int)ctx->kev.size() < 4 * n_chunks) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->kev.push_back(e);
  }
  ctx->kev_used = 4 * n_chunks;
  ctx->kev_pending = true;
  // signature hash table of a chunk (amp_dedup.cuh): sized for every heavy
  // item at load <= 1/2, so every insert finds its slot (no overflow, no
  // host check); entries carry an epoch tag above the key bits, so the table
  // is cleared only when it is (re)allocated or the tag wraps.  Only the
  // slots of distinct keys are touched (L2-resident), whatever the size.
  auto prepare_hash = [&](HashParams& hp) -> int {
    uint64_t T = 1024;
    while (T < 2 * ep.n_dp) T <<= 1;
    T = std::max<uint64_t>(T, ctx->hash_T);  // keep a larger table (and its epoch)
    const bool grown = ctx->dd_tkey.bytes < sizeof(uint64_t) * T;
    CK(ctx->dd_tkey.ensure(sizeof(uint64_t) * T));
    CK(ctx->dd_tval.ensure(sizeof(uint32_t) * T));
    CK(ctx->dd_slot.ensure(sizeof(uint32_t) * C));
    CK(ctx->dd_uniq.ensure(sizeof(uint32_t) * C));
    CK(ctx->dd_nuniq.ensure(2 * sizeof(unsigned long long)));
    const int esh = 64 - ctx->key_bits >= 8 ? ctx->key_bits : 64;
    if (esh >= 64) {
      CK(cudaMemsetAsync(ctx->dd_tkey.p, 0xff, sizeof(uint64_t) * T, ctx->stream));
    } else {
      const uint64_t max_epoch = (1ull << (64 - esh)) - 1;
      if (grown || ctx->hash_T != T || ctx->hash_esh != esh || ctx->hash_epoch >= max_epoch) {
        CK(cudaMemsetAsync(ctx->dd_tkey.p, 0, sizeof(uint64_t) * T, ctx->stream));
        ctx->hash_epoch = 0;
      }
      ++ctx->hash_epoch;
    }
    ctx->hash_T = T;
    ctx->hash_esh = esh;
    CK(cudaMemsetAsync(ctx->dd_nuniq.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
    hp = HashParams{};
    hp.work = ep.work;
    hp.cls = ep.cls;
    hp.bwcb = ep.bwcb;
    hp.n = ep.n_dp;
    hp.max_pp = ctx->max_pp;
    hp.code_bits = ctx->code_bits;
    hp.wide = ctx->wide ? ctx->wide_bits : 0;
    hp.mask = T - 1;
    hp.max_probe = T;
    hp.epoch = ctx->hash_epoch;
    hp.epoch_shift = esh;
    hp.sigkey = ep.sigkey;
    hp.tkey = ctx->dd_tkey.as<unsigned long long>();
    hp.tval = ctx->dd_tval.as<uint32_t>();
    hp.slot_of = ctx->dd_slot.as<uint32_t>();
    hp.uniq = ctx->dd_uniq.as<uint32_t>();
    hp.n_uniq = ctx->dd_nuniq.as<unsigned long long>();
    return AMP_OK;
  };
  // K_place_t inserts the keys itself (no key round trip, one launch less)
  const bool fuse_hash_ok = thread_mode && ep.sigkey && ctx->dedup && !d_given_cuts &&
                            std::getenv("AMP_NO_FUSE_HASH") == nullptr;
  HashParams fused_hp{};
  ep.skip_work = ep.est_fast && ctx->dedup && ctx->multi_b && fuse_hash_ok && ep.fuse_light &&
                 std::getenv("AMP_KEEP_WORK") == nullptr;
  if (overlap) {
    CK(cudaEventRecord(ctx->aux_start, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->aux, ctx->aux_start, 0));
    EvalParams ea = ep;
    ea.cta_topk = ep.cta_topk + (size_t)kk * ctx->est_ctas;
    ea.n_dp = 0;
    ea.fuse_hash = 0;
    int a = 0;
    for (uint64_t t0 = n_heavy; t0 < n_work; t0 += C, ++a) {
      cudaEvent_t* ev = &ctx->kev[4 * ((n_main + C - 1) / C + a)];
      CK(cudaEventRecord(ev[0], ctx->aux));
      CK(cudaEventRecord(ev[1], ctx->aux));
      CK(cudaEventRecord(ev[2], ctx->aux));
      ea.t0 = t0;
      ea.n_chunk = std::min<uint64_t>(C, n_work - t0);
      ea.first_chunk = t0 == n_heavy;
      k_est_t<16, true><<<aux_ctas, kEstTWarps * 32, 0, ctx->aux>>>(ea);
      DBG_SYNC("k_est_t");
      CK(cudaGetLastError());
      CK(cudaEventRecord(ev[3], ctx->aux));
      ctx->launches += 1;
    }
    CK(cudaEventRecord(ctx->aux_done, ctx->aux));
  }
  for (uint64_t t0 = 0; t0 < n_main; t0 += C) {
    cudaEvent_t* ev = &ctx->kev[4 * (t0 / C)];
    CK(cudaEventRecord(ev[0], ctx->stream));
    ep.t0 = t0;
    ep.n_chunk = std::min<uint64_t>(C, n_main - t0);
    ep.n_dp = n_heavy > t0 ? std::min<uint64_t>(ep.n_chunk, n_heavy - t0) : 0;
    ep.cuts_given = d_given_cuts != nullptr;
    if (d_given_cuts) {  // estimate only: the caller's cuts replace K_dp
      ep.n_dp = 0;
      CK(cudaMemcpyAsync(ctx->c_cuts.p, d_given_cuts + t0 * (ctx->max_pp + 1),
                         ep.n_chunk * (ctx->max_pp + 1), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ep.first_chunk = t0 == 0;
    ep.fuse_hash = 0;
    if (fuse_hash_ok && ep.n_dp > 0) {
      const int rc = prepare_hash(fused_hp);
      if (rc != AMP_OK) return rc;
      ep.fuse_hash = 1;
      ep.h_tkey = fused_hp.tkey;
      ep.h_tval = fused_hp.tval;
      ep.h_slot_of = fused_hp.slot_of;
      ep.h_uniq = fused_hp.uniq;
      ep.h_nuniq = fused_hp.n_uniq;
      ep.h_mask = fused_hp.mask;
      ep.h_max_probe = fused_hp.max_probe;
      ep.h_epoch = fused_hp.epoch;
      ep.h_eshift = fused_hp.epoch_shift;
    }
    const uint64_t warps = ep.n_chunk;
    const int place_grid = (int)std::min<uint64_t>((warps + 7) / 8, (uint64_t)ctx->sms * 16);
    if (thread_mode) {
      const int tg = (int)std::min<uint64_t>((ep.n_chunk + 255) / 256, (uint64_t)ctx->sms * 16);
      if (shape16)
        k_place_t<16, true><<<tg, 256, 0, ctx->stream>>>(ep);
      else if (ctx->D == 16)
        k_place_t<16><<<tg, 256, 0, ctx->stream>>>(ep);
      else
        k_place_t<0><<<tg, 256, 0, ctx->stream>>>(ep);
      DBG_SYNC("k_place_t");
    } else {
      k_place<<<place_grid, 256, place_smem, ctx->stream>>>(ep);
      DBG_SYNC("k_place");
    }
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned long long), ctx->stream));
    CK(cudaEventRecord(ev[1], ctx->stream));
    ep.rep_list = nullptr;
    ep.rep_of = nullptr;
    ep.memo_bad = nullptr;
    ep.n_rep = nullptr;
    ep.repcuts = nullptr;
    ep.run_slot = nullptr;
    ep.run_of_slot = nullptr;
    ep.run_pipe = nullptr;
    bool skip_dp = false;
    if (ctx->dedup && !d_given_cuts && ep.n_dp > 0) {
      // ---- memoisation: one DP per distinct signature (amp_dedup.cuh) ------
      const int g = (int)std::min<uint64_t>((ep.n_dp + 255) / 256, (uint64_t)ctx->sms * 8);
      HashParams hp{};
      if (ep.fuse_hash) {
        hp = fused_hp;  // table prepared before K_place_t, which inserted the keys
      } else {
        const int rc = prepare_hash(hp);
        if (rc != AMP_OK) return rc;
        k_hash_insert<<<g, 256, 0, ctx->stream>>>(hp);
        DBG_SYNC("k_hash_insert");
        ctx->launches += 1;
      }
      const int rc = run_sig_dp(ctx, ep, hp);
      if (rc != AMP_OK) return rc;
      hp.rep_of = ctx->dd_rep_of.as<uint32_t>();
      // K_est finds an item's signature through its hash slot (tval: slot ->
      // signature after K_sig_init); the generic bodies read rep_of
      if (ep.est_fast && std::getenv("AMP_NO_RUN_SLOT") == nullptr) {
        ep.run_slot = hp.slot_of;
        ep.run_of_slot = hp.tval;
      } else {
        k_hash_scatter<<<g, 256, 0, ctx->stream>>>(hp);
        DBG_SYNC("k_hash_scatter");
        ctx->launches += 1;
        ep.rep_of = hp.rep_of;
      }
      if (ctx->wide) {
        // hashed keys: verify every item against its representative; on a
        // collision (*bad) a guarded per-item K_dp writes every item's cuts
        // and K_est reads those instead
        CK(ctx->dd_bad.ensure(sizeof(uint32_t)));
        CK(cudaMemsetAsync(ctx->dd_bad.p, 0, sizeof(uint32_t), ctx->stream));
        k_hash_verify<<<g, 256, 0, ctx->stream>>>(hp, ctx->dd_rep_list.as<uint32_t>(), ctx->dd_bad.as<uint32_t>());
        DBG_SYNC("k_hash_verify");
        CK(cudaGetLastError());
        EvalParams eg = ep;
        eg.sig_guard = ctx->dd_bad.as<uint32_t>();
        eg.sig_keys = nullptr;
        eg.rep_list = nullptr;
        eg.n_rep = nullptr;
        eg.repcuts = nullptr;
        eg.exec_counters = nullptr;
        CK(cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned long long), ctx->stream));
        void* gargs[] = {&eg};
        CK(cudaLaunchKernel(ctx->eval_fn, dim3(ctx->n_ctas), dim3(ctx->eval_threads), gargs, ctx->smem_bytes,
                            ctx->stream));
        CK(cudaGetLastError());
        DBG_SYNC("k_dp_multi (collision fallback)");
        ctx->launches += 2;
        ep.memo_bad = ctx->dd_bad.as<uint32_t>();
      }
      ep.repcuts = ctx->dd_repcuts.as<uint8_t>();
      if (ep.est_fast && std::getenv("AMP_NO_RUN_PIPE") == nullptr) {
        // dp == 1 classes: the whole estimate per signature, by hash slot when
        // K_est looks signatures up by slot
        const bool by_slot = ep.run_slot != nullptr;
        CK(ctx->dd_runpipe.ensure(sizeof(double) * (by_slot ? ctx->hash_T : ep.n_dp)));
        k_run_pipe<<<g, 256, 0, ctx->stream>>>(ep, ctx->dd_rep_key.as<uint64_t>(), hp.n_uniq,
                                                 ctx->dd_runpipe.as<double>(),
                                                 by_slot ? hp.uniq : nullptr);
        DBG_SYNC("k_run_pipe");
        CK(cudaGetLastError());
        ctx->launches += 1;
        ep.run_pipe = ctx->dd_runpipe.as<double>();
      }
      skip_dp = true;  // K_dp's work is done (K_est reads the cuts by signature)
    }
    ctx->stats.dp_items += ep.n_dp;
    if (ep.n_dp > 0 && !skip_dp) {
      ctx->stats.dp_launches += 1;
      void* args[] = {&ep};
      CK(cudaLaunchKernel(ctx->eval_fn, dim3(ctx->n_ctas), dim3(ctx->eval_threads), args,
                          ctx->smem_bytes, ctx->stream));
      CK(cudaGetLastError());
      ctx->launches += 1;
    }
    CK(cudaEventRecord(ev[2], ctx->stream));
    if (ep.est_fast)
      k_est_t<16, true><<<ctx->est_ctas, kEstTWarps * 32, 0, ctx->stream>>>(ep);
    else if (est_thread && ctx->D == 16)
      k_est_t<16><<<ctx->est_ctas, kEstTWarps * 32, 0, ctx->stream>>>(ep);
    else if (est_thread)
      k_est_t<0><<<ctx->est_ctas, kEstTWarps * 32, 0, ctx->stream>>>(ep);
    else
      k_est<<<ctx->est_ctas, kEstWarps * 32, est_smem, ctx->stream>>>(ep);
    DBG_SYNC("k_est");
    CK(cudaGetLastError());
    CK(cudaEventRecord(ev[3], ctx->stream));
    ctx->launches += 2;
  }
  if (overlap) CK(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
  return AMP_OK;
}

int launch_merge(amp_ctx* ctx, const amp_record* d_in, int n_in, int k, amp_record* d_out,
                 cudaStream_t st) {
  if (n_in % k != 0 || n_in / k > kMergeMaxLists)
    return fail(ctx, AMP_E_INVALID, "merge input must be <= 1024 sorted lists of k records");
  CK(ctx->taken.ensure((size_t)n_in + 16));
  k_merge_topk<<<1, 1024, 0, st>>>(d_in, n_in, k, d_out, ctx->taken.as<unsigned char>());
  CK(cudaGetLastError());
  return AMP_OK;
}

int copy_details(amp_ctx* ctx, uint64_t n, const amp_details* det) {
  if (!det) return AMP_OK;
  if (det->cuts)
    CK(cudaMemcpyAsync(det->cuts, ctx->o_cuts.p, sizeof(int32_t) * n * (ctx->max_pp + 1),
                       cudaMemcpyDeviceToHost, ctx->stream));
  if (det->stage_times)
    CK(cudaMemcpyAsync(det->stage_times, ctx->o_stage.p, sizeof(double) * n * ctx->max_pp,
                       cudaMemcpyDeviceToHost, ctx->stream));
  if (det->edge_times)
    CK(cudaMemcpyAsync(det->edge_times, ctx->o_edge.p, sizeof(double) * n * ctx->max_pp,
                       cudaMemcpyDeviceToHost, ctx->stream));
  if (det->placement)
    CK(cudaMemcpyAsync(det->placement, ctx->o_place.p, sizeof(int32_t) * n * ctx->D,
                       cudaMemcpyDeviceToHost, ctx->stream));
  if (det->simulated)
    CK(cudaMemcpyAsync(det->simulated, ctx->o_sim.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                       ctx->stream));
  return AMP_OK;
}

}  // namespace

namespace {

// Device-resident run over a segment list: evaluate, merge the CTA lists into
// d_topk on the context stream, ordered after / before the caller's stream.
int run_device_segs(amp_ctx* ctx, const std::vector<Segment>& segs, int32_t k, amp_record* d_topk,
                    void* stream) {
  CK(cudaSetDevice(ctx->device));
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  // order the context stream after the caller's stream
  CK(cudaEventRecord(ctx->ev0, user));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev0, 0));
  uint64_t n_work = 0;
  for (const Segment& sg : segs) n_work += sg.count;
  int rc = AMP_OK;
  ctx->launches = 0;
  if (n_work > 0) {
    rc = launch_evaluate(ctx, &segs, nullptr, n_work, k, false, false, false);
    if (rc) return rc;
  } else {
    // nothing to evaluate: pad the CTA lists
    std::vector<amp_record> pad((size_t)k * ctx->est_ctas);
    for (auto& e : pad) {
      std::memset(&e, 0, sizeof(e));
      e.index = ~0ull;
      e.fail_code = -1;
      e.total = e.pipeline_time = e.dpsync_time = NAN;
    }
    CK(ctx->cta_topk.ensure(sizeof(amp_record) * pad.size()));
    CK(cudaMemcpyAsync(ctx->cta_topk.p, pad.data(), sizeof(amp_record) * pad.size(),
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  rc = launch_merge(ctx, ctx->cta_topk.as<amp_record>(),
                    k * (n_work > 0 ? ctx->n_topk_lists : ctx->est_ctas), k, d_topk, ctx->stream);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev2, ctx->stream));
  CK(cudaStreamWaitEvent(user, ctx->ev2, 0));
  account(ctx, 0, 0, nullptr, 0, &segs);
  ctx->stats.launches = ctx->launches + 1;
  ctx->stats.ctas = ctx->n_ctas;
  ctx->stats.kernel_ms = -1;  // resolved by amp_search_last_stats
  ctx->stats.total_ms = -1;
  return AMP_OK;
}

// Shards: every class is cut into min(P, n) contiguous placement blocks,
// weighted by its per-candidate work (DP inner iterations of its pruned
// program + a placement/estimate constant, as amp_search_partition), and
// the blocks go longest-processing-time-first (by class weight, a class's
// blocks together) to the least-loaded shard (ties: lowest shard).  With P >= n every shard gets one block of every
// class (the same class mix); with P = 1 (the plan() space, e.g. C4's 440
// uneven DP instances) it is LPT over the classes.  Deterministic: every
// rank computes the same plan.  Mirrored by distributed.lpt_shards.
//
// Signature-disjoint variant (n > 1, P >= n, enough pp <= 2 work to fill):
// every DP class (pp >= 3) is one unit — a signature contains its class, so
// no two shards solve the same DP instance, and the memoised DP work is
// split across the shards instead of repeated on each — dealt first, the
// largest DP programs first (round robin at equal weights); the pp <= 2
// classes (no DP) in min(P, n) blocks then balance the per-candidate load.
// Weights: 2 units per DP-class candidate (K_place + K_est), 1 per pp <= 2
// candidate (K_est only), times 128 D.
std::vector<std::vector<Segment>> shard_plan(const amp_ctx* ctx, int32_t n_shards, uint64_t begin = 0,
                                             uint64_t end = ~0ull) {
  struct Unit {
    double w, wc;
    uint64_t c, p0, p1;
  };
  const uint64_t P = ctx->P;
  std::vector<Unit> units;
  double heavy_max = 0, light_w = 0;
  for (uint64_t c = 0; c < ctx->classes.size(); ++c) {
    const uint64_t lo = std::max(begin, c * P), hi = std::min(end, (c + 1) * P);
    if (hi <= lo) continue;
    if (is_heavy(ctx, c)) heavy_max = std::max(heavy_max, 2.0 * (double)(hi - lo));
    else light_w += (double)(hi - lo);
  }
  const bool disjoint = n_shards > 1 && P >= (uint64_t)n_shards && heavy_max > 0 &&
                        light_w >= heavy_max * n_shards && std::getenv("AMP_SHARD_BLOCKS") == nullptr;
  for (uint64_t c = 0; c < ctx->classes.size(); ++c) {  // the class's part of [begin, end)
    const uint64_t lo = std::max(begin, c * P), hi = std::min(end, (c + 1) * P);
    if (hi <= lo) continue;
    const bool whole = disjoint && is_heavy(ctx, c);
    const uint64_t q0 = lo - c * P, n = hi - lo, nb = whole ? 1 : std::min<uint64_t>(n, (uint64_t)n_shards);
    // sort key: LPT by class weight (disjoint: DP classes first, largest
    // program first), a class's blocks adjacent
    const double wc = disjoint ? (whole ? 1e12 + ctx->class_inner[c] : 128.0 * ctx->D)
                               : ctx->class_inner[c] + 128.0 * ctx->D;
    const double wu = disjoint ? (whole ? 2.0 : 1.0) * 128.0 * ctx->D : wc;  // per-candidate load
    for (uint64_t b = 0; b < nb; ++b) {
      const uint64_t p0 = q0 + n * b / nb, p1 = q0 + n * (b + 1) / nb;
      if (p1 > p0) units.push_back(Unit{wu * (double)(p1 - p0), wc, c, p0, p1});
    }
  }
  // longest first by the class weight, a class's blocks adjacent (stable)
  std::stable_sort(units.begin(), units.end(), [](const Unit& a, const Unit& b) { return a.wc > b.wc; });
  std::vector<double> load(n_shards, 0.0);
  std::vector<std::vector<std::pair<double, Segment>>> v(n_shards);
  for (const Unit& u : units) {
    const int s = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    load[s] += u.w;
    Segment sg{};
    sg.first = u.c * P + u.p0;
    sg.count = u.p1 - u.p0;
    sg.p0 = u.p0;
    sg.cls = (int64_t)u.c;
    // dispatch order within a shard: pp >= 3 classes first, heaviest first
    v[s].emplace_back(ctx->class_inner[u.c] + (is_heavy(ctx, u.c) ? 1e30 : 0.0), sg);
  }
  std::vector<std::vector<Segment>> out(n_shards);
  for (int s = 0; s < n_shards; ++s) {
    std::stable_sort(v[s].begin(), v[s].end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    uint64_t off = 0;
    for (auto& e : v[s]) {
      e.second.offset = off;
      e.second.out = off;
      off += e.second.count;
      out[s].push_back(e.second);
    }
  }
  return out;
}

std::vector<Segment> make_shard_segments(const amp_ctx* ctx, int32_t shard, int32_t n_shards) {
  return shard_plan(ctx, n_shards)[shard];
}

// amp_search_run on a multi-GPU context: the range's LPT shard plan, one
// host thread per device evaluates its shard (K_place -> K_dp -> K_est, CTA
// lists -> device top-k), an NCCL all-gather of the k records over NVLink,
// the device merge on the first device; per-record outputs are copied from
// each device to their host positions.  Identical to the single-GPU run.
int run_multi(amp_ctx* ctx, uint64_t begin, uint64_t end, int32_t k, amp_record* topk, int32_t* n_topk,
              amp_record* all, const amp_details* det) {
  const int n = (int)ctx->subs.size() + 1, kk = std::max(1, k);
  const auto plan = shard_plan(ctx, n, begin, end);
  const bool want_det = det && (det->cuts || det->stage_times || det->edge_times);
  const bool want_place = det && det->placement, want_sim = all && det && det->simulated;
  std::vector<int> rcs(n, AMP_OK);
  auto dev_ctx = [&](int r) { return r == 0 ? ctx : ctx->subs[r - 1]; };
  auto on_all = [&](auto&& fn) {  // fn(r) on a thread per device
    std::vector<std::thread> th;
    for (int r = 1; r < n; ++r) th.emplace_back([&, r]() { rcs[r] = fn(r); });
    rcs[0] = fn(0);
    for (auto& t : th) t.join();
    for (int r = 0; r < n; ++r)
      if (rcs[r] != AMP_OK) {
        if (r) ctx->err = "device " + std::to_string(dev_ctx(r)->device) + ": " + dev_ctx(r)->err;
        return rcs[r];
      }
    return (int)AMP_OK;
  };
  // ---- phase 1: every shard to a device top-k (+ per-record outputs) -----
  int rc = on_all([&](int r) -> int {
    amp_ctx* c = dev_ctx(r);
    AllocStream g(c->stream);
    CK(cudaSetDevice(c->device));
    const std::vector<Segment>& segs = plan[r];
    uint64_t nw = 0;
    for (const Segment& sg : segs) nw += sg.count;
    c->launches = 0;
    CK(c->topk.ensure(sizeof(amp_record) * kk));
    if (nw > 0) {
      int e = launch_evaluate(c, &segs, nullptr, nw, kk, all != nullptr, want_det, want_place, nullptr, want_sim);
      if (e) return e;
      e = launch_merge(c, c->cta_topk.as<amp_record>(), kk * c->n_topk_lists, kk, c->topk.as<amp_record>(),
                       c->stream);
      if (e) return e;
    } else {
      std::vector<amp_record> pad(kk);
      for (auto& x : pad) {
        std::memset(&x, 0, sizeof x);
        x.index = ~0ull;
        x.fail_code = -1;
        x.total = x.pipeline_time = x.dpsync_time = NAN;
      }
      CK(cudaMemcpyAsync(c->topk.p, pad.data(), sizeof(amp_record) * kk, cudaMemcpyHostToDevice, c->stream));
    }
    // this shard's per-record outputs: one bulk copy per array (the shard's
    // records are contiguous on the device, segment after segment), then
    // each segment to its host position (P = 1 shards have a segment per
    // class: hundreds of small device copies otherwise)
    const int W = c->max_pp + 1, MP = c->max_pp, D = c->D;
    struct Out {
      bool on;
      const void* src;
      void* dst;
      size_t rec;  // bytes per record
      std::vector<unsigned char> h;
    };
    Out outs[] = {
        {all != nullptr, c->o_all.p, all, sizeof(amp_record), {}},
        {det && det->cuts, c->o_cuts.p, det ? det->cuts : nullptr, sizeof(int32_t) * W, {}},
        {det && det->stage_times, c->o_stage.p, det ? det->stage_times : nullptr, sizeof(double) * MP, {}},
        {det && det->edge_times, c->o_edge.p, det ? det->edge_times : nullptr, sizeof(double) * MP, {}},
        {det && det->placement, c->o_place.p, det ? det->placement : nullptr, sizeof(int32_t) * D, {}},
        {want_sim, c->o_sim.p, want_sim ? det->simulated : nullptr, sizeof(double), {}},
    };
    for (Out& o : outs)
      if (o.on && nw) {
        o.h.resize(o.rec * nw);
        CK(cudaMemcpyAsync(o.h.data(), o.src, o.rec * nw, cudaMemcpyDeviceToHost, c->stream));
      }
    CK(c->gathered.ensure(sizeof(amp_record) * kk * n));
    CK(cudaStreamSynchronize(c->stream));
    for (Out& o : outs)
      if (o.on && nw)
        for (const Segment& sg : segs)
          std::memcpy(static_cast<unsigned char*>(o.dst) + (sg.first - begin) * o.rec, o.h.data() + sg.out * o.rec,
                      sg.count * o.rec);
    account(c, 0, 0, nullptr, 0, &segs);
    resolve_kernel_times(c);
    return AMP_OK;
  });
  if (rc) return rc;
  // ---- phase 2: NCCL all-gather of the k records, merge on device 0 -------
  rc = on_all([&](int r) -> int {
    amp_ctx* c = dev_ctx(r);
    CK(cudaSetDevice(c->device));
    const ncclResult_t nr = ncclAllGather(c->topk.p, c->gathered.p, sizeof(amp_record) * kk, ncclUint8,
                                          ctx->comms[r], c->stream);
    if (nr != ncclSuccess) {
      c->err = std::string("ncclAllGather: ") + ncclGetErrorString(nr);
      return AMP_E_CUDA;
    }
    CK(cudaStreamSynchronize(c->stream));
    return AMP_OK;
  });
  if (rc) return rc;
  AllocStream g(ctx->stream);
  CK(cudaSetDevice(ctx->device));
  CK(ctx->mtopk.ensure(sizeof(amp_record) * kk));
  rc = launch_merge(ctx, ctx->gathered.as<amp_record>(), kk * n, kk, ctx->mtopk.as<amp_record>(), ctx->stream);
  if (rc) return rc;
  std::vector<amp_record> tk(kk);
  CK(cudaMemcpyAsync(tk.data(), ctx->mtopk.p, sizeof(amp_record) * kk, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int cnt = 0;
  for (int i = 0; i < k; ++i)
    if (tk[i].fail_code >= 0) topk[cnt++] = tk[i];
  if (n_topk) *n_topk = cnt;
  // stats: work summed over the devices, times the slowest device's
  amp_stats agg = ctx->stats;
  for (amp_ctx* sub : ctx->subs) {
    const amp_stats& o = sub->stats;
    agg.candidates += o.candidates;
    agg.dp_instances += o.dp_instances;
    agg.dp_inner += o.dp_inner;
    agg.fp64_ops += o.fp64_ops;
    agg.dp_cells += o.dp_cells;
    agg.dp_items += o.dp_items;
    agg.launches += o.launches;
    agg.place_ms = std::max(agg.place_ms, o.place_ms);
    agg.dp_ms = std::max(agg.dp_ms, o.dp_ms);
    agg.est_ms = std::max(agg.est_ms, o.est_ms);
    agg.dp_stage_ms = std::max(agg.dp_stage_ms, o.dp_stage_ms);
    agg.dp_fallback += o.dp_fallback;
  }
  agg.kernel_ms = agg.total_ms = std::max(agg.place_ms + agg.dp_ms + agg.est_ms, 0.0);
  ctx->stats = agg;
  return AMP_OK;
}

}  // namespace

extern "C" {

int amp_search_abi_version(void) { return AMP_SEARCH_ABI_VERSION; }

const char* amp_last_error(void) { return g_last_error.c_str(); }

int amp_search_create(amp_ctx** out, const amp_problem* problem,
                      const amp_search_config* config) {
  AllocStream alloc_guard(nullptr);  // setup() points it at the new stream
  if (!out) {
    g_last_error = "out is NULL";
    return AMP_E_INVALID;
  }
  *out = nullptr;
  amp_ctx* ctx = new amp_ctx();
  const int n_gpus = config ? config->n_gpus : 1;
  // a context per further device (same problem, same candidate space), set
  // up by a thread each while this thread sets up the first device's
  std::vector<amp_ctx*> subs(n_gpus > 1 ? n_gpus - 1 : 0, nullptr);
  std::vector<int> rcs(subs.size(), AMP_OK);
  std::vector<std::thread> th;
  for (int r = 1; r < n_gpus; ++r)
    th.emplace_back([&, r]() {
      amp_search_config c = *config;
      c.device = config->device + r;
      c.n_gpus = 1;
      AllocStream g(nullptr);
      subs[r - 1] = new amp_ctx();
      rcs[r - 1] = setup(subs[r - 1], problem, &c);
    });
  int rc = setup(ctx, problem, config);
  for (auto& t : th) t.join();
  if (n_gpus > 1) ctx->subs = subs;
  if (rc == AMP_OK && n_gpus > 1) {
    // and one NCCL communicator per device
    for (int r = 1; r < n_gpus && rc == AMP_OK; ++r)
      if (rcs[r - 1] != AMP_OK) {
        ctx->err = "device " + std::to_string(config->device + r) + ": " + subs[r - 1]->err;
        rc = rcs[r - 1];
      }
    if (rc == AMP_OK) {
      std::vector<int> devs(n_gpus);
      for (int r = 0; r < n_gpus; ++r) devs[r] = config->device + r;
      ctx->comm_devs = devs;
      {
        std::lock_guard<std::mutex> lk(g_comm_mu);
        auto it = g_comm_pool.find(devs);
        if (it != g_comm_pool.end() && !it->second.empty()) {
          ctx->comms = it->second.back();
          it->second.pop_back();
        }
      }
      if (ctx->comms.empty()) {
        ctx->comms.assign(n_gpus, nullptr);
        const ncclResult_t nr = ncclCommInitAll(ctx->comms.data(), n_gpus, devs.data());
        if (nr != ncclSuccess) {
          ctx->comms.clear();
          ctx->err = std::string("ncclCommInitAll: ") + ncclGetErrorString(nr);
          rc = AMP_E_CUDA;
        }
      }
    }
  }
  if (rc != AMP_OK) {
    g_last_error = ctx->err;
    amp_search_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return AMP_OK;
}

void amp_search_destroy(amp_ctx* ctx) {
  if (!ctx) return;
  if (!ctx->comms.empty()) {
    bool kept = false;
    if (ctx->err.empty() && std::getenv("AMP_NO_RECYCLE") == nullptr) {  // to the next context
      std::lock_guard<std::mutex> lk(g_comm_mu);
      g_comm_pool[ctx->comm_devs].push_back(ctx->comms);
      kept = true;
    }
    if (!kept)
      for (ncclComm_t c : ctx->comms)
        if (c) ncclCommDestroy(c);
    ctx->comms.clear();
  }
  for (amp_ctx* sub : ctx->subs) amp_search_destroy(sub);
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->ev2) cudaEventDestroy(ctx->ev2);
  for (cudaEvent_t e : ctx->kev) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->tev) cudaEventDestroy(e);
  if (ctx->aux) cudaStreamSynchronize(ctx->aux);
  if (ctx->aux_start) cudaEventDestroy(ctx->aux_start);
  if (ctx->aux_done) cudaEventDestroy(ctx->aux_done);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  cudaStream_t st = ctx->stream;
  if (st && ctx->err.empty() && std::getenv("AMP_NO_RECYCLE") == nullptr) {
    // hand the stream, hash table and clear trie marks to the device's next context
    std::lock_guard<std::mutex> lk(g_rec_mu);
    Recycled& r = g_rec[ctx->device];
    if (!r.used) {
      r.used = true;
      r.stream = st;
      r.tkey = ctx->dd_tkey.p;
      r.tkey_bytes = ctx->dd_tkey.bytes;
      r.T = ctx->hash_T;
      r.epoch = ctx->hash_epoch;
      r.esh = ctx->hash_esh;
      r.pres = ctx->tr_pres.p;
      r.pres_bytes = ctx->tr_pres.bytes;
      ctx->dd_tkey.p = nullptr;
      ctx->dd_tkey.bytes = 0;
      ctx->tr_pres.p = nullptr;
      ctx->tr_pres.bytes = 0;
      st = nullptr;
    }
  }
  delete ctx;  // buffers return to the pool, ordered on the context stream
  if (st) cudaStreamDestroy(st);
}

const char* amp_search_last_error(const amp_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

uint64_t amp_search_num_candidates(const amp_ctx* ctx) {
  return ctx ? (uint64_t)ctx->classes.size() * ctx->P : 0;
}

int32_t amp_search_num_classes(const amp_ctx* ctx) {
  return ctx ? static_cast<int32_t>(ctx->classes.size()) : 0;
}

int32_t amp_search_max_pp(const amp_ctx* ctx) { return ctx ? ctx->max_pp : 0; }

int amp_search_class(const amp_ctx* ctx, int32_t c, int32_t* pp, int32_t* dp, int32_t* tmp,
                     int32_t* mbs) {
  if (!ctx || c < 0 || c >= (int32_t)ctx->classes.size()) return AMP_E_INVALID;
  const ClassDev& cl = ctx->classes[c];
  if (pp) *pp = cl.pp;
  if (dp) *dp = cl.dp;
  if (tmp) *tmp = cl.tmp;
  if (mbs) *mbs = cl.mbs;
  return AMP_OK;
}

int amp_search_partition(const amp_ctx* ctx, int32_t n_parts, uint64_t* bounds) {
  if (!ctx || n_parts < 1 || !bounds) return AMP_E_INVALID;
  const uint64_t P = ctx->P, N = (uint64_t)ctx->classes.size() * P;
  // per-candidate weight: DP inner iterations + a constant for the
  // placement/estimate work of every candidate
  std::vector<double> w(ctx->classes.size());
  double total = 0;
  for (size_t c = 0; c < w.size(); ++c) {
    w[c] = ctx->class_inner[c] + 128.0 * ctx->D;  // ~place+est cost (r1b bench: ~2000 inner-equiv. at |D|=16)
    total += w[c] * (double)P;
  }
  bounds[0] = 0;
  size_t c = 0;
  double acc = 0;  // cumulative weight before class c
  for (int32_t part = 1; part < n_parts; ++part) {
    const double target = total * part / n_parts;
    while (c < w.size() && acc + w[c] * (double)P < target) {
      acc += w[c] * (double)P;
      ++c;
    }
    uint64_t b = N;
    if (c < w.size()) {
      const double within = (target - acc) / w[c];
      uint64_t off = (uint64_t)std::llround(within);
      if (off > P) off = P;
      b = (uint64_t)c * P + off;
    }
    bounds[part] = std::max(b, bounds[part - 1]);
  }
  bounds[n_parts] = N;
  return AMP_OK;
}

int amp_search_run(amp_ctx* ctx, uint64_t begin, uint64_t end, int32_t k, amp_record* topk,
                   int32_t* n_topk, amp_record* all, const amp_details* all_details) {
  AllocStream alloc_guard(ctx ? ctx->stream : nullptr);
  if (!ctx) return AMP_E_INVALID;
  const uint64_t N = amp_search_num_candidates(ctx);
  if (begin > end || end > N) return fail(ctx, AMP_E_INVALID, "range outside [0, num_candidates)");
  if (k < 0 || k > 4096) return fail(ctx, AMP_E_INVALID, "k must be in [0, 4096]");
  if (k > 0 && !topk) return fail(ctx, AMP_E_INVALID, "topk is NULL");
  CK(cudaSetDevice(ctx->device));
  const uint64_t n = end - begin;
  if (n_topk) *n_topk = 0;
  if (n == 0) return AMP_OK;
  if (!ctx->subs.empty()) return run_multi(ctx, begin, end, k, topk, n_topk, all, all_details);
  const auto segs = make_segments(ctx, begin, end);
  const bool det = all_details && (all_details->cuts || all_details->stage_times ||
                                   all_details->edge_times);
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  ctx->launches = 0;
  int rc = launch_evaluate(ctx, &segs, nullptr, n, k, all != nullptr, det,
                           all_details && all_details->placement, nullptr,
                           all != nullptr && all_details && all_details->simulated);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  const int kk = std::max(1, k);
  CK(ctx->topk.ensure(sizeof(amp_record) * kk));
  rc = launch_merge(ctx, ctx->cta_topk.as<amp_record>(), kk * ctx->n_topk_lists, kk,
                    ctx->topk.as<amp_record>(), ctx->stream);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev2, ctx->stream));
  std::vector<amp_record> tk(kk);
  CK(cudaMemcpyAsync(tk.data(), ctx->topk.p, sizeof(amp_record) * kk, cudaMemcpyDeviceToHost,
                     ctx->stream));
  if (all)
    CK(cudaMemcpyAsync(all, ctx->o_all.p, sizeof(amp_record) * n, cudaMemcpyDeviceToHost,
                       ctx->stream));
  rc = copy_details(ctx, n, all_details);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  int cnt = 0;
  for (int i = 0; i < k; ++i)
    if (tk[i].fail_code >= 0) topk[cnt++] = tk[i];
  if (n_topk) *n_topk = cnt;
  float ms1 = 0, ms2 = 0;
  cudaEventElapsedTime(&ms1, ctx->ev0, ctx->ev1);
  cudaEventElapsedTime(&ms2, ctx->ev0, ctx->ev2);
  account(ctx, begin, end, nullptr, 0);
  resolve_kernel_times(ctx);
  ctx->stats.kernel_ms = ms1;
  ctx->stats.total_ms = ms2;
  ctx->stats.launches = ctx->launches + 1;
  ctx->stats.ctas = ctx->n_ctas;
  return AMP_OK;
}

int amp_search_evaluate(amp_ctx* ctx, const uint64_t* indices, int32_t n, amp_record* out,
                        const amp_details* details) {
  AllocStream alloc_guard(ctx ? ctx->stream : nullptr);
  if (!ctx || n < 0 || (n > 0 && (!indices || !out))) return AMP_E_INVALID;
  if (n == 0) return AMP_OK;
  const uint64_t N = amp_search_num_candidates(ctx);
  for (int32_t i = 0; i < n; ++i)
    if (indices[i] >= N) return fail(ctx, AMP_E_INVALID, "index outside [0, num_candidates)");
  CK(cudaSetDevice(ctx->device));
  CK(upload(ctx->index_list, indices, (size_t)n));
  const bool det = details && (details->cuts || details->stage_times || details->edge_times);
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  ctx->launches = 0;
  int rc = launch_evaluate(ctx, nullptr, ctx->index_list.as<uint64_t>(), (uint64_t)n, 1, true,
                           det, details && details->placement, nullptr,
                           details && details->simulated);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaMemcpyAsync(out, ctx->o_all.p, sizeof(amp_record) * n, cudaMemcpyDeviceToHost,
                     ctx->stream));
  rc = copy_details(ctx, (uint64_t)n, details);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  account(ctx, 0, 0, indices, n);
  resolve_kernel_times(ctx);
  ctx->stats.kernel_ms = ms;
  ctx->stats.total_ms = ms;
  ctx->stats.launches = ctx->launches;
  ctx->stats.ctas = ctx->n_ctas;
  return AMP_OK;
}

int amp_search_estimate(amp_ctx* ctx, const uint64_t* indices, const int32_t* cuts, int32_t n,
                        amp_record* out, const amp_details* details) {
  AllocStream alloc_guard(ctx ? ctx->stream : nullptr);
  if (!ctx || n < 0 || (n > 0 && (!indices || !cuts || !out))) return AMP_E_INVALID;
  if (n == 0) return AMP_OK;
  const uint64_t N = amp_search_num_candidates(ctx);
  const int W = ctx->max_pp + 1;
  std::vector<uint8_t> c8((size_t)n * W, 0);
  for (int32_t i = 0; i < n; ++i) {
    if (indices[i] >= N) return fail(ctx, AMP_E_INVALID, "index outside [0, num_candidates)");
    const int pp = ctx->classes[indices[i] / ctx->P].pp;
    const int32_t* c = cuts + (size_t)i * W;
    if (pp <= ctx->L) {  // (pp > L fails in K_place before the cuts are read)
      bool ok = c[0] == 0 && c[pp] == ctx->L;
      for (int j = 0; j < pp && ok; ++j) ok = c[j] < c[j + 1];
      if (!ok)
        return fail(ctx, AMP_E_INVALID,
                    "cuts of candidate " + std::to_string(i) +
                        " must rise strictly from 0 to n_layers over pp stages");
    }
    for (int j = 0; j <= pp && j < W; ++j) c8[(size_t)i * W + j] = (uint8_t)c[j];
  }
  CK(cudaSetDevice(ctx->device));
  CK(upload(ctx->index_list, indices, (size_t)n));
  DevBuf d_cuts;
  CK(upload(d_cuts, c8.data(), c8.size()));
  const bool det = details && (details->cuts || details->stage_times || details->edge_times);
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  ctx->launches = 0;
  int rc = launch_evaluate(ctx, nullptr, ctx->index_list.as<uint64_t>(), (uint64_t)n, 1, true,
                           det, details && details->placement, d_cuts.as<uint8_t>(),
                           details && details->simulated);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaMemcpyAsync(out, ctx->o_all.p, sizeof(amp_record) * n, cudaMemcpyDeviceToHost,
                     ctx->stream));
  rc = copy_details(ctx, (uint64_t)n, details);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  resolve_kernel_times(ctx);
  ctx->stats.kernel_ms = ms;
  ctx->stats.total_ms = ms;
  ctx->stats.launches = ctx->launches;
  ctx->stats.ctas = ctx->n_ctas;
  ctx->stats.candidates = (uint64_t)n;
  ctx->stats.dp_inner = ctx->stats.fp64_ops = 0;
  return AMP_OK;
}

int amp_search_evaluate_placed(amp_ctx* ctx, const int32_t* classes, const int32_t* placements,
                               const int32_t* cuts, int32_t n, amp_record* out,
                               const amp_details* details) {
  AllocStream alloc_guard(ctx ? ctx->stream : nullptr);
  if (!ctx || n < 0 || (n > 0 && (!classes || !placements || !out))) return AMP_E_INVALID;
  if (n == 0) return AMP_OK;
  const int D = ctx->D, W = ctx->max_pp + 1;
  std::vector<uint64_t> idx(n);
  std::vector<uint8_t> c8;
  if (cuts) c8.assign((size_t)n * W, 0);
  std::vector<char> seen(D);
  for (int32_t i = 0; i < n; ++i) {
    if (classes[i] < 0 || classes[i] >= (int32_t)ctx->classes.size())
      return fail(ctx, AMP_E_INVALID, "class outside [0, num_classes)");
    idx[i] = (uint64_t)classes[i] * ctx->P;  // placement slot 0, overridden
    std::fill(seen.begin(), seen.end(), 0);
    for (int x = 0; x < D; ++x) {
      const int d = placements[(size_t)i * D + x];
      if (d < 0 || d >= D || seen[d])
        return fail(ctx, AMP_E_INVALID,
                    "placement " + std::to_string(i) + " is not a permutation of the devices");
      seen[d] = 1;
    }
    if (cuts) {
      const int pp = ctx->classes[classes[i]].pp;
      const int32_t* c = cuts + (size_t)i * W;
      if (pp <= ctx->L) {
        bool ok = c[0] == 0 && c[pp] == ctx->L;
        for (int j = 0; j < pp && ok; ++j) ok = c[j] < c[j + 1];
        if (!ok)
          return fail(ctx, AMP_E_INVALID,
                      "cuts of candidate " + std::to_string(i) +
                          " must rise strictly from 0 to n_layers over pp stages");
      }
      for (int j = 0; j <= pp && j < W; ++j) c8[(size_t)i * W + j] = (uint8_t)c[j];
    }
  }
  CK(cudaSetDevice(ctx->device));
  CK(upload(ctx->index_list, idx.data(), idx.size()));
  DevBuf d_place, d_cuts;
  CK(upload(d_place, placements, (size_t)n * D));
  if (cuts) CK(upload(d_cuts, c8.data(), c8.size()));
  const bool det = details && (details->cuts || details->stage_times || details->edge_times);
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  ctx->launches = 0;
  int rc = launch_evaluate(ctx, nullptr, ctx->index_list.as<uint64_t>(), (uint64_t)n, 1, true, det,
                           details && details->placement, cuts ? d_cuts.as<uint8_t>() : nullptr,
                           details && details->simulated, d_place.as<int32_t>());
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaMemcpyAsync(out, ctx->o_all.p, sizeof(amp_record) * n, cudaMemcpyDeviceToHost,
                     ctx->stream));
  rc = copy_details(ctx, (uint64_t)n, details);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  account(ctx, 0, 0, idx.data(), n);
  resolve_kernel_times(ctx);
  ctx->stats.kernel_ms = ms;
  ctx->stats.total_ms = ms;
  ctx->stats.launches = ctx->launches;
  ctx->stats.ctas = ctx->n_ctas;
  return AMP_OK;
}

int amp_search_run_device(amp_ctx* ctx, uint64_t begin, uint64_t end, int32_t k,
                          amp_record* d_topk, void* stream) {
  AllocStream alloc_guard(ctx ? ctx->stream : nullptr);
  if (!ctx || k < 1 || k > 4096 || !d_topk) return AMP_E_INVALID;
  const uint64_t N = amp_search_num_candidates(ctx);
  if (begin > end || end > N) return fail(ctx, AMP_E_INVALID, "range outside [0, num_candidates)");
  return run_device_segs(ctx, make_segments(ctx, begin, end), k, d_topk, stream);
}

int amp_search_run_device_shard(amp_ctx* ctx, int32_t shard, int32_t n_shards, int32_t k,
                                amp_record* d_topk, void* stream) {
  AllocStream alloc_guard(ctx ? ctx->stream : nullptr);
  if (!ctx || k < 1 || k > 4096 || !d_topk) return AMP_E_INVALID;
  if (n_shards < 1 || shard < 0 || shard >= n_shards)
    return fail(ctx, AMP_E_INVALID, "shard must be in [0, n_shards)");
  return run_device_segs(ctx, make_shard_segments(ctx, shard, n_shards), k, d_topk, stream);
}

uint64_t amp_search_shard_size(const amp_ctx* ctx, int32_t shard, int32_t n_shards) {
  if (!ctx || n_shards < 1 || shard < 0 || shard >= n_shards) return 0;
  uint64_t n = 0;
  for (const Segment& sg : make_shard_segments(ctx, shard, n_shards)) n += sg.count;
  return n;
}

int amp_search_shard_ranges(const amp_ctx* ctx, int32_t shard, int32_t n_shards, uint64_t* ranges,
                            int32_t cap, int32_t* n_ranges) {
  if (!ctx || n_shards < 1 || shard < 0 || shard >= n_shards || !n_ranges) return AMP_E_INVALID;
  const auto segs = make_shard_segments(ctx, shard, n_shards);
  *n_ranges = (int32_t)segs.size();
  if (!ranges) return AMP_OK;
  if (cap < (int32_t)segs.size()) return AMP_E_INVALID;
  for (size_t i = 0; i < segs.size(); ++i) {
    ranges[2 * i] = segs[i].first;
    ranges[2 * i + 1] = segs[i].first + segs[i].count;
  }
  return AMP_OK;
}

int amp_search_merge_topk_device(amp_ctx* ctx, const amp_record* d_in, int32_t n_in, int32_t k,
                                 amp_record* d_out, void* stream) {
  AllocStream alloc_guard(ctx ? ctx->stream : nullptr);
  if (!ctx || !d_in || !d_out || n_in < 1 || k < 1 || k > 4096) return AMP_E_INVALID;
  CK(cudaSetDevice(ctx->device));
  return launch_merge(ctx, d_in, n_in, k, d_out, reinterpret_cast<cudaStream_t>(stream));
}

int amp_search_last_stats(const amp_ctx* ctx_c, amp_stats* out) {
  amp_ctx* ctx = const_cast<amp_ctx*>(ctx_c);
  if (!ctx || !out) return AMP_E_INVALID;
  if (ctx->stats.kernel_ms < 0) {  // device run: resolve the events now
    CK(cudaEventSynchronize(ctx->ev2));
    float ms1 = 0, ms2 = 0;
    cudaEventElapsedTime(&ms1, ctx->ev0, ctx->ev1);
    cudaEventElapsedTime(&ms2, ctx->ev0, ctx->ev2);
    ctx->stats.kernel_ms = ms1;
    ctx->stats.total_ms = ms2;
  }
  resolve_kernel_times(ctx);
  *out = ctx->stats;
  return AMP_OK;
}

int amp_dp_solve_batch(int32_t device, const amp_dp_instance* inst, int32_t n, int32_t* cuts_out,
                       int32_t cut_stride, double* cost_out, int32_t* status_out) {
  amp_ctx tmp_ctx;  // error sink
  amp_ctx* ctx = &tmp_ctx;
  auto bail = [&](int rc) {
    g_last_error = ctx->err;
    return rc;
  };
  if (n < 0 || (n > 0 && (!inst || !cuts_out || !cost_out))) {
    ctx->err = "invalid arguments";
    return bail(AMP_E_INVALID);
  }
  if (n == 0) return AMP_OK;
  int max_L = 1, max_k = 1;
  std::vector<DpBatchItem> items(n);
  size_t tot_times = 0, tot_edges = 0;
  for (int i = 0; i < n; ++i) {
    const auto& it = inst[i];
    int status = 0;
    if (it.n_layers < 1 || it.n_layers > kMaxLayers || it.stages < 1 || it.stages > it.n_layers ||
        it.gas < 1 || !it.layer_times || (it.stages > 1 && !it.edge_costs))
      status = 1;
    if (it.stages + 1 > cut_stride) status = 1;
    items[i] = DpBatchItem{it.n_layers, it.stages, it.gas, status, nullptr, nullptr};
    if (status_out) status_out[i] = status;
    if (status) continue;
    max_L = std::max(max_L, it.n_layers);
    max_k = std::max(max_k, it.stages);
    tot_times += it.n_layers;
    tot_edges += (size_t)std::max(0, it.stages - 1) * it.n_layers;
  }
  int rcs = cudaSetDevice(device);
  if (rcs != cudaSuccess) {
    ctx->err = cudaGetErrorString((cudaError_t)rcs);
    return bail(AMP_E_CUDA);
  }
  std::vector<double> times(tot_times + 1), edges(tot_edges + 1);
  std::vector<size_t> toff(n), eoff(n);
  size_t ta = 0, ea = 0;
  for (int i = 0; i < n; ++i) {
    if (items[i].status) continue;
    toff[i] = ta;
    eoff[i] = ea;
    std::memcpy(&times[ta], inst[i].layer_times, sizeof(double) * inst[i].n_layers);
    ta += inst[i].n_layers;
    const size_t ne = (size_t)std::max(0, inst[i].stages - 1) * inst[i].n_layers;
    if (ne) std::memcpy(&edges[ea], inst[i].edge_costs, sizeof(double) * ne);
    ea += ne;
  }
  DevBuf d_times, d_edges, d_items, d_cuts, d_cost, d_bp, d_slice, d_dom, d_seg, d_w;
  int rc;
#define CKB(call)                                                    \
  do {                                                               \
    cudaError_t e_ = (call);                                         \
    if (e_ != cudaSuccess) {                                         \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      return bail(e_ == cudaErrorMemoryAllocation ? AMP_E_OOM : AMP_E_CUDA); \
    }                                                                \
  } while (0)
  CKB(upload(d_times, times.data(), times.size()));
  CKB(upload(d_edges, edges.data(), edges.size()));
  for (int i = 0; i < n; ++i) {
    if (items[i].status) continue;
    items[i].times = d_times.as<double>() + toff[i];
    items[i].edges = d_edges.as<double>() + eoff[i];
  }
  CKB(upload(d_items, items.data(), items.size()));
  CKB(d_cuts.ensure(sizeof(int32_t) * (size_t)n * cut_stride));
  CKB(d_cost.ensure(sizeof(double) * n));
  const int nv = 1 + max_L * (max_L + 1) / 2;
  int npow2 = 2;
  while (npow2 < nv) npow2 <<= 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int grid = std::min(n, sms * 2);
  const size_t bp_stride = ((size_t)(max_k + 1) * (max_L + 1) * nv + 255) & ~size_t(255);
  const size_t slice_stride = (size_t)(max_L + 1) * nv;
  CKB(d_bp.ensure(bp_stride * grid));
  CKB(d_slice.ensure(sizeof(double) * slice_stride * grid));
  CKB(d_dom.ensure(sizeof(double) * (size_t)npow2 * grid));
  CKB(d_seg.ensure(sizeof(uint16_t) * (size_t)(max_L + 1) * (max_L + 1) * grid));
  CKB(d_w.ensure(sizeof(WEnt) * (size_t)(max_L + 1) * max_L * grid));
  DpBatchParams bpp{};
  bpp.items = d_items.as<DpBatchItem>();
  bpp.n = n;
  bpp.max_L = max_L;
  bpp.max_k = max_k;
  bpp.npow2 = npow2;
  bpp.cut_stride = cut_stride;
  bpp.cuts_out = d_cuts.as<int32_t>();
  bpp.cost_out = d_cost.as<double>();
  bpp.bp = d_bp.as<uint8_t>();
  bpp.bp_stride = bp_stride;
  bpp.slice = d_slice.as<double>();
  bpp.slice_stride = slice_stride;
  bpp.domain = d_dom.as<double>();
  bpp.seg = d_seg.as<uint16_t>();
  bpp.wtab = d_w.as<WEnt>();
  const size_t smem = sizeof(double) * (npow2 + 2 * (max_L + 1)) + sizeof(int) * (max_k + 2);
  CKB(cudaFuncSetAttribute(k_dp_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_dp_batch<<<grid, 512, smem>>>(bpp);
  CKB(cudaGetLastError());
  std::vector<int32_t> cuts((size_t)n * cut_stride);
  CKB(cudaMemcpy(cuts.data(), d_cuts.p, sizeof(int32_t) * cuts.size(), cudaMemcpyDeviceToHost));
  CKB(cudaMemcpy(cost_out, d_cost.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) {
    if (items[i].status) {
      cost_out[i] = NAN;
      for (int q = 0; q < cut_stride; ++q) cuts_out[(size_t)i * cut_stride + q] = -1;
      continue;
    }
    for (int q = 0; q < cut_stride; ++q)
      cuts_out[(size_t)i * cut_stride + q] =
          q <= items[i].stages ? cuts[(size_t)i * cut_stride + q] : -1;
  }
  (void)rc;
#undef CKB
  return AMP_OK;
}

int amp_fp64_peak(int32_t device, double* dadd_per_s, double* ms_out) {
  if (cudaSetDevice(device) != cudaSuccess) return AMP_E_CUDA;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return AMP_E_OOM;
  const int grid = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_dadd_peak<<<grid, threads>>>(d, 64, 1e-300);  // warm-up
  cudaEventRecord(a);
  k_dadd_peak<<<grid, threads>>>(d, iters, 1e-300);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  if (e != cudaSuccess) {
    g_last_error = cudaGetErrorString(e);
    return AMP_E_CUDA;
  }
  const double ops = (double)grid * threads * iters * 16 * 8;
  if (dadd_per_s) *dadd_per_s = ops / (ms * 1e-3);
  if (ms_out) *ms_out = ms;
  return AMP_OK;
}

}  // extern "C"
