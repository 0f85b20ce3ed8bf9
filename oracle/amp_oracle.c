/*
 * amp_oracle.c — TEST INFRASTRUCTURE ONLY (see amp_oracle.h).
 *
 * CPU restatement of the reference parplan hot path in plain C.  Each
 * function cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Arithmetic is IEEE double with the reference's
 * exact operation order; compile with -ffp-contract=off (oracle/Makefile).
 *
 * Deliberate differences from the reference, none of which changes a
 * result bit:
 *   - the DP keeps one rolling cost slice per stage plus int16 backpointers
 *     instead of the full (L+1)(k+1)M double/int tables
 *     (pipeline_dp.cpp:99-100); the recurrence and tie-break are unchanged;
 *   - failures are returned as AMP_FAIL_* codes instead of exception text
 *     (the host layer rebuilds the text).
 */
#include "amp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* context                                                              */
/* ------------------------------------------------------------------ */

typedef struct {
  int32_t layer, tmp, mbs;
  int64_t order;
  double seconds;
} prof_entry;

struct oracle_ctx {
  int32_t L, D, gbs;
  int32_t fallback_enabled;
  double bytes_per_param, device_flops, tmp_bandwidth;
  int32_t has_ceiling;
  double ceiling;
  double* param_count;  /* [L] */
  double* flops;        /* [L] */
  uint8_t* flops_ok;    /* [L] */
  double* act;          /* [L-1] */
  int32_t* node_id;     /* [D] */
  double* bw;           /* [D*D], +inf diagonal */
  prof_entry* prof;     /* sorted by (layer, tmp, mbs), duplicates removed */
  int64_t n_prof;
  int32_t n_cls;
  int32_t (*cls)[4];    /* pp, dp, tmp, mbs */
  int32_t max_pp;
  int32_t* base_order;  /* heuristic device order */
  uint64_t P, seed;
};

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* divisors (optimizer.cpp:29-41): all d | n, ascending. */
static int divisors(int n, int* out) {
  int c = 0;
  for (int d = 1; d * d <= n; ++d) {
    if (n % d == 0) {
      out[c++] = d;
      if (d != n / d) out[c++] = n / d;
    }
  }
  qsort(out, (size_t)c, sizeof(int), cmp_int);
  return c;
}

static int cmp_prof(const void* a, const void* b) {
  const prof_entry* x = (const prof_entry*)a;
  const prof_entry* y = (const prof_entry*)b;
  if (x->layer != y->layer) return x->layer < y->layer ? -1 : 1;
  if (x->tmp != y->tmp) return x->tmp < y->tmp ? -1 : 1;
  if (x->mbs != y->mbs) return x->mbs < y->mbs ? -1 : 1;
  return (x->order > y->order) - (x->order < y->order);
}

static const int32_t* g_sort_node; /* only used inside oracle_create */
static int cmp_dev(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  if (g_sort_node[x] != g_sort_node[y]) return g_sort_node[x] < g_sort_node[y] ? -1 : 1;
  return (x > y) - (x < y);
}

oracle_ctx* oracle_create(const amp_problem* p, uint64_t placements_per_class, uint64_t seed) {
  if (!p || p->n_layers < 1 || p->n_devices < 1 || p->gbs < 1 || placements_per_class < 1)
    return NULL;
  oracle_ctx* c = (oracle_ctx*)calloc(1, sizeof(oracle_ctx));
  const int L = p->n_layers, D = p->n_devices;
  c->L = L;
  c->D = D;
  c->gbs = p->gbs;
  c->fallback_enabled = p->fallback_enabled;
  c->bytes_per_param = p->bytes_per_param;
  c->device_flops = p->fallback_device_flops;
  c->tmp_bandwidth = p->fallback_tmp_bandwidth;
  c->has_ceiling = p->has_max_params_per_device;
  c->ceiling = p->max_params_per_device;
  c->P = placements_per_class;
  c->seed = seed;
  c->param_count = (double*)malloc(sizeof(double) * L);
  c->flops = (double*)malloc(sizeof(double) * L);
  c->flops_ok = (uint8_t*)malloc((size_t)L);
  c->act = (double*)malloc(sizeof(double) * (L > 1 ? L - 1 : 1));
  for (int i = 0; i < L; ++i) {
    c->param_count[i] = p->param_count[i];
    c->flops_ok[i] = p->flops_present ? p->flops_present[i] : 0;
    c->flops[i] = (c->flops_ok[i] && p->flops_per_sample) ? p->flops_per_sample[i] : 0.0;
  }
  for (int i = 0; i + 1 < L; ++i) c->act[i] = p->activation_volumes[i];
  c->node_id = (int32_t*)malloc(sizeof(int32_t) * D);
  memcpy(c->node_id, p->node_id, sizeof(int32_t) * D);
  c->bw = (double*)malloc(sizeof(double) * (size_t)D * D);
  memcpy(c->bw, p->bandwidth, sizeof(double) * (size_t)D * D);
  /* json_io.cpp:119-123: self-transfer is the infinite sentinel. */
  for (int i = 0; i < D; ++i) c->bw[(size_t)i * D + i] = INFINITY;

  /* ProfileTable::set overwrites (types.cpp:82-84): keep the last entry. */
  c->prof = (prof_entry*)malloc(sizeof(prof_entry) * (size_t)(p->n_profile_entries + 1));
  for (int64_t e = 0; e < p->n_profile_entries; ++e) {
    c->prof[e].layer = p->profile_layer[e];
    c->prof[e].tmp = p->profile_tmp[e];
    c->prof[e].mbs = p->profile_mbs[e];
    c->prof[e].order = e;
    c->prof[e].seconds = p->profile_seconds[e];
  }
  qsort(c->prof, (size_t)p->n_profile_entries, sizeof(prof_entry), cmp_prof);
  int64_t w = 0;
  for (int64_t e = 0; e < p->n_profile_entries; ++e) {
    if (w > 0 && c->prof[w - 1].layer == c->prof[e].layer && c->prof[w - 1].tmp == c->prof[e].tmp &&
        c->prof[w - 1].mbs == c->prof[e].mbs) {
      c->prof[w - 1] = c->prof[e]; /* later order wins */
    } else {
      c->prof[w++] = c->prof[e];
    }
  }
  c->n_prof = w;

  /* plan() candidate list (optimizer.cpp:288-293 via enumerate_degrees
   * 129-137 and enumerate_mbs 143-148). */
  int* dv = (int*)malloc(sizeof(int) * (D + 1));
  int* dv2 = (int*)malloc(sizeof(int) * (D + 1));
  int* mv = (int*)malloc(sizeof(int) * (p->gbs + 1));
  int cap = 64, n = 0;
  c->cls = (int32_t(*)[4])malloc(sizeof(int32_t[4]) * cap);
  int nd = divisors(D, dv);
  for (int a = 0; a < nd; ++a) {
    const int pp = dv[a];
    int nd2 = divisors(D / pp, dv2);
    for (int b = 0; b < nd2; ++b) {
      const int dp = dv2[b];
      const int tmp = D / (pp * dp);
      if (p->gbs % dp != 0) continue;
      int nm = divisors(p->gbs / dp, mv);
      for (int q = 0; q < nm; ++q) {
        if (n == cap) {
          cap *= 2;
          c->cls = (int32_t(*)[4])realloc(c->cls, sizeof(int32_t[4]) * cap);
        }
        c->cls[n][0] = pp;
        c->cls[n][1] = dp;
        c->cls[n][2] = tmp;
        c->cls[n][3] = mv[q];
        if (pp <= c->L && pp > c->max_pp) c->max_pp = pp; /* (pp > L fails first) */
        ++n;
      }
    }
  }
  c->n_cls = n;
  free(dv);
  free(dv2);
  free(mv);

  /* heuristic_placement device order (placement.cpp:37-49). */
  c->base_order = (int32_t*)malloc(sizeof(int32_t) * D);
  for (int i = 0; i < D; ++i) c->base_order[i] = i;
  g_sort_node = c->node_id;
  qsort(c->base_order, (size_t)D, sizeof(int32_t), cmp_dev);
  g_sort_node = NULL;
  return c;
}

void oracle_destroy(oracle_ctx* c) {
  if (!c) return;
  free(c->param_count);
  free(c->flops);
  free(c->flops_ok);
  free(c->act);
  free(c->node_id);
  free(c->bw);
  free(c->prof);
  free(c->cls);
  free(c->base_order);
  free(c);
}

uint64_t oracle_num_candidates(const oracle_ctx* c) { return (uint64_t)c->n_cls * c->P; }
int32_t oracle_num_classes(const oracle_ctx* c) { return c->n_cls; }
int32_t oracle_max_pp(const oracle_ctx* c) { return c->max_pp; }

int oracle_class(const oracle_ctx* c, int32_t k, int32_t* pp, int32_t* dp, int32_t* tmp,
                 int32_t* mbs) {
  if (k < 0 || k >= c->n_cls) return -1;
  *pp = c->cls[k][0];
  *dp = c->cls[k][1];
  *tmp = c->cls[k][2];
  *mbs = c->cls[k][3];
  return 0;
}

/* ------------------------------------------------------------------ */
/* layer times                                                          */
/* ------------------------------------------------------------------ */

static const prof_entry* prof_find(const oracle_ctx* c, int layer, int tmp, int mbs) {
  int64_t lo = 0, hi = c->n_prof;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    const prof_entry* e = &c->prof[mid];
    int less = e->layer != layer ? e->layer < layer : (e->tmp != tmp ? e->tmp < tmp : e->mbs < mbs);
    if (less) lo = mid + 1;
    else hi = mid;
  }
  if (lo < c->n_prof && c->prof[lo].layer == layer && c->prof[lo].tmp == tmp &&
      c->prof[lo].mbs == mbs)
    return &c->prof[lo];
  return NULL;
}

/* ModelGraph::layer_activation_volume (types.cpp:42-50). */
static double layer_activation_volume(const oracle_ctx* c, int layer) {
  if (c->L <= 1) return 0.0;
  if (layer < c->L - 1) return c->act[layer];
  return c->act[layer - 1];
}

/* LayerTimeResolver::layer_time (cost_model.cpp:74-86) with
 * analytic_layer_time (61-68) and allreduce_time (40-52).
 * Returns 0 ok, AMP_FAIL_PROFILE_MISS, or AMP_FAIL_ALLREDUCE_BANDWIDTH
 * (fail_value in *bad). */
static int layer_time_full(const oracle_ctx* c, int layer, int tmp, int mbs, double* out,
                           double* bad) {
  const prof_entry* e = prof_find(c, layer, tmp, mbs);
  if (e) {
    *out = e->seconds;
    return 0;
  }
  if (!c->fallback_enabled) return AMP_FAIL_PROFILE_MISS;
  const double message = layer_activation_volume(c, layer) * mbs;
  const double bandwidth = c->tmp_bandwidth;
  if (!c->flops_ok[layer]) return AMP_FAIL_PROFILE_MISS;
  const double compute = (double)mbs * c->flops[layer] / ((double)tmp * c->device_flops);
  double ar;
  if (tmp == 1) {
    ar = 0.0;
  } else {
    if (!(bandwidth > 0)) {
      *bad = bandwidth;
      return AMP_FAIL_ALLREDUCE_BANDWIDTH;
    }
    ar = 2.0 * (double)(tmp - 1) * message / ((double)tmp * bandwidth);
  }
  *out = compute + ar;
  return 0;
}

int oracle_layer_time(const oracle_ctx* c, int32_t layer, int32_t tmp, int32_t mbs, double* out) {
  double bad = 0;
  return layer_time_full(c, layer, tmp, mbs, out, &bad) ? 1 : 0;
}

/* ------------------------------------------------------------------ */
/* layer-partition DP                                                   */
/* ------------------------------------------------------------------ */

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* SegmentTimes (pipeline_dp.cpp:39-44) + tolerance_domain (55-68). */
static void prefix_sums(const double* t, int L, double* prefix) {
  prefix[0] = 0.0;
  for (int i = 0; i < L; ++i) prefix[i + 1] = prefix[i] + t[i];
}

static int32_t domain_from_prefix(const double* prefix, int L, double* out) {
  int32_t n = 0;
  out[n++] = 0.0;
  for (int a = 0; a < L; ++a)
    for (int b = a + 1; b <= L; ++b) out[n++] = prefix[b] - prefix[a];
  qsort(out, (size_t)n, sizeof(double), cmp_double);
  int32_t w = 0;
  for (int32_t i = 0; i < n; ++i)
    if (w == 0 || !(out[w - 1] == out[i])) out[w++] = out[i];
  return w;
}

int32_t oracle_tolerance_domain(const double* layer_times, int32_t L, double* out) {
  double* prefix = (double*)malloc(sizeof(double) * (L + 1));
  prefix_sums(layer_times, L, prefix);
  int32_t M = domain_from_prefix(prefix, L, out);
  free(prefix);
  return M;
}

static int32_t lower_bound_d(const double* d, int32_t n, double v) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    int32_t mid = (lo + hi) / 2;
    if (d[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* optimal_assignment core (pipeline_dp.cpp:70-149). */
int oracle_optimal_assignment(const double* layer_times, int32_t L, int32_t stages, int32_t gas,
                              const double* edge_costs, int32_t* cuts_out, double* cost_out,
                              int32_t* domain_size, double* inner_iterations) {
  /* check_stage_count (22-30) and gas (73-75). */
  if (stages < 1 || stages > L || gas < 1) return 1;
  double* prefix = (double*)malloc(sizeof(double) * (L + 1));
  prefix_sums(layer_times, L, prefix);
  const size_t nvals = 1 + (size_t)L * (L + 1) / 2;
  double* domain = (double*)malloc(sizeof(double) * nvals);
  const int32_t M = domain_from_prefix(prefix, L, domain);

  /* seg_index (83-91). */
  int32_t* seg = (int32_t*)calloc((size_t)(L + 1) * (L + 1), sizeof(int32_t));
  for (int a = 0; a < L; ++a)
    for (int b = a + 1; b <= L; ++b)
      seg[a * (L + 1) + b] = lower_bound_d(domain, M, prefix[b] - prefix[a]);

  /* Rolling slice cost[j-1] (prev) -> cost[j] (cur); backpointers for all j. */
  double* prev = (double*)malloc(sizeof(double) * (size_t)(L + 1) * M);
  double* cur = (double*)malloc(sizeof(double) * (size_t)(L + 1) * M);
  int16_t* last_cut = (int16_t*)malloc(sizeof(int16_t) * (size_t)(stages + 1) * (L + 1) * M);
  for (size_t x = 0; x < (size_t)(L + 1) * M; ++x) prev[x] = INFINITY;
  const double g1 = (double)(gas - 1);
  /* base case j = 1 (102-107). */
  for (int i = 1; i <= L; ++i) {
    const double t1 = prefix[i] - prefix[0];
    for (int m = 0; m < M; ++m) {
      const double x = t1 - domain[m];
      prev[(size_t)i * M + m] = g1 * (0.0 < x ? x : 0.0) + t1;
    }
  }
  double inner = 0.0;
  double* edge_at_cut = (double*)malloc(sizeof(double) * L);
  /* recursion (109-131): strict '<' keeps the smallest cut on ties. */
  for (int j = 2; j <= stages; ++j) {
    for (int cut = j - 1; cut < L; ++cut) edge_at_cut[cut] = edge_costs[(size_t)(j - 2) * L + cut];
    for (size_t x = 0; x < (size_t)(L + 1) * M; ++x) cur[x] = INFINITY;
    for (int i = j; i <= L; ++i) {
      for (int m = 0; m < M; ++m) {
        double best = INFINITY;
        int best_cut = -1;
        for (int cut = j - 1; cut < i; ++cut) {
          const double t2 = prefix[i] - prefix[cut];
          const int s = seg[cut * (L + 1) + i];
          const double sub = prev[(size_t)cut * M + (s > m ? s : m)];
          const double x = t2 - domain[m];
          const double g = sub + g1 * (0.0 < x ? x : 0.0) + t2 + edge_at_cut[cut];
          if (g < best) {
            best = g;
            best_cut = cut;
          }
        }
        inner += (double)(i - j + 1);
        cur[(size_t)i * M + m] = best;
        last_cut[((size_t)j * (L + 1) + i) * M + m] = (int16_t)best_cut;
      }
    }
    double* t = prev;
    prev = cur;
    cur = t;
  }
  /* prev now holds stage `stages` (or stage 1 when stages == 1). */
  *cost_out = prev[(size_t)L * M + 0];
  /* backtrack (134-148). */
  cuts_out[stages] = L;
  int i = L, m = 0;
  for (int j = stages; j >= 2; --j) {
    const int cut = last_cut[((size_t)j * (L + 1) + i) * M + m];
    cuts_out[j - 1] = cut;
    const int s = seg[cut * (L + 1) + i];
    m = s > m ? s : m;
    i = cut;
  }
  cuts_out[0] = 0;
  if (domain_size) *domain_size = M;
  if (inner_iterations) *inner_iterations = inner;
  free(prefix);
  free(domain);
  free(seg);
  free(prev);
  free(cur);
  free(last_cut);
  free(edge_at_cut);
  return 0;
}

/* ------------------------------------------------------------------ */
/* placement                                                            */
/* ------------------------------------------------------------------ */

uint64_t oracle_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

void oracle_placement(const oracle_ctx* c, uint64_t index, int32_t* rank_to_device) {
  const uint64_t p = index % c->P;
  memcpy(rank_to_device, c->base_order, sizeof(int32_t) * c->D);
  if (p == 0) return; /* heuristic_placement (placement.cpp:27-66) */
  uint64_t r = oracle_splitmix64(c->seed ^ p);
  for (int k = c->D - 1; k >= 1; --k) {
    const int j = (int)(r % (uint64_t)(k + 1));
    const int32_t t = rank_to_device[k];
    rank_to_device[k] = rank_to_device[j];
    rank_to_device[j] = t;
    r = oracle_splitmix64(r);
  }
}

/* ------------------------------------------------------------------ */
/* evaluate_candidate + estimate                                        */
/* ------------------------------------------------------------------ */

/* Placement::device_at (types.hpp:117-120). */
#define DEV(q, r, s) (place[((size_t)(q) * dp + (r)) * tmp + (s)])
#define LINK(a, b) (c->bw[(size_t)(a) * c->D + (b)])
/* std::min(a, b) == (b < a) ? b : a */
#define STD_MIN(a, b) ((b) < (a) ? (b) : (a))
#define STD_MAX(a, b) ((a) < (b) ? (b) : (a))

static double params_in_range(const oracle_ctx* c, int first, int last) {
  /* ModelGraph::params_in_range (types.cpp:34-40) */
  double sum = 0.0;
  for (int i = first; i < last; ++i) sum += c->param_count[i];
  return sum;
}

/* ------------------------------------------------------------------ */
/* DP memo (SURVEY.md §8(d) "full-N memoized CPU oracle"): optimal_assignment
 * is a pure function of the class (layer times, gas, stage count) and the
 * boundary bandwidths (the edge function), so a per-worker table keyed by
 * (class, bws bits) returns the cuts the DP would compute.                */
/* ------------------------------------------------------------------ */
typedef struct {
  int nb;           /* bandwidth slots per key (max_pp - 1, >= 1) */
  int nc;           /* cut slots per value (max_pp + 1) */
  uint64_t cap, n;  /* power of two; entries */
  uint8_t* used;
  int32_t* cls;
  double* bws;      /* [cap][nb] */
  int32_t* cuts;    /* [cap][nc] */
  pthread_mutex_t* mu; /* shared by the run's workers (DPs run outside it) */
} dp_memo;

static void memo_init(dp_memo* m, int max_pp, uint64_t cap) {
  m->nb = max_pp > 1 ? max_pp - 1 : 1;
  m->nc = max_pp + 1;
  m->cap = cap;
  m->n = 0;
  m->used = (uint8_t*)calloc(cap, 1);
  m->cls = (int32_t*)malloc(sizeof(int32_t) * cap);
  m->bws = (double*)calloc(cap * m->nb, sizeof(double));
  m->cuts = (int32_t*)malloc(sizeof(int32_t) * cap * m->nc);
  m->mu = NULL;
}

static void memo_free(dp_memo* m) {
  free(m->used);
  free(m->cls);
  free(m->bws);
  free(m->cuts);
}

static uint64_t memo_hash(int k, const double* bws, int nb) {
  uint64_t h = oracle_splitmix64((uint64_t)k);
  for (int q = 0; q < nb; ++q) {
    uint64_t v;
    memcpy(&v, &bws[q], 8);
    h = oracle_splitmix64(h ^ v);
  }
  return h;
}

/* slot of (k, bws) (bws padded with zeros to nb): found or the free slot */
static uint64_t memo_slot(const dp_memo* m, int k, const double* bws) {
  uint64_t h = memo_hash(k, bws, m->nb) & (m->cap - 1);
  while (m->used[h] &&
         !(m->cls[h] == k && memcmp(m->bws + h * m->nb, bws, sizeof(double) * m->nb) == 0))
    h = (h + 1) & (m->cap - 1);
  return h;
}

static void memo_put(dp_memo* m, int k, const double* bws, const int32_t* cuts, int pp) {
  if (2 * (m->n + 1) > m->cap) { /* grow x2, re-insert */
    dp_memo g;
    memo_init(&g, m->nc - 1, m->cap * 2);
    for (uint64_t i = 0; i < m->cap; ++i)
      if (m->used[i]) {
        const uint64_t t = memo_slot(&g, m->cls[i], m->bws + i * m->nb);
        g.used[t] = 1;
        g.cls[t] = m->cls[i];
        memcpy(g.bws + t * g.nb, m->bws + i * m->nb, sizeof(double) * m->nb);
        memcpy(g.cuts + t * g.nc, m->cuts + i * m->nc, sizeof(int32_t) * m->nc);
      }
    g.n = m->n;
    g.mu = m->mu;
    memo_free(m);
    *m = g;
  }
  const uint64_t h = memo_slot(m, k, bws);
  if (m->used[h]) return; /* another worker solved it meanwhile */
  m->used[h] = 1;
  m->cls[h] = k;
  memcpy(m->bws + h * m->nb, bws, sizeof(double) * m->nb);
  memcpy(m->cuts + h * m->nc, cuts, sizeof(int32_t) * (pp + 1));
  ++m->n;
}

static void evaluate_impl(const oracle_ctx* c, uint64_t index, amp_record* rec, int32_t* cuts_out,
                          double* stage_out, double* edge_out, dp_memo* memo);

void oracle_evaluate(const oracle_ctx* c, uint64_t index, amp_record* rec, int32_t* cuts_out,
                     double* stage_out, double* edge_out) {
  evaluate_impl(c, index, rec, cuts_out, stage_out, edge_out, NULL);
}

static void evaluate_impl(const oracle_ctx* c, uint64_t index, amp_record* rec, int32_t* cuts_out,
                          double* stage_out, double* edge_out, dp_memo* memo) {
  const int L = c->L;
  const int k = (int)(index / c->P);
  const int pp = c->cls[k][0], dp = c->cls[k][1], tmp = c->cls[k][2], mbs = c->cls[k][3];
  memset(rec, 0, sizeof(*rec));
  rec->index = index;
  rec->pp = pp;
  rec->dp = dp;
  rec->tmp = tmp;
  rec->mbs = mbs;
  rec->total = rec->pipeline_time = rec->dpsync_time = NAN;
  rec->fail_layer = -1;
  const int maxpp = c->max_pp;
  if (cuts_out)
    for (int q = 0; q <= maxpp; ++q) cuts_out[q] = -1;
  if (stage_out)
    for (int q = 0; q < maxpp; ++q) stage_out[q] = NAN;
  if (edge_out)
    for (int q = 0; q < maxpp; ++q) edge_out[q] = NAN;

  /* optimizer.cpp:149-152 */
  if (pp > L) {
    rec->fail_code = AMP_FAIL_PP_GT_L;
    return;
  }
  int32_t* place = (int32_t*)malloc(sizeof(int32_t) * c->D);
  oracle_placement(c, index, place);
  const int gas = c->gbs / (dp * mbs);

  /* placement_edge_cost (optimizer.cpp:130-139) via min_edge_bandwidth
   * (cost_model.cpp:164-174). */
  double* bws = (double*)calloc(maxpp > 1 ? maxpp - 1 : 1, sizeof(double)); /* (memo key pad) */
  for (int q = 0; q + 1 < pp; ++q) {
    double b = INFINITY;
    for (int r = 0; r < dp; ++r)
      for (int s = 0; s < tmp; ++s) b = STD_MIN(b, LINK(DEV(q, r, s), DEV(q + 1, r, s)));
    bws[q] = b;
  }

  /* segment_times (pipeline_dp.cpp:46-53): first failing layer wins. */
  double* t = (double*)malloc(sizeof(double) * L);
  for (int l = 0; l < L; ++l) {
    double bad = 0;
    int f = layer_time_full(c, l, tmp, mbs, &t[l], &bad);
    if (f) {
      rec->fail_code = f;
      rec->fail_layer = l;
      rec->fail_value = bad;
      goto done;
    }
  }
  /* the DP's edge function throws on the first stage boundary whose
   * bandwidth is invalid (p2p_time, cost_model.cpp:54-59). */
  for (int q = 0; q + 1 < pp; ++q) {
    if (!(bws[q] > 0)) {
      rec->fail_code = AMP_FAIL_P2P_BANDWIDTH;
      rec->fail_value = bws[q];
      goto done;
    }
  }
  {
    double* edges = (double*)malloc(sizeof(double) * (size_t)(pp > 1 ? pp - 1 : 1) * L);
    for (int q = 0; q + 1 < pp; ++q) {
      edges[(size_t)q * L + 0] = 0.0;
      for (int cut = 1; cut < L; ++cut)
        edges[(size_t)q * L + cut] = c->act[cut - 1] * mbs / bws[q];
    }
    int32_t* cuts = (int32_t*)malloc(sizeof(int32_t) * (pp + 1));
    double dpcost;
    int hit = 0;
    if (memo) {
      pthread_mutex_lock(memo->mu);
      const uint64_t slot = memo_slot(memo, k, bws);
      if ((hit = memo->used[slot]))
        memcpy(cuts, memo->cuts + slot * memo->nc, sizeof(int32_t) * (pp + 1));
      pthread_mutex_unlock(memo->mu);
    }
    if (!hit) {
      oracle_optimal_assignment(t, L, pp, gas, edges, cuts, &dpcost, NULL, NULL);
      if (memo) {
        pthread_mutex_lock(memo->mu);
        memo_put(memo, k, bws, cuts, pp);
        pthread_mutex_unlock(memo->mu);
      }
    }
    free(edges);

    /* per-device parameter ceiling (optimizer.cpp:159-169). */
    if (c->has_ceiling) {
      double worst = 0.0;
      for (int j = 0; j < pp; ++j)
        worst = STD_MAX(worst, params_in_range(c, cuts[j], cuts[j + 1]) / tmp);
      if (worst > c->ceiling) {
        rec->fail_code = AMP_FAIL_CEILING;
        free(cuts);
        goto done;
      }
    }

    /* estimate (cost_model.cpp:176-212). */
    double* st = (double*)malloc(sizeof(double) * pp);
    for (int j = 0; j < pp; ++j) { /* stage_time (88-98) */
      double sum = 0.0;
      for (int l = cuts[j]; l < cuts[j + 1]; ++l) sum += t[l];
      st[j] = sum;
    }
    double slowest_stage = st[0]; /* std::max_element: first maximum */
    for (int j = 1; j < pp; ++j)
      if (slowest_stage < st[j]) slowest_stage = st[j];
    double* e = (double*)malloc(sizeof(double) * (pp > 1 ? pp - 1 : 1));
    double* best_e = (double*)malloc(sizeof(double) * (pp > 1 ? pp - 1 : 1));
    double slowest = -1.0;
    for (int r = 0; r < dp; ++r) {
      for (int q = 0; q + 1 < pp; ++q) { /* replica_edge_times (145-162) */
        const int cut = cuts[q + 1];
        const double volume = c->act[cut - 1] * mbs;
        double b = INFINITY;
        for (int s = 0; s < tmp; ++s) b = STD_MIN(b, LINK(DEV(q, r, s), DEV(q + 1, r, s)));
        e[q] = volume / b; /* p2p_time: b > 0 is implied by the DP's check */
      }
      /* pipeline_time (100-120) */
      double sum = 0.0;
      for (int q = 0; q + 1 < pp; ++q) sum += e[q];
      for (int j = 0; j < pp; ++j) sum += st[j];
      const double tr = (double)(gas - 1) * slowest_stage + sum;
      if (tr > slowest) {
        slowest = tr;
        for (int q = 0; q + 1 < pp; ++q) best_e[q] = e[q];
      }
    }
    /* dpsync_time (122-143) */
    double worst = 0.0;
    int failed = 0;
    if (dp != 1) {
      for (int j = 0; j < pp && !failed; ++j) {
        const double stage_params = params_in_range(c, cuts[j], cuts[j + 1]);
        const double message = stage_params * c->bytes_per_param / tmp;
        for (int s = 0; s < tmp && !failed; ++s) {
          double b = INFINITY; /* make_comm_group (23-38) */
          for (int r1 = 0; r1 < dp; ++r1)
            for (int r2 = r1 + 1; r2 < dp; ++r2) b = STD_MIN(b, LINK(DEV(j, r1, s), DEV(j, r2, s)));
          if (!(b > 0)) {
            rec->fail_code = AMP_FAIL_ALLREDUCE_BANDWIDTH;
            rec->fail_value = b;
            failed = 1;
            break;
          }
          const double tt = 2.0 * (double)(dp - 1) * message / ((double)dp * b);
          worst = STD_MAX(worst, tt);
        }
      }
    }
    if (!failed) {
      rec->pipeline_time = slowest;
      rec->dpsync_time = worst;
      rec->total = slowest + worst;
      if (cuts_out)
        for (int q = 0; q <= pp; ++q) cuts_out[q] = cuts[q];
      if (stage_out)
        for (int q = 0; q < pp; ++q) stage_out[q] = st[q];
      if (edge_out)
        for (int q = 0; q + 1 < pp; ++q) edge_out[q] = best_e[q];
    }
    free(st);
    free(e);
    free(best_e);
    free(cuts);
  }
done:
  free(place);
  free(bws);
  free(t);
}

/* ------------------------------------------------------------------ */
/* thread pool (optimizer.cpp:212-229) and ranking                      */
/* ------------------------------------------------------------------ */

typedef struct {
  const oracle_ctx* c;
  uint64_t begin, end;
  atomic_uint_fast64_t next;
  amp_record* records;
  int32_t* cuts;
  double* stage;
  double* edge;
  dp_memo* memo;
} run_state;

static void* run_worker(void* arg) {
  run_state* s = (run_state*)arg;
  const int maxpp = s->c->max_pp;
  for (;;) {
    uint64_t i = atomic_fetch_add(&s->next, 1);
    if (i >= s->end - s->begin) break;
    evaluate_impl(s->c, s->begin + i, &s->records[i], s->cuts ? s->cuts + i * (maxpp + 1) : NULL,
                  s->stage ? s->stage + i * maxpp : NULL, s->edge ? s->edge + i * maxpp : NULL,
                  s->memo);
  }
  return NULL;
}

static void run_impl(const oracle_ctx* c, uint64_t begin, uint64_t end, int32_t threads,
                     amp_record* records, int32_t* cuts, double* stage_times, double* edge_times,
                     int memo);

void oracle_run(const oracle_ctx* c, uint64_t begin, uint64_t end, int32_t threads,
                amp_record* records, int32_t* cuts, double* stage_times, double* edge_times) {
  run_impl(c, begin, end, threads, records, cuts, stage_times, edge_times, 0);
}

void oracle_run_memo(const oracle_ctx* c, uint64_t begin, uint64_t end, int32_t threads,
                     amp_record* records, int32_t* cuts, double* stage_times, double* edge_times) {
  run_impl(c, begin, end, threads, records, cuts, stage_times, edge_times, 1);
}

static void run_impl(const oracle_ctx* c, uint64_t begin, uint64_t end, int32_t threads,
                     amp_record* records, int32_t* cuts, double* stage_times, double* edge_times,
                     int memo) {
  if (end <= begin) return;
  run_state s;
  dp_memo m;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  if (memo) {
    memo_init(&m, c->max_pp, 1u << 12);
    m.mu = &mu;
  }
  s.memo = memo ? &m : NULL;
  s.c = c;
  s.begin = begin;
  s.end = end;
  atomic_init(&s.next, 0);
  s.records = records;
  s.cuts = cuts;
  s.stage = stage_times;
  s.edge = edge_times;
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > end - begin) threads = (int32_t)(end - begin);
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int w = 1; w < threads; ++w) pthread_create(&tid[w], NULL, run_worker, &s);
  run_worker(&s);
  for (int w = 1; w < threads; ++w) pthread_join(tid[w], NULL);
  free(tid);
  if (memo) memo_free(&m);
}

static const amp_record* g_rank_records;
/* rank_records comparator (optimizer.cpp:264-278) with the degree key
 * extended to the candidate index (class-major, so identical for P == 1). */
static int cmp_rank(const void* a, const void* b) {
  const amp_record* x = &g_rank_records[*(const int64_t*)a];
  const amp_record* y = &g_rank_records[*(const int64_t*)b];
  const int fx = x->fail_code != 0, fy = y->fail_code != 0;
  if (fx != fy) return fx ? 1 : -1;
  if (!fx && x->total != y->total) return x->total < y->total ? -1 : 1;
  return (x->index > y->index) - (x->index < y->index);
}

void oracle_rank(const amp_record* records, int64_t n, int64_t* order) {
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  g_rank_records = records;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_rank);
  g_rank_records = NULL;
}
