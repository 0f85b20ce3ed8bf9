// amp_anneal.cpp — the annealing search over domino-tiling placements
// (reference placement.cpp:299-398, the paper's Algorithm 2) on the engine.
//
// COMPATIBILITY PORT of placement.cpp's host-side chain (device_grid,
// the backtracking domino tiling, strategy_key, the Metropolis loop): a
// bit-exact std::mt19937_64 draw sequence forces the reference's control
// flow and draw order, so this part follows placement.cpp:68-398 closely.
// The B200 work is the proposals' DP + estimate on the GPU (below).
//
// The chain itself is sequential and host-side, as in the reference: the
// same std::mt19937_64 stream (rng.hpp:25-44), the same draw order (degree
// flip, mbs, tiling orientations with backtracking, acceptance), the same
// temperature schedule and acceptance test.  Every proposal's layer
// partition DP and cost estimate — the reference's per-iteration cost —
// run on the GPU through amp_search_evaluate_placed (K_place with the
// caller's placement, K_dp, K_est).  The recorded chain, the initial cost
// and the top-`budget` ranking (std::sort with the reference comparator)
// are returned, so a caller reproduces the reference's anneal report.
//
// This file is a client of the C ABI only (no device code).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <optional>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/amp_search.h"

namespace {

struct Rng {  // rng.hpp:25-44
  std::mt19937_64 gen;
  explicit Rng(uint64_t seed) : gen(seed) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  int below(int n) { return static_cast<int>(gen() % static_cast<uint64_t>(n)); }
};

std::vector<int> divisors(int n) {  // optimizer.cpp:29-41
  std::vector<int> out;
  for (int d = 1; d * d <= n; ++d)
    if (n % d == 0) {
      out.push_back(d);
      if (d != n / d) out.push_back(n / d);
    }
  std::sort(out.begin(), out.end());
  return out;
}

std::vector<int> enumerate_mbs(int gbs, int dp) {  // optimizer.cpp:57-62
  if (dp < 1 || gbs % dp != 0) return {};
  return divisors(gbs / dp);
}

struct Deg {
  int pp = 1, dp = 1, tmp = 1;
};

struct Grid {  // placement.cpp:68-108 device_grid
  int rows = 1, cols = 1;
  std::vector<int> cells;
  int at(int r, int c) const { return cells[r * cols + c]; }
};

struct Problem {
  int L = 0, D = 0, gbs = 0;
  std::vector<int> node;           // device -> node id
  std::vector<int> order;          // devices by (node, id)
  std::map<int, int> node_size;    // std::map, like devices_by_node()
};

Grid device_grid(const Problem& P) {
  const int n = P.D;
  Grid g;
  g.rows = 1;
  for (int r = 1; r * r <= n; ++r)
    if (n % r == 0) g.rows = r;
  g.cols = n / g.rows;
  const int node_size = P.node_size.begin()->second;  // nodes.front()
  bool uniform = true;
  for (const auto& kv : P.node_size) uniform &= kv.second == node_size;
  const bool column_major = uniform && g.cols % node_size != 0 && g.rows % node_size == 0;
  g.cells.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    const int row = column_major ? i % g.rows : i / g.cols;
    const int col = column_major ? i / g.rows : i % g.cols;
    g.cells[row * g.cols + col] = P.order[i];
  }
  return g;
}

struct Domino {
  int row, col;
  bool vertical;
};

class TilingSearch {  // placement.cpp:112-190
 public:
  TilingSearch(const Deg& d, const Grid& g, Rng& rng)
      : deg_(d), grid_(g), rng_(rng), covered_(g.cells.size(), 0) {}
  std::optional<std::vector<Domino>> run() {
    if (fill()) return dominos_;
    return std::nullopt;
  }

 private:
  bool fits(int row, int col, int h, int w) const {
    if (row + h > grid_.rows || col + w > grid_.cols) return false;
    for (int i = row; i < row + h; ++i)
      for (int j = col; j < col + w; ++j)
        if (covered_[i * grid_.cols + j]) return false;
    return true;
  }
  void mark(int row, int col, int h, int w, char v) {
    for (int i = row; i < row + h; ++i)
      for (int j = col; j < col + w; ++j) covered_[i * grid_.cols + j] = v;
  }
  bool fill() {
    const auto first = std::find(covered_.begin(), covered_.end(), 0);
    if (first == covered_.end()) return true;
    const int idx = static_cast<int>(first - covered_.begin());
    const int row = idx / grid_.cols, col = idx % grid_.cols;
    std::vector<bool> orientations;
    if (deg_.tmp == deg_.dp) {
      orientations = {rng_.uniform() < 0.5};
    } else if (rng_.uniform() < 0.5) {
      orientations = {true, false};
    } else {
      orientations = {false, true};
    }
    for (bool vertical : orientations) {
      const int h = vertical ? deg_.tmp : deg_.dp;
      const int w = vertical ? deg_.dp : deg_.tmp;
      if (!fits(row, col, h, w)) continue;
      mark(row, col, h, w, 1);
      dominos_.push_back({row, col, vertical});
      if (fill()) return true;
      dominos_.pop_back();
      mark(row, col, h, w, 0);
    }
    return false;
  }
  Deg deg_;
  const Grid& grid_;
  Rng& rng_;
  std::vector<char> covered_;
  std::vector<Domino> dominos_;
};

// sample_domino_tiling + tiling_to_placement (placement.cpp:192-229)
std::optional<std::vector<int>> sample_placement(const Deg& d, const Grid& g, Rng& rng) {
  auto dominos = TilingSearch(d, g, rng).run();
  if (!dominos) return std::nullopt;
  std::sort(dominos->begin(), dominos->end(), [](const Domino& a, const Domino& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  std::vector<int> r2d((size_t)d.pp * d.dp * d.tmp);
  for (int stage = 0; stage < d.pp; ++stage) {
    const Domino& dm = (*dominos)[stage];
    for (int r = 0; r < d.dp; ++r)
      for (int sh = 0; sh < d.tmp; ++sh) {
        const int row = dm.vertical ? dm.row + sh : dm.row + r;
        const int col = dm.vertical ? dm.col + r : dm.col + sh;
        r2d[((size_t)stage * d.dp + r) * d.tmp + sh] = g.at(row, col);
      }
  }
  return r2d;
}

struct Strat {
  Deg deg;
  int mbs = 1;
  std::vector<int> place, cuts;
  amp_record est{};
};

std::string strategy_key(const Strat& s) {  // placement.cpp:231-243
  std::string key = std::to_string(s.deg.pp) + "/" + std::to_string(s.deg.dp) + "/" +
                    std::to_string(s.deg.tmp) + "/" + std::to_string(s.mbs) + "|";
  for (int d : s.place) key += std::to_string(d) + ",";
  key += "|";
  for (int c : s.cuts) key += std::to_string(c) + ",";
  return key;
}

struct Engine {
  amp_ctx* ctx;
  int max_pp, D;
  std::map<std::tuple<int, int, int, int>, int> cls;
  amp_record failed{};
  bool has_failed = false;

  // solve_candidate + estimate for a batch of proposals on the GPU
  // (placement.cpp:252-259, cost_model.cpp:176-212).  Returns AMP_OK, an
  // engine error, or AMP_E_CANDIDATE with the failing record in `failed`
  // (the reference throws out of anneal there).
  // Batch evaluation of speculative proposals: records (failures as data)
  // and cuts for every entry; the caller decides which one was on the
  // chain's path (the reference throws only there).
  int evaluate_all(std::vector<Strat*>& v, std::vector<amp_record>& out) {
    const int n = (int)v.size();
    out.assign(n, amp_record{});
    if (n == 0) return AMP_OK;
    std::vector<int32_t> c(n), pl((size_t)n * D), cu((size_t)n * (max_pp + 1), -1);
    for (int i = 0; i < n; ++i) {
      auto it = cls.find({v[i]->deg.pp, v[i]->deg.dp, v[i]->deg.tmp, v[i]->mbs});
      if (it == cls.end()) return AMP_E_INVALID;
      c[i] = it->second;
      std::copy(v[i]->place.begin(), v[i]->place.end(), pl.begin() + (size_t)i * D);
    }
    amp_details det{};
    det.cuts = cu.data();
    const int rc = amp_search_evaluate_placed(ctx, c.data(), pl.data(), nullptr, n, out.data(), &det);
    if (rc != AMP_OK) return rc;
    for (int i = 0; i < n; ++i) {
      v[i]->est = out[i];
      v[i]->cuts.assign(cu.begin() + (size_t)i * (max_pp + 1),
                        cu.begin() + (size_t)i * (max_pp + 1) + v[i]->deg.pp + 1);
    }
    return AMP_OK;
  }

  int evaluate(std::vector<Strat*>& v) {
    const int n = (int)v.size();
    if (n == 0) return AMP_OK;
    std::vector<int32_t> c(n), pl((size_t)n * D), cu((size_t)n * (max_pp + 1), -1);
    for (int i = 0; i < n; ++i) {
      auto it = cls.find({v[i]->deg.pp, v[i]->deg.dp, v[i]->deg.tmp, v[i]->mbs});
      if (it == cls.end()) return AMP_E_INVALID;
      c[i] = it->second;
      std::copy(v[i]->place.begin(), v[i]->place.end(), pl.begin() + (size_t)i * D);
    }
    std::vector<amp_record> out(n);
    amp_details det{};
    det.cuts = cu.data();
    const int rc = amp_search_evaluate_placed(ctx, c.data(), pl.data(), nullptr, n, out.data(), &det);
    if (rc != AMP_OK) return rc;
    for (int i = 0; i < n; ++i) {
      if (out[i].fail_code != AMP_FAIL_NONE) {
        failed = out[i];
        has_failed = true;
        return AMP_E_CANDIDATE;
      }
      v[i]->est = out[i];
      v[i]->cuts.assign(cu.begin() + (size_t)i * (max_pp + 1),
                        cu.begin() + (size_t)i * (max_pp + 1) + v[i]->deg.pp + 1);
    }
    return AMP_OK;
  }
};

int megatron_choice(const Problem& P, int mbs, Deg* out) {  // optimizer.cpp:64-79
  int min_node = P.D;
  for (const auto& kv : P.node_size) min_node = std::min(min_node, kv.second);
  bool found = false;
  Deg best;
  for (int pp : divisors(P.D))
    for (int dp : divisors(P.D / pp)) {
      const Deg d{pp, dp, P.D / (pp * dp)};
      if (d.tmp > min_node || d.pp > P.L) continue;
      if (P.gbs % d.dp != 0 || (P.gbs / d.dp) % mbs != 0) continue;
      if (!found || std::pair(d.tmp * d.pp, d.tmp) < std::pair(best.tmp * best.pp, best.tmp)) {
        best = d;
        found = true;
      }
    }
  if (found) *out = best;
  return found;
}

}  // namespace

extern "C" int amp_search_anneal(amp_ctx* ctx, const amp_problem* problem,
                                 const amp_anneal_config* cfg, amp_anneal_entry* record,
                                 int32_t* record_place, int32_t* record_cuts, int32_t cap,
                                 int32_t* n_record, int32_t* top, int32_t* n_top,
                                 double* initial_cost, amp_record* failed) {
  if (!ctx || !problem || !cfg || !record || !n_record || !n_top || !initial_cost)
    return AMP_E_INVALID;
  if (cfg->iterations < 1) return AMP_E_INVALID;  // "anneal needs at least one iteration"
  Problem P;
  P.L = problem->n_layers;
  P.D = problem->n_devices;
  P.gbs = problem->gbs;
  P.node.assign(problem->node_id, problem->node_id + P.D);
  P.order.resize(P.D);
  for (int i = 0; i < P.D; ++i) {
    P.order[i] = i;
    P.node_size[P.node[i]] += 1;
  }
  std::sort(P.order.begin(), P.order.end(), [&](int a, int b) {
    return P.node[a] != P.node[b] ? P.node[a] < P.node[b] : a < b;
  });
  Engine E;
  E.ctx = ctx;
  E.max_pp = amp_search_max_pp(ctx);
  E.D = P.D;
  for (int c = 0; c < amp_search_num_classes(ctx); ++c) {
    int32_t pp, dp, tmp, mbs;
    amp_search_class(ctx, c, &pp, &dp, &tmp, &mbs);
    E.cls[{pp, dp, tmp, mbs}] = c;
  }
  auto fail_out = [&](int rc) {
    if (rc == AMP_E_CANDIDATE && failed) *failed = E.failed;
    return rc;
  };

  // ---- initial_strategy (placement.cpp:261-297) -----------------------------
  std::vector<Strat> init;
  for (int mbs : divisors(P.gbs)) {
    Deg d;
    if (!megatron_choice(P, mbs, &d)) continue;
    Strat s;
    s.deg = d;
    s.mbs = mbs;
    s.place = P.order;  // heuristic_placement
    init.push_back(s);
  }
  Strat current;
  if (!init.empty()) {
    // each initial candidate is solved and estimated in order; the reference
    // throws at the first failing one, so evaluate one at a time up to it
    std::optional<size_t> best;
    for (size_t i = 0; i < init.size(); ++i) {
      std::vector<Strat*> one{&init[i]};
      const int rc = E.evaluate(one);
      if (rc != AMP_OK) return fail_out(rc);
      if (!best || init[i].est.total < init[*best].est.total) best = i;
    }
    current = init[*best];
  } else {
    bool found = false;
    for (int pp : divisors(P.D)) {
      for (int dp : divisors(P.D / pp)) {
        const Deg d{pp, dp, P.D / (pp * dp)};
        if (d.pp > P.L) continue;
        const auto m = enumerate_mbs(P.gbs, d.dp);
        if (m.empty()) continue;
        current.deg = d;
        current.mbs = m.front();
        current.place = P.order;
        found = true;
        break;
      }
      if (found) break;
    }
    if (!found) return AMP_E_INVALID;  // "no feasible strategy exists ..."
    std::vector<Strat*> one{&current};
    const int rc = E.evaluate(one);
    if (rc != AMP_OK) return fail_out(rc);
  }

  // ---- the chain (placement.cpp:318-370) -------------------------------------
  Rng rng(cfg->seed);
  const Grid grid = device_grid(P);
  std::map<std::string, int> recorded;
  int nrec = 0;
  auto record_state = [&](const Strat& s, int iteration, bool accepted) -> int {
    const std::string key = strategy_key(s);
    if (recorded.count(key)) return AMP_OK;
    if (nrec >= cap) return AMP_E_INVALID;
    recorded[key] = nrec;
    amp_anneal_entry& e = record[nrec];
    std::memset(&e, 0, sizeof e);
    e.estimated = s.est;
    e.iteration = iteration;
    e.accepted = accepted ? 1 : 0;
    if (record_place)
      std::copy(s.place.begin(), s.place.end(), record_place + (size_t)nrec * P.D);
    if (record_cuts) {
      int32_t* c = record_cuts + (size_t)nrec * (E.max_pp + 1);
      std::fill(c, c + E.max_pp + 1, -1);
      std::copy(s.cuts.begin(), s.cuts.end(), c);
    }
    ++nrec;
    return AMP_OK;
  };
  *initial_cost = current.est.total;
  if (record_state(current, 0, true) != AMP_OK) return AMP_E_INVALID;
  // The chain, speculatively: the mt19937_64 stream is the same on the
  // accept and the reject branch (the acceptance draw happens either way),
  // and a proposal depends only on the current state and that stream — not
  // on any cost.  So the proposals of every branch of the next `depth`
  // iterations (a binary tree: accept / reject) are generated on the host
  // first, evaluated in ONE batched GPU call (amp_search_evaluate_placed),
  // and the chain then walks the tree with the real costs: bit-identical to
  // the sequential chain, `depth` iterations per GPU round trip.
  // AMP_ANNEAL_DEPTH (default 6; 1 = the sequential chain).
  double temperature = cfg->initial_temperature;
  const int n = P.D;
  const char* dv = std::getenv("AMP_ANNEAL_DEPTH");
  const int spec = std::max(1, std::min(12, dv ? std::atoi(dv) : 6));
  struct Node {
    Strat cur;                  // state entering the iteration (degrees, mbs, placement)
    Rng rng_in, rng_out;        // the stream entering / leaving the iteration
    std::optional<Strat> next;  // its proposal (none: every attempt failed)
    double u = 0.0;             // the acceptance draw
    int child[2] = {-1, -1};    // [reject, accept] (no proposal: child[0] only)
  };
  auto propose = [&](const Strat& cur, Rng& r) {  // placement.cpp:329-359
    std::optional<Strat> next;
    for (int attempt = 0; attempt < cfg->neighbor_retries && !next; ++attempt) {
      Deg deg = cur.deg;
      if (r.uniform() > 0.5) {
        const auto choices = divisors(n / deg.dp);
        deg.tmp = choices[r.below(static_cast<int>(choices.size()))];
      } else {
        const auto choices = divisors(n / deg.tmp);
        deg.dp = choices[r.below(static_cast<int>(choices.size()))];
      }
      deg.pp = n / (deg.dp * deg.tmp);
      if (deg.pp > P.L) continue;
      const auto mbs_options = enumerate_mbs(P.gbs, deg.dp);
      if (mbs_options.empty()) continue;
      const int mbs = mbs_options[r.below(static_cast<int>(mbs_options.size()))];
      auto place = sample_placement(deg, grid, r);
      if (!place) continue;
      Strat st;
      st.deg = deg;
      st.mbs = mbs;
      st.place = std::move(*place);
      next = std::move(st);
    }
    return next;
  };
  for (int i = 1; i <= cfg->iterations;) {
    const int depth = std::min(spec, cfg->iterations - i + 1);
    std::vector<Node> tree;
    tree.reserve((size_t)2 << depth);
    tree.push_back(Node{current, rng, rng, std::nullopt});
    std::vector<int> level{0};
    for (int l = 0; l < depth; ++l) {
      std::vector<int> nxt;
      for (int id : level) {
        Rng r = tree[id].rng_in;
        std::optional<Strat> prop = propose(tree[id].cur, r);
        if (prop) tree[id].u = r.uniform();  // drawn on both branches
        tree[id].rng_out = r;
        tree[id].next = std::move(prop);
        if (l + 1 == depth) continue;
        const Strat cur = tree[id].cur;
        const std::optional<Strat> acc = tree[id].next;
        tree[id].child[0] = (int)tree.size();
        tree.push_back(Node{cur, r, r, std::nullopt});
        nxt.push_back(tree[id].child[0]);
        if (acc) {
          tree[id].child[1] = (int)tree.size();
          tree.push_back(Node{*acc, r, r, std::nullopt});
          nxt.push_back(tree[id].child[1]);
        }
      }
      level = std::move(nxt);
    }
    std::vector<Strat*> props;
    for (Node& nd : tree)
      if (nd.next) props.push_back(&*nd.next);
    std::vector<amp_record> recs;
    const int rc = E.evaluate_all(props, recs);  // solve_candidate + estimate, every branch
    if (rc != AMP_OK) return fail_out(rc);
    // walk the tree with the real costs (placement.cpp:360-370)
    int id = 0;
    for (int l = 0; l < depth; ++l, ++i) {
      temperature = std::max(temperature * cfg->cooling, cfg->min_temperature);
      Node& nd = tree[id];
      rng = nd.rng_out;
      if (!nd.next) {  // keep the current state
        if (l + 1 < depth) id = nd.child[0];
        continue;
      }
      Strat& nx = *nd.next;
      if (nx.est.fail_code != AMP_FAIL_NONE) {  // the reference throws here
        E.failed = nx.est;
        E.has_failed = true;
        return fail_out(AMP_E_CANDIDATE);
      }
      const double acc_prob = std::exp(std::min(current.est.total - nx.est.total, 0.0) / temperature);
      const bool accept = nd.u < acc_prob;
      if (accept) {
        current = nx;
        if (record_state(current, i, true) != AMP_OK) return AMP_E_INVALID;
      } else if (cfg->record_all) {
        if (record_state(nx, i, false) != AMP_OK) return AMP_E_INVALID;
      }
      if (l + 1 < depth) id = nd.child[accept ? 1 : 0];
    }
  }
  *n_record = nrec;

  // ---- top `budget` by (total, degrees, mbs) (placement.cpp:372-395) ------------
  std::vector<size_t> order(nrec);
  for (int i = 0; i < nrec; ++i) order[i] = (size_t)i;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const amp_record& ra = record[a].estimated;
    const amp_record& rb = record[b].estimated;
    if (ra.total != rb.total) return ra.total < rb.total;
    return std::tuple(ra.pp, ra.dp, ra.tmp, ra.mbs) < std::tuple(rb.pp, rb.dp, rb.tmp, rb.mbs);
  });
  int nt = 0;
  for (size_t i = 0; i < order.size() && i < (size_t)std::max(0, cfg->budget); ++i)
    if (top) top[nt++] = (int32_t)order[i];
  *n_top = nt;
  return AMP_OK;
}
