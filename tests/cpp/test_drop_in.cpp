// test_drop_in.cpp — the C++ drop-in shim against the reference itself.
//
// Builds seeded worlds the way the reference's own tests do
// (proj/tests/test_optimizer.cpp:30-68 make_cluster/make_model/full_profile)
// and checks that parplan_gpu::plan (GPU engine through the C ABI) returns
// exactly what parplan::plan returns in the same process: ranking, every
// strategy field, every CostBreakdown double, simulated times, failure
// texts and best_index.  Exit status 0 on full agreement.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "parplan/optimizer.hpp"
#include "parplan_plan_gpu.hpp"

using namespace parplan;

namespace {

int g_fail = 0;

#define EXPECT(cond, ...)                                   \
  do {                                                      \
    if (!(cond)) {                                          \
      if (g_fail < 20) {                                    \
        std::printf("MISMATCH %s:%d: ", __FILE__, __LINE__); \
        std::printf(__VA_ARGS__);                           \
        std::printf("\n");                                  \
      }                                                     \
      ++g_fail;                                             \
    }                                                       \
  } while (0)

bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

Cluster make_cluster(int devices, int nodes, double intra, double inter, std::mt19937_64& g) {
  Cluster cluster;
  const int per_node = devices / nodes;
  for (int i = 0; i < devices; ++i) cluster.devices.push_back({i, i / per_node, "gpu"});
  cluster.bandwidth.assign(devices, std::vector<double>(devices, inter));
  for (int i = 0; i < devices; ++i) {
    for (int j = 0; j < devices; ++j)
      if (i / per_node == j / per_node) cluster.bandwidth[i][j] = intra * (1 + (i / per_node) % 2);
    cluster.bandwidth[i][i] = kInfiniteBandwidth;
  }
  // a few asymmetric-tier links (kept symmetric)
  for (int t = 0; t < devices / 2; ++t) {
    const int a = (int)(g() % devices), b = (int)(g() % devices);
    if (a == b) continue;
    cluster.bandwidth[a][b] = cluster.bandwidth[b][a] = inter * 0.5;
  }
  return cluster;
}

ModelGraph make_model(int L, std::mt19937_64& g) {
  std::uniform_real_distribution<double> pos(0.5, 3.0);
  ModelGraph model;
  for (int i = 0; i < L; ++i) model.layers.push_back({i, "block", pos(g) * 1e6, pos(g) * 1e10});
  for (int i = 0; i + 1 < L; ++i) model.activation_volumes.push_back(pos(g) * 1e6);
  return model;
}

ProfileTable full_profile(const ModelGraph& m, int devices, int gbs, std::mt19937_64& g,
                          bool holes) {
  std::uniform_real_distribution<double> pos(0.5, 3.0);
  ProfileTable profile;
  for (int layer = 0; layer < m.layer_count(); ++layer) {
    const double scale = pos(g);
    for (int tmp : divisors(devices))
      for (int mbs : divisors(gbs)) {
        if (holes && tmp >= 4 && layer == m.layer_count() / 2) continue;
        profile.set(layer, tmp, mbs, 0.001 * mbs * scale / tmp);
      }
  }
  return profile;
}

void compare(const PlanResult& a, const PlanResult& b, const char* tag) {
  EXPECT(a.candidates.size() == b.candidates.size(), "%s: sizes %zu vs %zu", tag,
         a.candidates.size(), b.candidates.size());
  EXPECT(a.best_index == b.best_index, "%s: best_index %d vs %d", tag, a.best_index, b.best_index);
  for (size_t i = 0; i < a.candidates.size() && i < b.candidates.size(); ++i) {
    const auto& x = a.candidates[i];
    const auto& y = b.candidates[i];
    EXPECT(x.rank == y.rank, "%s[%zu] rank", tag, i);
    EXPECT(x.strategy.degrees == y.strategy.degrees && x.strategy.mbs == y.strategy.mbs,
           "%s[%zu] degrees/mbs", tag, i);
    EXPECT(x.failure == y.failure, "%s[%zu] failure '%s' vs '%s'", tag, i,
           x.failure.value_or("").c_str(), y.failure.value_or("").c_str());
    // (failed records too: the ceiling / all-reduce failures keep their strategy)
    EXPECT(x.strategy.placement == y.strategy.placement, "%s[%zu] placement", tag, i);
    EXPECT(x.strategy.assignment == y.strategy.assignment, "%s[%zu] cuts", tag, i);
    if (x.failure || y.failure) continue;
    EXPECT(same(x.estimated.total, y.estimated.total), "%s[%zu] total %a vs %a", tag, i,
           x.estimated.total, y.estimated.total);
    EXPECT(same(x.estimated.pipeline_time, y.estimated.pipeline_time), "%s[%zu] pipeline", tag, i);
    EXPECT(same(x.estimated.dpsync_time, y.estimated.dpsync_time), "%s[%zu] dpsync", tag, i);
    EXPECT(x.estimated.per_stage_times.size() == y.estimated.per_stage_times.size(),
           "%s[%zu] stage count", tag, i);
    for (size_t q = 0; q < x.estimated.per_stage_times.size(); ++q)
      EXPECT(same(x.estimated.per_stage_times[q], y.estimated.per_stage_times[q]),
             "%s[%zu] stage %zu", tag, i, q);
    EXPECT(x.estimated.per_edge_times.size() == y.estimated.per_edge_times.size(),
           "%s[%zu] edge count", tag, i);
    for (size_t q = 0; q < x.estimated.per_edge_times.size(); ++q)
      EXPECT(same(x.estimated.per_edge_times[q], y.estimated.per_edge_times[q]),
             "%s[%zu] edge %zu", tag, i, q);
    EXPECT(x.simulated.has_value() == y.simulated.has_value() &&
               (!x.simulated || same(*x.simulated, *y.simulated)),
           "%s[%zu] simulated", tag, i);
  }
}

}  // namespace

int main(int argc, char** argv) {
  // argv[1]: GPUs per context (the drop-in drives devices 0 .. n-1 itself)
  const int n_gpus = argc > 1 ? std::atoi(argv[1]) : 1;
  std::printf("n_gpus = %d\n", n_gpus);
  std::mt19937_64 g(2210);
  int worlds = 0;
  for (int trial = 0; trial < 24; ++trial) {
    const int devices = trial % 3 == 0 ? 4 : (trial % 3 == 1 ? 8 : 16);
    const int nodes = devices >= 8 ? devices / 4 : 1;
    const int L = 3 + (int)(g() % 18);
    const int gbs = trial % 2 ? 16 : 32;
    Cluster cluster = make_cluster(devices, nodes, 100e9, 10e9, g);
    ModelGraph model = make_model(L, g);
    PlanOptions o;
    o.budget = 10;
    o.workers = 4;
    ProfileTable profile;
    switch (trial % 4) {
      case 0:
        profile = full_profile(model, devices, gbs, g, false);
        break;
      case 1:
        profile = full_profile(model, devices, gbs, g, true);  // profile misses
        break;
      case 2:  // analytic fallback, no profile
        o.cost_options.fallback.enabled = true;
        o.cost_options.fallback.device_flops = 1e14;
        o.cost_options.fallback.tmp_bandwidth = 50e9;
        break;
      case 3:
        profile = full_profile(model, devices, gbs, g, false);
        o.max_params_per_device = 4e6;  // ceiling failures
        break;
    }
    const PlanResult ref = parplan::plan(model, cluster, profile, gbs, o);
    const PlanResult gpu = parplan_gpu::plan(model, cluster, profile, gbs, o, 0, n_gpus);
    char tag[64];
    std::snprintf(tag, sizeof tag, "world%d(L=%d,D=%d)", trial, L, devices);
    compare(gpu, ref, tag);
    ++worlds;
  }
  std::printf("%s: %d worlds, %d mismatches\n", g_fail ? "FAIL" : "ALL OK", worlds, g_fail);
  return g_fail ? 1 : 0;
}
