// parplan_plan_gpu.cpp — drop-in GPU replacement for parplan::plan.
//
// This is the host code a parplan maintainer compiles into the reference
// library: it keeps parplan::plan's signature and
// semantics (proj/include/parplan/optimizer.hpp:74-75) and replaces the
// worker pool + evaluate_candidate + rank_records region
// (proj/src/optimizer.cpp:202-231) with one call into the B200 engine through
// the C ABI of include/amp_search.h.  The simulator validation of the top
// `budget` stays the reference's own simulate() (optimizer.cpp:235-249).
//
// Build: g++ -std=c++20 -I<parplan>/include -I<repo>/include -c parplan_plan_gpu.cpp
//        and link <repo>/paper_2210_07297_b200/libamp_search.so
#include "parplan_plan_gpu.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "amp_search.h"
#include "parplan/simulator.hpp"

namespace parplan_gpu {

namespace {

using namespace parplan;

// std::to_string(double) as used in the reference's messages.
std::string failure_text(const amp_record& r, int L) {
  switch (r.fail_code) {
    case AMP_FAIL_PP_GT_L:  // optimizer.cpp:149-152
      return "infeasible: pp = " + std::to_string(r.pp) + " exceeds layer count " +
             std::to_string(L);
    case AMP_FAIL_PROFILE_MISS:  // types.cpp:106-110
      return ProfileMissError(r.fail_layer, r.tmp, r.mbs).what();
    case AMP_FAIL_CEILING:  // optimizer.cpp:165-167
      return "exceeds per-device parameter ceiling";
    case AMP_FAIL_P2P_BANDWIDTH:  // cost_model.cpp:54-59
      return "invalid p2p bandwidth " + std::to_string(r.fail_value);
    case AMP_FAIL_ALLREDUCE_BANDWIDTH:  // cost_model.cpp:47-50
      return "invalid bandwidth " + std::to_string(r.fail_value) + " in all-reduce group";
    default:
      return "unknown failure";
  }
}

struct Encoded {
  std::vector<double> param, flops, act, bw, seconds;
  std::vector<uint8_t> flops_ok;
  std::vector<int32_t> node, layer, tmp, mbs;
  amp_problem p{};
};

void encode(const ModelGraph& model, const Cluster& cluster, const ProfileTable& profile, int gbs,
            const PlanOptions& o, Encoded& e) {
  const int L = model.layer_count(), D = cluster.device_count();
  for (const auto& l : model.layers) {
    e.param.push_back(l.param_count);
    e.flops.push_back(l.flops_per_sample.value_or(0.0));
    e.flops_ok.push_back(l.flops_per_sample.has_value());
  }
  e.act = model.activation_volumes;
  if (e.act.empty()) e.act.push_back(0.0);
  e.node.resize(D);
  for (const auto& d : cluster.devices) e.node[d.id] = d.node_id;
  e.bw.resize((size_t)D * D);
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) e.bw[(size_t)i * D + j] = cluster.link(i, j);
  for (const auto& [key, s] : profile.entries()) {
    e.layer.push_back(key.layer);
    e.tmp.push_back(key.tmp);
    e.mbs.push_back(key.mbs);
    e.seconds.push_back(s);
  }
  amp_problem& p = e.p;
  p.n_layers = L;
  p.n_devices = D;
  p.gbs = gbs;
  p.fallback_enabled = o.cost_options.fallback.enabled;
  p.param_count = e.param.data();
  p.flops_per_sample = e.flops.data();
  p.flops_present = e.flops_ok.data();
  p.activation_volumes = e.act.data();
  p.node_id = e.node.data();
  p.bandwidth = e.bw.data();
  p.n_profile_entries = (int64_t)e.layer.size();
  p.profile_layer = e.layer.data();
  p.profile_tmp = e.tmp.data();
  p.profile_mbs = e.mbs.data();
  p.profile_seconds = e.seconds.data();
  p.bytes_per_param = o.cost_options.bytes_per_param;
  p.fallback_device_flops = o.cost_options.fallback.device_flops;
  p.fallback_tmp_bandwidth = o.cost_options.fallback.tmp_bandwidth;
  p.has_max_params_per_device = o.max_params_per_device.has_value();
  p.max_params_per_device = o.max_params_per_device.value_or(0.0);
}

}  // namespace

PlanResult plan(const ModelGraph& model, const Cluster& cluster, const ProfileTable& profile,
                int gbs, const PlanOptions& options, int device, int n_gpus) {
  Encoded e;
  encode(model, cluster, profile, gbs, options, e);
  amp_search_config cfg{};
  cfg.placements_per_class = 1;  // the plan() candidate list
  cfg.device = device;
  cfg.n_gpus = n_gpus;  // > 1: one context drives the GPUs (LPT shards, NCCL all-gather)
  amp_ctx* ctx = nullptr;
  if (int rc = amp_search_create(&ctx, &e.p, &cfg); rc != AMP_OK)
    throw std::runtime_error(std::string("amp_search_create: ") + amp_last_error());
  const uint64_t n = amp_search_num_candidates(ctx);
  const int max_pp = amp_search_max_pp(ctx);
  const int D = cluster.device_count();
  std::vector<amp_record> recs(n);
  std::vector<int32_t> cuts(n * (max_pp + 1)), place(n * D);
  std::vector<double> stage(n * max_pp), edge(n * max_pp);
  amp_details det{cuts.data(), stage.data(), edge.data(), place.data()};
  int32_t ntop = 0;
  const int rc = amp_search_run(ctx, 0, n, 0, nullptr, &ntop, recs.data(), &det);
  const std::string err = rc == AMP_OK ? "" : amp_search_last_error(ctx);
  amp_search_destroy(ctx);
  if (rc != AMP_OK) throw std::runtime_error("amp_search_run: " + err);

  // rank_records key (optimizer.cpp:178-196): index order == (pp, dp, tmp, mbs)
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const bool fa = recs[a].fail_code != 0, fb = recs[b].fail_code != 0;
    if (fa != fb) return !fa;
    if (!fa && recs[a].total != recs[b].total) return recs[a].total < recs[b].total;
    return recs[a].index < recs[b].index;
  });
  PlanResult result;
  result.candidates.resize(n);
  for (size_t r = 0; r < n; ++r) {
    const size_t i = order[r];
    const amp_record& a = recs[i];
    CandidateRecord& c = result.candidates[r];
    c.strategy.degrees = ParallelismDegrees{a.pp, a.dp, a.tmp};
    c.strategy.mbs = a.mbs;
    c.rank = (int)r + 1;
    // evaluate_candidate assigns record.strategy before the parameter
    // ceiling and estimate (optimizer.cpp:157-171): those two failures keep
    // the placement and the DP cuts
    if (a.fail_code == 0 || a.fail_code == AMP_FAIL_CEILING || a.fail_code == AMP_FAIL_ALLREDUCE_BANDWIDTH) {
      c.strategy.placement = Placement(
          c.strategy.degrees, std::vector<int>(place.begin() + i * D, place.begin() + (i + 1) * D));
      c.strategy.assignment.cut_boundaries.assign(cuts.begin() + i * (max_pp + 1),
                                                  cuts.begin() + i * (max_pp + 1) + a.pp + 1);
    }
    if (a.fail_code != 0) {
      c.failure = failure_text(a, model.layer_count());
      continue;
    }
    c.estimated.total = a.total;
    c.estimated.pipeline_time = a.pipeline_time;
    c.estimated.dpsync_time = a.dpsync_time;
    c.estimated.per_stage_times.assign(stage.begin() + i * max_pp,
                                       stage.begin() + i * max_pp + a.pp);
    c.estimated.per_edge_times.assign(edge.begin() + i * max_pp,
                                      edge.begin() + i * max_pp + a.pp - 1);
  }
  // Validate the top predicted strategies with the simulator
  // (optimizer.cpp:235-249, unchanged).
  for (size_t i = 0; i < result.candidates.size() && i < static_cast<size_t>(options.budget);
       ++i) {
    auto& record = result.candidates[i];
    if (record.failure) continue;
    SimOptions sim_options;
    sim_options.cost_options = options.cost_options;
    record.simulated =
        simulate(record.strategy, model, cluster, profile, gbs, sim_options).iteration_time;
    if (result.best_index < 0 ||
        *record.simulated < *result.candidates[result.best_index].simulated)
      result.best_index = static_cast<int>(i);
  }
  return result;
}

}  // namespace parplan_gpu
