// ref_bridge.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI wrapper around the UNMODIFIED reference library so that tests and
// the bench's CPU arm can call it through ctypes.  oracle/Makefile compiles
// this file together with the reference sources where they lie
// (/root/reference/proj/src/{types,cost_model,pipeline_dp,placement,
// optimizer,simulator}.cpp) into oracle/_ref/libparplan_ref.so.  Nothing here
// re-implements reference arithmetic except the two pieces the survey names
// as the sweep driver's restatements: the splitmix64 shuffle of the device
// order and the 3-line placement_edge_cost
// (optimizer.cpp:130-139, which is in an anonymous namespace upstream).
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../include/amp_search.h"
#include "parplan/cost_model.hpp"
#include "parplan/optimizer.hpp"
#include "parplan/pipeline_dp.hpp"
#include "parplan/placement.hpp"
#include "parplan/simulator.hpp"
#include "parplan/types.hpp"

using namespace parplan;

namespace {

struct World {
  ModelGraph model;
  Cluster cluster;
  ProfileTable profile;
  CostModelOptions cost;
  std::optional<double> ceiling;
  int gbs = 1;
};

World make_world(const amp_problem* p) {
  World w;
  const int L = p->n_layers, D = p->n_devices;
  for (int i = 0; i < L; ++i) {
    LayerSpec spec;
    spec.id = i;
    spec.kind = "layer";
    spec.param_count = p->param_count[i];
    if (p->flops_present && p->flops_present[i]) spec.flops_per_sample = p->flops_per_sample[i];
    w.model.layers.push_back(spec);
  }
  w.model.activation_volumes.assign(p->activation_volumes, p->activation_volumes + (L - 1));
  for (int d = 0; d < D; ++d) w.cluster.devices.push_back({d, p->node_id[d], "gpu"});
  w.cluster.bandwidth.assign(D, std::vector<double>(D));
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j)
      w.cluster.bandwidth[i][j] = i == j ? kInfiniteBandwidth : p->bandwidth[(size_t)i * D + j];
  for (int64_t e = 0; e < p->n_profile_entries; ++e)
    w.profile.set(p->profile_layer[e], p->profile_tmp[e], p->profile_mbs[e], p->profile_seconds[e]);
  w.cost.bytes_per_param = p->bytes_per_param;
  w.cost.fallback.enabled = p->fallback_enabled != 0;
  w.cost.fallback.device_flops = p->fallback_device_flops;
  w.cost.fallback.tmp_bandwidth = p->fallback_tmp_bandwidth;
  if (p->has_max_params_per_device) w.ceiling = p->max_params_per_device;
  w.gbs = p->gbs;
  return w;
}

std::vector<std::tuple<int, int, int, int>> class_list(const World& w) {
  std::vector<std::tuple<int, int, int, int>> out;
  for (const auto& d : enumerate_degrees(w.cluster.device_count()))
    for (int mbs : enumerate_mbs(w.gbs, d.dp)) out.emplace_back(d.pp, d.dp, d.tmp, mbs);
  return out;
}

int fail_code_of(const std::string& what) {
  if (what.rfind("infeasible: pp", 0) == 0) return AMP_FAIL_PP_GT_L;
  if (what.rfind("profile miss", 0) == 0) return AMP_FAIL_PROFILE_MISS;
  if (what.find("ceiling") != std::string::npos) return AMP_FAIL_CEILING;
  if (what.rfind("invalid p2p bandwidth", 0) == 0) return AMP_FAIL_P2P_BANDWIDTH;
  if (what.find("in all-reduce group") != std::string::npos) return AMP_FAIL_ALLREDUCE_BANDWIDTH;
  return 99;
}

void fill_record(const CandidateRecord& r, uint64_t index, int maxpp, amp_record* rec,
                 int32_t* cuts, double* stage, double* edge, char* text, int text_stride) {
  std::memset(rec, 0, sizeof(*rec));
  rec->index = index;
  rec->pp = r.strategy.degrees.pp;
  rec->dp = r.strategy.degrees.dp;
  rec->tmp = r.strategy.degrees.tmp;
  rec->mbs = r.strategy.mbs;
  rec->fail_layer = -1;
  if (cuts)
    for (int q = 0; q <= maxpp; ++q) cuts[q] = -1;
  if (stage)
    for (int q = 0; q < maxpp; ++q) stage[q] = NAN;
  if (edge)
    for (int q = 0; q < maxpp; ++q) edge[q] = NAN;
  if (text && text_stride > 0) text[0] = 0;
  if (r.failure) {
    rec->fail_code = fail_code_of(*r.failure);
    rec->total = rec->pipeline_time = rec->dpsync_time = NAN;
    if (text && text_stride > 0) {
      std::strncpy(text, r.failure->c_str(), text_stride - 1);
      text[text_stride - 1] = 0;
    }
    return;
  }
  rec->total = r.estimated.total;
  rec->pipeline_time = r.estimated.pipeline_time;
  rec->dpsync_time = r.estimated.dpsync_time;
  if (cuts)
    for (size_t q = 0; q < r.strategy.assignment.cut_boundaries.size(); ++q)
      cuts[q] = r.strategy.assignment.cut_boundaries[q];
  if (stage)
    for (size_t q = 0; q < r.estimated.per_stage_times.size(); ++q)
      stage[q] = r.estimated.per_stage_times[q];
  if (edge)
    for (size_t q = 0; q < r.estimated.per_edge_times.size(); ++q)
      edge[q] = r.estimated.per_edge_times[q];
}

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Sweep driver, one candidate: the reference call chain of
// evaluate_candidate (optimizer.cpp:141-176) with the placement replaced by
// the shuffled heuristic order for p >= 1.
CandidateRecord sweep_candidate(const World& w, const ParallelismDegrees& degrees, int mbs,
                                uint64_t p, uint64_t seed) {
  CandidateRecord record;
  record.strategy.degrees = degrees;
  record.strategy.mbs = mbs;
  try {
    if (degrees.pp > w.model.layer_count()) {
      throw ValidationError("infeasible: pp = " + std::to_string(degrees.pp) +
                            " exceeds layer count " + std::to_string(w.model.layer_count()));
    }
    Placement placement = heuristic_placement(degrees, w.cluster).placement;
    if (p != 0) {
      std::vector<int> order = placement.flat();
      uint64_t r = splitmix64(seed ^ p);
      for (int k = static_cast<int>(order.size()) - 1; k >= 1; --k) {
        std::swap(order[k], order[r % static_cast<uint64_t>(k + 1)]);
        r = splitmix64(r);
      }
      placement = Placement(degrees, std::move(order));
    }
    const LayerTimeResolver resolver(w.model, w.profile, w.cost);
    const int gas = w.gbs / (degrees.dp * mbs);
    std::vector<double> bandwidths;
    for (int q = 0; q + 1 < degrees.pp; ++q)
      bandwidths.push_back(min_edge_bandwidth(placement, w.cluster, q));
    const ModelGraph& model = w.model;
    const EdgeCostFn edge = [&model, mbs, bandwidths](int cut_layer, int edge_index) {
      return p2p_time(model.activation_volumes[cut_layer - 1] * mbs, bandwidths[edge_index]);
    };
    auto solved = optimal_assignment(w.model, degrees.pp, gas, degrees.tmp, mbs, resolver, edge);
    record.strategy = Strategy{degrees, placement, mbs, std::move(solved.assignment)};
    if (w.ceiling) {
      double worst = 0.0;
      for (int j = 0; j < degrees.pp; ++j)
        worst = std::max(worst, w.model.params_in_range(record.strategy.assignment.stage_begin(j),
                                                        record.strategy.assignment.stage_end(j)) /
                                    degrees.tmp);
      if (worst > *w.ceiling) throw ValidationError("exceeds per-device parameter ceiling");
    }
    record.estimated = estimate(record.strategy, w.model, w.cluster, w.profile, w.gbs, w.cost);
  } catch (const std::exception& e) {
    record.failure = e.what();
  }
  return record;
}

}  // namespace

extern "C" {

// parplan::plan on the problem; candidates written in RANKED order with
// their class index in amp_record.index.  simulated[n] is NaN when not run.
int ref_plan(const amp_problem* p, int32_t budget, int32_t workers, amp_record* out,
             int32_t* cuts, double* stage, double* edge, double* simulated,
             int32_t* best_index, char* fail_text, int32_t fail_text_stride, int32_t max_pp) {
  try {
    World w = make_world(p);
    const auto classes = class_list(w);
    PlanOptions o;
    o.budget = budget;
    o.workers = workers;
    o.cost_options = w.cost;
    o.max_params_per_device = w.ceiling;
    PlanResult r = plan(w.model, w.cluster, w.profile, w.gbs, o);
    for (size_t i = 0; i < r.candidates.size(); ++i) {
      const auto& c = r.candidates[i];
      uint64_t idx = 0;
      for (size_t k = 0; k < classes.size(); ++k)
        if (classes[k] == std::make_tuple(c.strategy.degrees.pp, c.strategy.degrees.dp,
                                          c.strategy.degrees.tmp, c.strategy.mbs))
          idx = k;
      fill_record(c, idx, max_pp, &out[i], cuts ? cuts + i * (max_pp + 1) : nullptr,
                  stage ? stage + i * max_pp : nullptr, edge ? edge + i * max_pp : nullptr,
                  fail_text ? fail_text + i * fail_text_stride : nullptr, fail_text_stride);
      if (simulated) simulated[i] = c.simulated ? *c.simulated : NAN;
    }
    if (best_index) *best_index = r.best_index;
    return static_cast<int>(r.candidates.size());
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_num_classes(const amp_problem* p) {
  World w = make_world(p);
  return static_cast<int>(class_list(w).size());
}

// Sweep: evaluate [begin, end) of the class-major space (P placements per
// class) on `threads` std::threads, outputs in index order.
int ref_sweep(const amp_problem* p, uint64_t P, uint64_t seed, uint64_t begin, uint64_t end,
              int32_t threads, amp_record* out, int32_t* cuts, double* stage, double* edge,
              char* fail_text, int32_t fail_text_stride, int32_t max_pp) {
  try {
    World w = make_world(p);
    const auto classes = class_list(w);
    const uint64_t n = end - begin;
    std::atomic<uint64_t> next{0};
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    auto work = [&] {
      for (uint64_t i; (i = next.fetch_add(1)) < n;) {
        const uint64_t idx = begin + i;
        const auto& [pp, dp, tmp, mbs] = classes[idx / P];
        CandidateRecord r = sweep_candidate(w, ParallelismDegrees{pp, dp, tmp}, mbs, idx % P, seed);
        fill_record(r, idx, max_pp, &out[i], cuts ? cuts + i * (max_pp + 1) : nullptr,
                    stage ? stage + i * max_pp : nullptr, edge ? edge + i * max_pp : nullptr,
                    fail_text ? fail_text + i * fail_text_stride : nullptr, fail_text_stride);
        if (r.failure && out[i].fail_code == AMP_FAIL_PROFILE_MISS) {
          // ProfileMissError carries the key (types.hpp:174-178)
          const std::string& s = *r.failure;
          const auto a = s.find("layer=");
          if (a != std::string::npos) out[i].fail_layer = std::atoi(s.c_str() + a + 6);
        }
      }
    };
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Same call chain over an explicit list of candidate indices (a strided
// sample of a large sweep for the CPU baseline).
int ref_sweep_indices(const amp_problem* p, uint64_t P, uint64_t seed, const uint64_t* indices,
                      int64_t n, int32_t threads, amp_record* out, int32_t max_pp) {
  try {
    World w = make_world(p);
    const auto classes = class_list(w);
    std::atomic<int64_t> next{0};
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    auto work = [&] {
      for (int64_t i; (i = next.fetch_add(1)) < n;) {
        const uint64_t idx = indices[i];
        const auto& [pp, dp, tmp, mbs] = classes[idx / P];
        CandidateRecord r = sweep_candidate(w, ParallelismDegrees{pp, dp, tmp}, mbs, idx % P, seed);
        fill_record(r, idx, max_pp, &out[i], nullptr, nullptr, nullptr, nullptr, 0);
      }
    };
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// optimal_assignment(SegmentTimes, ...) (pipeline_dp.cpp:70-149) with the
// EdgeCostFn tabulated as edge_costs[q * L + cut].
int ref_optimal_assignment(const double* layer_times, int32_t L, int32_t stages, int32_t gas,
                           const double* edge_costs, int32_t* cuts, double* cost) {
  try {
    const SegmentTimes times(std::vector<double>(layer_times, layer_times + L));
    const EdgeCostFn edges = [edge_costs, L](int cut, int q) {
      return edge_costs[static_cast<size_t>(q) * L + cut];
    };
    const auto r = optimal_assignment(times, stages, gas, edges);
    for (int q = 0; q <= stages; ++q) cuts[q] = r.assignment.cut_boundaries[q];
    *cost = r.cost;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_brute_force(const double* layer_times, int32_t L, int32_t stages, int32_t gas,
                    const double* edge_costs, int32_t* cuts, double* cost) {
  try {
    const SegmentTimes times(std::vector<double>(layer_times, layer_times + L));
    const EdgeCostFn edges = [edge_costs, L](int cut, int q) {
      return edge_costs[static_cast<size_t>(q) * L + cut];
    };
    const auto r = brute_force_assignment(times, stages, gas, edges);
    for (int q = 0; q <= stages; ++q) cuts[q] = r.assignment.cut_boundaries[q];
    *cost = r.cost;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_tolerance_domain(const double* layer_times, int32_t L, double* out) {
  const SegmentTimes times(std::vector<double>(layer_times, layer_times + L));
  const auto d = tolerance_domain(times);
  std::memcpy(out, d.data(), d.size() * sizeof(double));
  return static_cast<int>(d.size());
}

// estimate() of an explicit strategy (cost_model.cpp:176-212).
int ref_estimate(const amp_problem* p, int32_t pp, int32_t dp, int32_t tmp, int32_t mbs,
                 const int32_t* rank_to_device, const int32_t* cut_boundaries, double* total,
                 double* pipeline, double* dpsync, double* stage, double* edge, char* err,
                 int32_t err_len) {
  try {
    World w = make_world(p);
    ParallelismDegrees deg{pp, dp, tmp};
    Strategy s{deg,
               Placement(deg, std::vector<int>(rank_to_device, rank_to_device + pp * dp * tmp)),
               mbs, LayerAssignment{std::vector<int>(cut_boundaries, cut_boundaries + pp + 1)}};
    const auto b = estimate(s, w.model, w.cluster, w.profile, w.gbs, w.cost);
    *total = b.total;
    *pipeline = b.pipeline_time;
    *dpsync = b.dpsync_time;
    for (size_t q = 0; q < b.per_stage_times.size(); ++q) stage[q] = b.per_stage_times[q];
    for (size_t q = 0; q < b.per_edge_times.size(); ++q) edge[q] = b.per_edge_times[q];
    return 0;
  } catch (const std::exception& e) {
    if (err && err_len > 0) {
      std::strncpy(err, e.what(), err_len - 1);
      err[err_len - 1] = 0;
    }
    return 1;
  }
}

// simulate() of an explicit strategy (simulator.cpp:140-198).
int ref_simulate(const amp_problem* p, int32_t pp, int32_t dp, int32_t tmp, int32_t mbs,
                 const int32_t* rank_to_device, const int32_t* cut_boundaries, double* iteration) {
  try {
    World w = make_world(p);
    ParallelismDegrees deg{pp, dp, tmp};
    Strategy s{deg,
               Placement(deg, std::vector<int>(rank_to_device, rank_to_device + pp * dp * tmp)),
               mbs, LayerAssignment{std::vector<int>(cut_boundaries, cut_boundaries + pp + 1)}};
    SimOptions o;
    o.cost_options = w.cost;
    *iteration = simulate(s, w.model, w.cluster, w.profile, w.gbs, o).iteration_time;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // extern "C"

extern "C" {

// parplan::anneal on the problem (placement.cpp:299-398, the unmodified
// reference chain): initial and best cost, recorded states; 0 on success,
// -1 if the reference threw.
int ref_anneal(const amp_problem* p, int32_t iterations, uint64_t seed, int32_t budget,
               int32_t record_all, double* initial_cost, double* best_cost, int32_t* n_record) {
  try {
    World w = make_world(p);
    AnnealOptions o;
    o.iterations = iterations;
    o.seed = seed;
    o.budget = budget;
    o.record_all = record_all != 0;
    o.cost_options = w.cost;
    const AnnealResult r = anneal(w.model, w.cluster, w.profile, w.gbs, o);
    if (initial_cost) *initial_cost = r.initial_cost;
    if (best_cost) *best_cost = r.best_cost;
    if (n_record) *n_record = (int32_t)r.record.size();
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
