// gen_report.cpp — TEST INFRASTRUCTURE ONLY.
//
// Writes the reference's own report.json for a plan() run
// (report.cpp:28-53 write_report, the CLI `plan` path of
// parplan_main.cpp:196-216), so tests/golden/report_*.json pin the drop-in
// CLI's report byte for byte.  Built by oracle/Makefile (_ref/gen_report)
// from the reference sources where they lie, with nlohmann/json 3.11.3 from
// the venv (the reference's vendored copy is absent).
//
//   gen_report <model> <cluster> <profile> <gbs> <budget> <out.json>
//              [fallback_device_flops fallback_tmp_bw] [max_params]
//   GEN_MODE=layer-balance|param-balance: the CLI `baseline` path instead
//   (megatron_baseline, optimizer.cpp:253-279; parplan_main.cpp:285-296)
// Exit codes follow the CLI: 1 error, 3 all candidates failed on a profile
// miss (parplan_main.cpp:73-82).
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>

#include <cstdio>
#include <fstream>

#include "parplan/json_io.hpp"
#include "parplan/optimizer.hpp"
#include "parplan/placement.hpp"
#include "parplan/report.hpp"
#include "parplan/simulator.hpp"

int main(int argc, char** argv) {
  if (argc < 7) {
    std::cerr << "usage: gen_report model cluster profile gbs budget out [flops tmp_bw] [max]\n";
    return 1;
  }
  try {
    const parplan::ModelGraph model = parplan::load_model(argv[1]);
    const parplan::Cluster cluster = parplan::load_cluster(argv[2]);
    const parplan::ProfileTable profile = parplan::load_profile(argv[3]);
    parplan::PlanOptions opts;
    opts.budget = std::atoi(argv[5]);
    opts.workers = 0;
    if (argc >= 9) {
      const double flops = std::atof(argv[7]), bw = std::atof(argv[8]);
      if (flops > 0) {
        opts.cost_options.fallback.enabled = true;
        opts.cost_options.fallback.device_flops = flops;
        if (bw > 0) opts.cost_options.fallback.tmp_bandwidth = bw;
      }
    }
    if (argc >= 10 && std::atof(argv[9]) > 0) opts.max_params_per_device = std::atof(argv[9]);
    if (const char* mode = std::getenv("GEN_MODE"); mode && std::strncmp(mode, "anneal", 6) == 0) {
      // CLI `anneal` (parplan_main.cpp:219-256): GEN_MODE=anneal:<iters>:<seed>[:trace]
      parplan::AnnealOptions ao;
      ao.budget = opts.budget;
      ao.cost_options = opts.cost_options;
      int iters = 200;
      unsigned long long seed = 0;
      char tr[16] = {0};
      std::sscanf(mode, "anneal:%d:%llu:%15s", &iters, &seed, tr);
      ao.iterations = iters;
      ao.seed = seed;
      parplan::AnnealResult result =
          parplan::anneal(model, cluster, profile, std::atoi(argv[4]), ao);
      std::vector<parplan::CandidateRecord> candidates;
      for (size_t i = 0; i < result.top.size(); ++i) {
        parplan::CandidateRecord record;
        record.strategy = result.top[i].strategy;
        record.estimated = result.top[i].estimated;
        record.rank = static_cast<int>(i) + 1;
        parplan::SimOptions sim_options;
        sim_options.cost_options = opts.cost_options;
        record.simulated = parplan::simulate(record.strategy, model, cluster, profile,
                                             std::atoi(argv[4]), sim_options).iteration_time;
        candidates.push_back(std::move(record));
      }
      parplan::write_report(candidates, argv[6]);
      parplan::print_candidate_table(std::cout, candidates);
      if (tr[0]) {
        std::ofstream out(std::string(argv[6]) + ".trace");
        for (const auto& entry : result.record) {
          nlohmann::json line = parplan::strategy_to_json(entry.strategy);
          line["iteration"] = entry.iteration;
          line["accepted"] = entry.accepted;
          line["estimated_total"] = entry.estimated.total;
          out << line.dump() << "\n";
        }
      }
      return 0;
    }
    if (const char* mode = std::getenv("GEN_MODE")) {
      const auto bal = std::strcmp(mode, "param-balance") == 0 ? parplan::BalanceMode::kParamBalance
                                                               : parplan::BalanceMode::kLayerBalance;
      const auto cands = parplan::megatron_baseline(model, cluster, profile, std::atoi(argv[4]), bal,
                                                    opts.cost_options);
      bool ok = false;
      for (const auto& c : cands) ok |= !c.failure;
      if (!ok) {
        const std::string why = cands.empty() ? "no candidates" : *cands.front().failure;
        std::cerr << "error: every candidate failed; first failure: " << why << "\n";
        return why.find("profile miss") != std::string::npos ? 3 : 1;
      }
      parplan::write_report(cands, argv[6]);
      parplan::print_candidate_table(std::cout, cands);
      return 0;
    }
    const parplan::PlanResult r = parplan::plan(model, cluster, profile, std::atoi(argv[4]), opts);
    bool any_ok = false;
    for (const auto& c : r.candidates) any_ok |= !c.failure;
    if (!any_ok) {
      const std::string why = r.candidates.empty() ? "no candidates" : *r.candidates.front().failure;
      std::cerr << "error: every candidate failed; first failure: " << why << "\n";
      return why.find("profile miss") != std::string::npos ? 3 : 1;
    }
    parplan::write_report(r.candidates, argv[6]);
    parplan::print_candidate_table(std::cout, r.candidates);
    if (r.best_index >= 0)
      std::cout << "best by simulation: rank " << r.candidates[r.best_index].rank << "\n";
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
