// gen_golden.cpp — TEST INFRASTRUCTURE ONLY.
//
// Regenerates tests/golden/dp_*.json by running the reference itself
// (compiled from /root/reference/proj/src by oracle/Makefile target
// _ref/gen_golden).  The random instances are drawn exactly like the
// reference's own tests — std::mt19937_64 + std::uniform_real_distribution
// of libstdc++ — so the fixtures pin:
//   dp_kat.json        test_pipeline_dp.cpp:110-144, 231-259 known answers
//   dp_seed31.json     test_pipeline_dp.cpp:158-185 (400 instances vs brute force)
//   dp_seed37.json     test_pipeline_dp.cpp:187-210 (gas = 1)
//   dp_seed101.json    acceptance_main.cpp:79-121 (1000 instances)
//   dp_seed113.json    acceptance_main.cpp:399-424 (L = 16 / 32, k = 4)
// Floats are written as C99 hex literals ("%a") so they round-trip exactly.
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "parplan/pipeline_dp.hpp"

using namespace parplan;

namespace {

std::string hex(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "\"%a\"", v);
  return buf;
}

struct Inst {
  std::string name;
  std::vector<double> times;
  int k, gas;
  std::vector<double> edges;  // [(k-1) * L], edges[q*L + cut]
};

void emit(FILE* f, const std::vector<Inst>& v, bool brute) {
  std::fprintf(f, "{\"instances\": [\n");
  for (size_t n = 0; n < v.size(); ++n) {
    const Inst& in = v[n];
    const int L = static_cast<int>(in.times.size());
    const SegmentTimes times(in.times);
    const EdgeCostFn edges = [&](int cut, int q) { return in.edges[static_cast<size_t>(q) * L + cut]; };
    const auto r = optimal_assignment(times, in.k, in.gas, edges);
    std::fprintf(f, "{\"name\": \"%s\", \"L\": %d, \"k\": %d, \"gas\": %d, \"times\": [", in.name.c_str(),
                 L, in.k, in.gas);
    for (int i = 0; i < L; ++i) std::fprintf(f, "%s%s", i ? ", " : "", hex(in.times[i]).c_str());
    std::fprintf(f, "], \"edges\": [");
    for (size_t i = 0; i < in.edges.size(); ++i)
      std::fprintf(f, "%s%s", i ? ", " : "", hex(in.edges[i]).c_str());
    std::fprintf(f, "], \"cuts\": [");
    for (size_t i = 0; i < r.assignment.cut_boundaries.size(); ++i)
      std::fprintf(f, "%s%d", i ? ", " : "", r.assignment.cut_boundaries[i]);
    std::fprintf(f, "], \"cost\": %s, \"domain_size\": %zu", hex(r.cost).c_str(),
                 tolerance_domain(times).size());
    if (brute && L <= 14) {
      const auto b = brute_force_assignment(times, in.k, in.gas, edges);
      std::fprintf(f, ", \"brute_cost\": %s", hex(b.cost).c_str());
    }
    std::fprintf(f, "}%s\n", n + 1 < v.size() ? "," : "");
  }
  std::fprintf(f, "]}\n");
}

Inst make(const std::string& name, std::vector<double> t, int k, int gas,
          const std::function<double(int, int)>& e) {
  Inst in{name, t, k, gas, {}};
  const int L = static_cast<int>(t.size());
  in.edges.assign(static_cast<size_t>(std::max(0, k - 1)) * L, 0.0);
  for (int q = 0; q + 1 < k; ++q)
    for (int cut = 1; cut < L; ++cut) in.edges[static_cast<size_t>(q) * L + cut] = e(cut, q);
  return in;
}

void write(const std::string& dir, const std::string& file, const std::vector<Inst>& v, bool brute) {
  const std::string path = dir + "/" + file;
  FILE* f = std::fopen(path.c_str(), "w");
  emit(f, v, brute);
  std::fclose(f);
  std::printf("wrote %s (%zu instances)\n", path.c_str(), v.size());
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "tests/golden";
  {  // known answers
    std::vector<Inst> v;
    v.push_back(make("uniform4_k2", std::vector<double>(4, 1.0), 2, 2, [](int, int) { return 1.0; }));
    for (int gas : {1, 2, 8})
      v.push_back(make("single_stage_gas" + std::to_string(gas), {0.5, 1.5, 1.0}, 1, gas,
                       [](int, int) { return 0.0; }));
    v.push_back(make("heavy_head", {4, 1, 1, 1, 1}, 2, 8, [](int, int) { return 0.0; }));
    v.push_back(make("two_layers", {1.0, 2.0}, 2, 4, [](int, int) { return 0.5; }));
    v.push_back(make("stage_pair_edges", {1.0, 1.0, 1.0, 1.0}, 2, 1,
                     [](int cut, int) { return cut == 2 ? 100.0 : 0.0; }));
    v.push_back(make("ties_uniform30_k4", std::vector<double>(30, 0.25), 4, 3,
                     [](int, int q) { return 0.01 * (q + 1); }));
    write(dir, "dp_kat.json", v, true);
  }
  {  // test_pipeline_dp.cpp:158-185
    std::mt19937_64 gen(31);
    std::uniform_real_distribution<double> pos(0.01, 10.0);
    const int gas_choices[] = {1, 2, 8};
    std::vector<Inst> v;
    for (int trial = 0; trial < 400; ++trial) {
      const int L = 2 + static_cast<int>(gen() % 9);
      const int k = 1 + static_cast<int>(gen() % std::min(4, L));
      const int gas = gas_choices[gen() % 3];
      std::vector<double> t(L);
      for (auto& x : t) x = pos(gen);
      std::vector<double> e(L, 0.0);
      for (auto& x : e) x = pos(gen) * 0.1;
      v.push_back(make("seed31_" + std::to_string(trial), t, k, gas, [&](int cut, int) { return e[cut]; }));
    }
    write(dir, "dp_seed31.json", v, true);
  }
  {  // test_pipeline_dp.cpp:187-210
    std::mt19937_64 gen(37);
    std::uniform_real_distribution<double> pos(0.01, 10.0);
    std::vector<Inst> v;
    for (int trial = 0; trial < 100; ++trial) {
      const int L = 3 + static_cast<int>(gen() % 6);
      const int k = 2 + static_cast<int>(gen() % 2);
      std::vector<double> t(L);
      for (auto& x : t) x = pos(gen);
      std::vector<double> e(L);
      for (auto& x : e) x = pos(gen);
      v.push_back(make("seed37_" + std::to_string(trial), t, k, 1, [&](int cut, int) { return e[cut]; }));
    }
    write(dir, "dp_seed37.json", v, true);
  }
  {  // acceptance_main.cpp:79-121
    std::mt19937_64 gen(101);
    std::uniform_real_distribution<double> pos(0.01, 10.0);
    const int gas_choices[] = {1, 2, 8};
    std::vector<Inst> v;
    for (int trial = 0; trial < 1000; ++trial) {
      const int L = 2 + static_cast<int>(gen() % 9);
      const int k = 1 + static_cast<int>(gen() % std::min(4, L));
      const int gas = gas_choices[gen() % 3];
      std::vector<double> t(L);
      for (auto& x : t) x = pos(gen);
      std::vector<double> e(L);
      for (auto& x : e) x = pos(gen) * 0.2;
      v.push_back(make("seed101_" + std::to_string(trial), t, k, gas, [&](int cut, int) { return e[cut]; }));
    }
    write(dir, "dp_seed101.json", v, true);
  }
  {  // acceptance_main.cpp:399-424 instances (L = 16 and 32, k = 4, gas = 4)
    std::mt19937_64 gen(113);
    std::uniform_real_distribution<double> pos(0.01, 1.0);
    std::vector<Inst> v;
    for (int L : {16, 32}) {
      std::vector<double> t(L);
      for (auto& x : t) x = pos(gen);
      v.push_back(make("seed113_L" + std::to_string(L), t, 4, 4, [](int, int) { return 0.01; }));
    }
    // larger stage counts on the same shapes (L up to 96, k up to 32)
    std::mt19937_64 g2(127);
    std::uniform_real_distribution<double> p2(0.01, 3.0);
    for (int trial = 0; trial < 24; ++trial) {
      const int L = 16 + static_cast<int>(g2() % 81);
      const int k = 1 + static_cast<int>(g2() % std::min(32, L));
      const int gas = 1 + static_cast<int>(g2() % 16);
      std::vector<double> t(L);
      for (auto& x : t) x = p2(g2);
      std::vector<double> e(static_cast<size_t>(std::max(0, k - 1)) * L);
      for (auto& x : e) x = p2(g2) * 0.05;
      v.push_back(make("large_" + std::to_string(trial), t, k, gas,
                       [&](int cut, int q) { return e[static_cast<size_t>(q) * L + cut]; }));
    }
    write(dir, "dp_large.json", v, false);
  }
  return 0;
}
