// amp_simulate.cpp — host-side pipeline simulator used by plan() to validate
// its top `budget` candidates (reference optimizer.cpp:235-249).
//
// Restates simulate() (reference proj/src/simulator.cpp:140-198) and its
// event loop run_replica (75-136): per replica, gas micro-batches stream
// through the stages; a stage starts a micro-batch once its input arrived
// and it is idle; the outgoing transfer overlaps the sender's next
// micro-batch; transfers on one boundary are FIFO; ties resolve in
// (time, stage, micro-batch, transfer-first) order.  This is not on the
// batched hot path (it runs on <= budget strategies); the same arithmetic
// order as the reference is kept so best_index matches exactly.
#include <algorithm>
#include <cmath>
#include <deque>
#include <map>
#include <queue>
#include <tuple>
#include <vector>

#include "../../include/amp_search.h"

namespace {

struct Pending {
  double time;
  int stage;
  int microbatch;
  bool is_transfer;
};

struct PendingOrder {  // simulator.cpp:50-63
  bool operator()(const Pending& a, const Pending& b) const {
    if (a.time != b.time) return a.time > b.time;
    if (a.stage != b.stage) return a.stage > b.stage;
    if (a.microbatch != b.microbatch) return a.microbatch > b.microbatch;
    return a.is_transfer < b.is_transfer;
  }
};

struct StageState {
  bool busy = false;
  int next_microbatch = 0;
  std::vector<char> input_ready;
  std::deque<int> send_queue;
  bool link_busy = false;
};

double run_replica(const std::vector<double>& stage_times, const std::vector<double>& edge_times,
                   int gas) {
  const int stages = static_cast<int>(stage_times.size());
  std::vector<StageState> state(stages);
  for (int j = 0; j < stages; ++j) state[j].input_ready.assign(gas, j == 0 ? 1 : 0);
  std::priority_queue<Pending, std::vector<Pending>, PendingOrder> queue;
  auto try_start_compute = [&](int stage, double now) {
    StageState& st = state[stage];
    if (st.busy || st.next_microbatch >= gas || !st.input_ready[st.next_microbatch]) return;
    st.busy = true;
    queue.push({now + stage_times[stage], stage, st.next_microbatch, false});
  };
  auto try_start_transfer = [&](int stage, double now) {
    StageState& st = state[stage];
    if (st.link_busy || st.send_queue.empty()) return;
    st.link_busy = true;
    const int u = st.send_queue.front();
    st.send_queue.pop_front();
    queue.push({now + edge_times[stage], stage, u, true});
  };
  double finish = 0.0;
  try_start_compute(0, 0.0);
  while (!queue.empty()) {
    const Pending ev = queue.top();
    queue.pop();
    if (ev.is_transfer) {
      state[ev.stage].link_busy = false;
      state[ev.stage + 1].input_ready[ev.microbatch] = 1;
      try_start_transfer(ev.stage, ev.time);
      try_start_compute(ev.stage + 1, ev.time);
    } else {
      StageState& st = state[ev.stage];
      st.busy = false;
      st.next_microbatch = ev.microbatch + 1;
      if (ev.stage + 1 < stages) {
        st.send_queue.push_back(ev.microbatch);
        try_start_transfer(ev.stage, ev.time);
      } else if (ev.microbatch == gas - 1) {
        finish = ev.time;
      }
      try_start_compute(ev.stage, ev.time);
    }
  }
  return finish;
}

// LayerTimeResolver::layer_time (cost_model.cpp:74-86); false on miss.
bool layer_time(const amp_problem* p, const std::map<std::tuple<int, int, int>, double>& prof,
                int layer, int tmp, int mbs, double* out) {
  auto it = prof.find({layer, tmp, mbs});
  if (it != prof.end()) {
    *out = it->second;
    return true;
  }
  if (!p->fallback_enabled || !p->flops_present || !p->flops_present[layer]) return false;
  const int L = p->n_layers;
  const double vol = L <= 1 ? 0.0
                            : (layer < L - 1 ? p->activation_volumes[layer]
                                             : p->activation_volumes[layer - 1]);
  const double message = vol * mbs;
  const double compute =
      mbs * p->flops_per_sample[layer] / (tmp * p->fallback_device_flops);
  double ar = 0.0;
  if (tmp != 1) {
    if (!(p->fallback_tmp_bandwidth > 0)) return false;
    ar = 2.0 * (tmp - 1) * message / (tmp * p->fallback_tmp_bandwidth);
  }
  *out = compute + ar;
  return true;
}

}  // namespace

extern "C" int amp_simulate(const amp_problem* p, int32_t pp, int32_t dp, int32_t tmp,
                            int32_t mbs, const int32_t* rank_to_device,
                            const int32_t* cut_boundaries, double* iteration_time) {
  if (!p || !rank_to_device || !cut_boundaries || !iteration_time) return AMP_E_INVALID;
  const int L = p->n_layers, D = p->n_devices;
  if (pp < 1 || dp < 1 || tmp < 1 || pp * dp * tmp != D || mbs < 1) return AMP_E_INVALID;
  if (p->gbs % dp != 0 || (p->gbs / dp) % mbs != 0) return AMP_E_INVALID;
  if (cut_boundaries[0] != 0 || cut_boundaries[pp] != L) return AMP_E_INVALID;
  for (int j = 0; j < pp; ++j)
    if (cut_boundaries[j] >= cut_boundaries[j + 1]) return AMP_E_INVALID;
  std::map<std::tuple<int, int, int>, double> prof;
  for (int64_t e = 0; e < p->n_profile_entries; ++e)
    prof[{p->profile_layer[e], p->profile_tmp[e], p->profile_mbs[e]}] = p->profile_seconds[e];
  const int gas = p->gbs / (dp * mbs);
  auto dev = [&](int q, int r, int s) { return rank_to_device[((size_t)q * dp + r) * tmp + s]; };
  auto link = [&](int a, int b) {
    return a == b ? INFINITY : p->bandwidth[(size_t)a * D + b];
  };
  std::vector<double> stage_times(pp);
  for (int j = 0; j < pp; ++j) {  // stage_time (cost_model.cpp:88-98)
    double sum = 0.0;
    for (int l = cut_boundaries[j]; l < cut_boundaries[j + 1]; ++l) {
      double t;
      if (!layer_time(p, prof, l, tmp, mbs, &t)) return AMP_E_INVALID;
      sum += t;
    }
    stage_times[j] = sum;
  }
  double makespan = 0.0;
  std::vector<double> edges(pp > 1 ? pp - 1 : 0);
  for (int r = 0; r < dp; ++r) {  // replica_edge_times (cost_model.cpp:145-162)
    for (int q = 0; q + 1 < pp; ++q) {
      const int cut = cut_boundaries[q + 1];
      const double volume = p->activation_volumes[cut - 1] * mbs;
      double b = INFINITY;
      for (int s = 0; s < tmp; ++s) b = std::min(b, link(dev(q, r, s), dev(q + 1, r, s)));
      if (!(b > 0)) return AMP_E_INVALID;
      edges[q] = volume / b;
    }
    makespan = std::max(makespan, run_replica(stage_times, edges, gas));
  }
  double worst = 0.0;  // dpsync_time (cost_model.cpp:122-143)
  if (dp != 1) {
    for (int j = 0; j < pp; ++j) {
      double sp = 0.0;
      for (int l = cut_boundaries[j]; l < cut_boundaries[j + 1]; ++l) sp += p->param_count[l];
      const double message = sp * p->bytes_per_param / tmp;
      for (int s = 0; s < tmp; ++s) {
        double b = INFINITY;
        for (int r1 = 0; r1 < dp; ++r1)
          for (int r2 = r1 + 1; r2 < dp; ++r2) b = std::min(b, link(dev(j, r1, s), dev(j, r2, s)));
        if (!(b > 0)) return AMP_E_INVALID;
        worst = std::max(worst, 2.0 * (dp - 1) * message / (dp * b));
      }
    }
  }
  *iteration_time = makespan + worst;
  return AMP_OK;
}
