// hp_eval.cpp — winner post-processing (planner.cpp:681-684): the full
// PlanEvaluation of evaluate_plan_unchecked(record_trace) (evaluate.cpp:
// 78-107) from the node times the GPU simulated (k_plan_trace). What is left
// for the host is bookkeeping in the reference's order: busy sums in each
// stage's op order (sim.cpp:114), the trace sort (sim.cpp:162-167), retained
// activations (sim.cpp:172-189), the DP-sync tail and bubble ratios
// (evaluate.cpp:88-99, sim.cpp:197-209) and peak memory (evaluate.cpp:101-105).
#include <algorithm>
#include <tuple>
#include <utility>
#include <vector>

#include "hp_device.hpp"
#include "hp_eval.hpp"

namespace hpe {

hph::Status evaluate_plan_full(hpd::Arena& a, const hph::Problem& p, const hp_plan& pl, hp_plan_eval* ev,
                               hp_stage_eval* out, hp_trace_event* trace, uint64_t trace_cap) {
  const int P = pl.n_stages;
  const long long M = pl.micro_batches_per_dp_replica;
  const uint64_t n_trace = 4ULL * P * M - 2ULL * M;
  if (trace && trace_cap < n_trace) return hph::Status{HP_BAD_CONFIG, "trace buffer too small"};
  hpd::PlanNodes nd;
  hph::Status s = hpd::plan_node_times(a, p, pl, nd);
  if (!s.ok()) return s;
  const size_t PM = (size_t)P * (size_t)M;
  const double* fs = nd.nodes.data();
  const double* fe = fs + PM;
  const double* bs = fs + 2 * PM;
  const double* be = fs + 3 * PM;
  const double* sfs = fs + 4 * PM;
  const double* sfe = fs + 5 * PM;
  const double* sbs = fs + 6 * PM;
  const double* sbe = fs + 7 * PM;
  const bool gpipe = pl.schedule == HP_GPIPE;

  // pipeline time: max over every op and send end (sim.cpp:118,133,143); each
  // stage's and channel's ends are non-decreasing, so their finals suffice
  double pipeline = 0.0;
  for (int i = 0; i < P; ++i)
    for (int k = 0; k < 3; ++k) pipeline = std::max(pipeline, nd.fin[3 * i + k]);

  std::vector<double> busy(P, 0.0);
  for (int i = 0; i < P; ++i) {
    const double f = nd.dur[5 * i], b = nd.dur[5 * i + 1];
    // stage_ops order (sim.cpp:43-59): the busy sum adds in execution order
    double acc = 0.0;
    if (gpipe) {
      for (long long m = 0; m < M; ++m) acc += f;
      for (long long m = 0; m < M; ++m) acc += b;
    } else {
      const long long w = std::min<long long>(P - i, M);
      for (long long m = 0; m < w; ++m) acc += f;
      long long next = w;
      for (long long m = 0; m < M; ++m) {
        acc += b;
        if (next < M) {
          acc += f;
          ++next;
        }
      }
    }
    busy[i] = acc;
  }

  // retained activations (sim.cpp:172-189): +1 at forward start (end - fwd),
  // -1 at backward end; the release first at equal instants
  std::vector<int> peak(P, 0);
  std::vector<std::pair<double, int>> deltas;
  for (int i = 0; i < P; ++i) {
    deltas.clear();
    deltas.reserve(2 * M);
    const double f = nd.dur[5 * i];
    for (long long m = 0; m < M; ++m) {
      deltas.emplace_back(fe[i * M + m] - f, +1);
      deltas.emplace_back(be[i * M + m], -1);
    }
    std::sort(deltas.begin(), deltas.end());
    int held = 0, pk = 0;
    for (const auto& x : deltas) {
      held += x.second;
      pk = std::max(pk, held);
    }
    peak[i] = pk;
  }

  // DP-sync tail (evaluate.cpp:88-97)
  double iteration = 0.0;
  for (int i = 0; i < P; ++i) {
    busy[i] += nd.dur[5 * i + 4];
    iteration = std::max(iteration, nd.fin[3 * i] + nd.dur[5 * i + 4]);
  }
  iteration = std::max(pipeline, iteration);
  // bubble_ratio (sim.cpp:197-209)
  double agg = 0.0;
  std::vector<double> bub(P, 0.0);
  if (iteration > 0.0) {
    double busy_sum = 0.0;
    for (int i = 0; i < P; ++i) {
      bub[i] = 1.0 - busy[i] / iteration;
      busy_sum += busy[i];
    }
    agg = 1.0 - busy_sum / (static_cast<double>(P) * iteration);
  }

  hpc::Consts c;
  hph::fill_consts(p, c);
  const double B = static_cast<double>(pl.micro_batch_size > 0 ? pl.micro_batch_size : p.train.micro_batch_size);
  long long devices = 0;
  for (int i = 0; i < P; ++i) {
    const hp_stage& st = pl.stages[i];
    hp_stage_eval& o = out[i];
    o.fwd_s = nd.dur[5 * i];
    o.bwd_s = nd.dur[5 * i + 1];
    o.send_fwd_s = nd.dur[5 * i + 2];
    o.send_bwd_s = nd.dur[5 * i + 3];
    o.dp_sync_s = nd.dur[5 * i + 4];
    o.busy_s = busy[i];
    o.compute_end_s = nd.fin[3 * i];
    o.bubble_ratio = bub[i];
    // stage_memory(stage, ..., peak_in_flight) (cost_model.cpp:75-86)
    o.peak_memory_bytes = hpc::stage_memory(c, st.layer_end - st.layer_begin, st.tp_degree, B, peak[i]);
    o.peak_in_flight = peak[i];
    o._pad = 0;
    devices += static_cast<long long>(st.dp_degree) * st.tp_degree;
  }
  ev->iteration_time_s = iteration;
  ev->pipeline_time_s = pipeline;
  ev->aggregate_bubble_ratio = agg;
  ev->micro_batches = M;
  ev->total_devices = devices;
  ev->n_stages = P;
  ev->_pad = 0;
  ev->n_trace = n_trace;

  if (trace) {
    // sim.cpp:97-98,121,133,143 events; sorted (start, stage, kind, mb)
    uint64_t k = 0;
    for (int i = 0; i < P; ++i)
      for (long long m = 0; m < M; ++m) {
        const size_t x = (size_t)i * M + m;
        trace[k++] = hp_trace_event{i, 0, (int32_t)m, 0, fs[x], fe[x]};
        trace[k++] = hp_trace_event{i, 1, (int32_t)m, 0, bs[x], be[x]};
        if (i + 1 < P) trace[k++] = hp_trace_event{i, 2, (int32_t)m, 0, sfs[x], sfe[x]};
        if (i > 0) trace[k++] = hp_trace_event{i, 3, (int32_t)m, 0, sbs[x], sbe[x]};
      }
    std::sort(trace, trace + k, [](const hp_trace_event& x, const hp_trace_event& y) {
      return std::make_tuple(x.start_s, x.stage, x.kind, x.microbatch) <
             std::make_tuple(y.start_s, y.stage, y.kind, y.microbatch);
    });
  }
  return hph::Status{};
}

}  // namespace hpe
