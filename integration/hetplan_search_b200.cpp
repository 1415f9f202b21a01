// hetplan_search_b200.cpp — drop-in hetplan::search over the B200 engine.
//
// Defines the reference's own entry point
//   SearchOutcome hetplan::search(const ModelSpec&, const ClusterSpec&,
//                                 const TrainConfig&, const PlannerConfig&, int jobs)
// (planner.hpp:115-116; reference body planner.cpp:579-685) by flattening the
// specs into the C ABI of include/hetplan_b200.h, running hp_search on the
// GPU and rebuilding SearchOutcome: the winner plan (make_plan,
// planner.cpp:553-575), its full evaluation with trace (planner.cpp:681-684:
// hp_evaluate_plan_full), the candidate counts and the search log
// (hp_search_log). `jobs` (the reference's worker threads) selects how many
// of the box's GPUs search in parallel (hp_search_multi, NCCL between them). Errors keep the
// reference's exception types: ConfigError for spec/planner problems,
// InfeasibleError with the first 200 distinct "candidate -> reason" lines
// (planner.cpp:666-678).
//
// A maintainer links this file in place of planner.cpp's search() (see
// INTEGRATION.md); integration/Makefile does exactly that against the
// unmodified reference sources to run the reference's callers on the GPU.
//
// Environment: HETPLAN_B200_DEVICE (CUDA device of single-GPU searches,
// default 0); HETPLAN_B200_DEVICES="0,1,..." (the GPUs, overriding jobs);
// HETPLAN_B200_LOG=0 skips the search log for callers that never read it.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "hetplan/errors.hpp"
#include "hetplan/evaluate.hpp"
#include "hetplan/planner.hpp"
#include "hetplan_b200.h"

namespace hetplan {
namespace {

struct Flat {
  std::vector<hp_group> groups;
  std::vector<hp_link> links;
  std::vector<int32_t> pps;
  std::vector<int64_t> mbs;
  hp_problem prob{};
};

// First group of that name, like ClusterSpec::find_group (types.cpp:26-31);
// -1 lets hp_search report the reference's validation message.
int group_index(const ClusterSpec& c, const std::string& name) {
  for (std::size_t g = 0; g < c.groups.size(); ++g)
    if (c.groups[g].name == name) return static_cast<int>(g);
  return -1;
}

void flatten(const ModelSpec& m, const ClusterSpec& c, const TrainConfig& t, const PlannerConfig& pc,
             Flat& f) {
  if (c.groups.size() > HP_MAX_GROUPS)
    throw ConfigError("cluster: at most " + std::to_string(HP_MAX_GROUPS) + " device groups supported");
  hp_model& hm = f.prob.model;
  hm.num_layers = m.num_layers;
  hm.num_heads = m.num_heads;
  hm.hidden_size = m.hidden_size;
  hm.seq_length = m.seq_length;
  hm.vocab_size = m.vocab_size;
  hm.bytes_per_element = m.bytes_per_element;
  hm.activation_bytes_per_token_per_hidden = m.activation_bytes_per_token_per_hidden;
  hm.edge_layer_cost_multiplier = m.edge_layer_cost_multiplier;
  for (const DeviceGroup& g : c.groups) {
    hp_group h{};
    h.name = g.name.c_str();  // borrowed: the specs outlive the call
    h.peak_tflops = g.peak_tflops;
    h.memory_bytes = g.memory_bytes;
    h.node_count = g.node_count;
    h.devices_per_node = g.devices_per_node;
    h.compute_efficiency = g.compute_efficiency;
    h.bwd_fwd_ratio = g.bwd_fwd_ratio;
    f.groups.push_back(h);
  }
  for (const Link& l : c.links) {
    hp_link h{};
    h.scope = l.endpoints.kind == ScopeKind::IntraNode             ? HP_INTRA_NODE
              : l.endpoints.kind == ScopeKind::InterNodeHomogeneous ? HP_INTER_NODE
                                                                    : HP_INTER_GROUP;
    h.path = l.path_kind == PathKind::CpuStaged ? HP_CPU_STAGED : HP_GPU_DIRECT;
    h.group_a = group_index(c, l.endpoints.group_a);
    h.group_b = l.endpoints.kind == ScopeKind::InterGroup ? group_index(c, l.endpoints.group_b) : -1;
    h.group_a_name = l.endpoints.group_a.c_str();
    h.group_b_name = l.endpoints.group_b.c_str();
    h.bandwidth_bits_per_s = l.bandwidth_bits_per_s;
    h.latency_s = l.latency_s;
    h.efficiency = l.efficiency;
    h.staging_copy_bytes_per_s = l.staging_copy_bytes_per_s;
    f.links.push_back(h);
  }
  f.prob.cluster.n_groups = static_cast<int32_t>(f.groups.size());
  f.prob.cluster.n_links = static_cast<int32_t>(f.links.size());
  f.prob.cluster.groups = f.groups.data();
  f.prob.cluster.links = f.links.data();
  f.prob.train.global_batch_size = t.global_batch_size;
  f.prob.train.micro_batch_size = t.micro_batch_size;
  f.prob.train.optimizer_state_multiplier = t.optimizer_state_multiplier;
  for (int pp : pc.pipeline_degrees) f.pps.push_back(pp);
  for (long long b : pc.micro_batch_candidates) f.mbs.push_back(b);
  hp_planner& hp = f.prob.planner;
  hp.n_pipeline_degrees = static_cast<int32_t>(f.pps.size());
  hp.n_micro_batch_candidates = static_cast<int32_t>(f.mbs.size());
  hp.pipeline_degrees = f.pps.data();
  hp.micro_batch_candidates = f.mbs.data();
  hp.memory_headroom = pc.memory_headroom;
  hp.exhaustive_split_limit = pc.exhaustive_split_limit;
  hp.stage_order_beam_width = pc.stage_order_beam_width;
  hp.uniform_split_only = pc.uniform_split_only;
  hp.allow_group_interleaving = pc.allow_group_interleaving;
  hp.time_bound_pruning = pc.time_bound_pruning;
  hp.schedule = pc.schedule == Schedule::GPipe ? HP_GPIPE : HP_1F1B;
}

ParallelPlan unflatten(const hp_plan& p, const ClusterSpec& c) {
  ParallelPlan plan;
  plan.schedule = p.schedule == HP_GPIPE ? Schedule::GPipe : Schedule::OneFOneB;
  plan.micro_batches_per_dp_replica = p.micro_batches_per_dp_replica;
  plan.micro_batch_size = p.micro_batch_size;
  for (int i = 0; i < p.n_stages; ++i) {
    const hp_stage& s = p.stages[i];
    StageAssignment a;
    a.layer_range = {s.layer_begin, s.layer_end};
    a.group = c.groups[s.group].name;
    a.nodes_used = s.nodes_used;
    a.tp_degree = s.tp_degree;
    a.dp_degree = s.dp_degree;
    plan.stages.push_back(std::move(a));
  }
  return plan;
}

// Engine contexts per process (the reference's search is re-entrant per
// call; calls here are serialised): one single-GPU context, and one
// multi-GPU group per device list.
std::mutex g_mu;
hp_ctx* g_ctx = nullptr;
hp_multi* g_multi = nullptr;
std::vector<int32_t> g_multi_devs;

hp_ctx* context() {
  if (!g_ctx) {
    const char* dev = std::getenv("HETPLAN_B200_DEVICE");
    if (hp_create(&g_ctx, dev ? std::atoi(dev) : 0) != HP_OK)
      throw std::runtime_error("hetplan_b200: no usable CUDA device");
  }
  return g_ctx;
}

[[noreturn]] void raise_msg(hp_status st, const std::string& msg) {
  if (st == HP_BAD_CONFIG) throw ConfigError(msg);
  if (st == HP_INFEASIBLE) throw InfeasibleError(msg);
  throw std::runtime_error("hetplan_b200: " + msg);
}

[[noreturn]] void raise(hp_ctx* ctx, hp_status st) { raise_msg(st, hp_last_error(ctx)); }

// GPUs for a search: HETPLAN_B200_DEVICES="0,1,..." if set, else `jobs`
// ("parallel search workers", tools/main.cpp:43) capped at the visible GPUs.
std::vector<int32_t> devices_for(int jobs) {
  std::vector<int32_t> d;
  if (const char* e = std::getenv("HETPLAN_B200_DEVICES")) {
    std::string s(e);
    size_t pos = 0;
    while (pos < s.size()) {
      size_t q = s.find(',', pos);
      if (q == std::string::npos) q = s.size();
      if (q > pos) d.push_back(std::atoi(s.substr(pos, q - pos).c_str()));
      pos = q + 1;
    }
    return d;
  }
  const int n = std::min(std::max(jobs, 1), std::max(hp_device_count(), 1));
  for (int i = 0; i < n; ++i) d.push_back(i);
  return d;
}

hp_multi* multi(const std::vector<int32_t>& devs) {
  if (!g_multi || g_multi_devs != devs) {
    if (g_multi) hp_multi_destroy(g_multi);
    g_multi = nullptr;
    hp_multi* m = nullptr;
    hp_status st = hp_multi_create(&m, devs.data(), static_cast<int32_t>(devs.size()));
    if (st != HP_OK) {
      std::string msg = hp_multi_last_error(m);
      hp_multi_destroy(m);
      raise_msg(st, msg);
    }
    g_multi = m;
    g_multi_devs = devs;
  }
  return g_multi;
}

// The winner's PlanEvaluation (planner.cpp:681-684) from
// hp_evaluate_plan_full: GPU simulation with every node time, trace and
// per-stage vectors (evaluate.hpp:38-44, sim.hpp:34-53).
PlanEvaluation evaluate_winner(hp_ctx* ctx, const hp_problem& prob, const hp_plan& plan) {
  const int P = plan.n_stages;
  const uint64_t cap = 4ULL * P * plan.micro_batches_per_dp_replica - 2ULL * plan.micro_batches_per_dp_replica;
  hp_plan_eval ev{};
  std::vector<hp_stage_eval> st(P);
  std::vector<hp_trace_event> tr(cap);
  hp_status s = hp_evaluate_plan_full(ctx, &prob, &plan, &ev, st.data(), tr.data(), cap);
  if (s != HP_OK) raise(ctx, s);
  PlanEvaluation out;
  out.pipeline_time_s = ev.pipeline_time_s;
  out.micro_batches = ev.micro_batches;
  out.total_devices = ev.total_devices;
  out.costs.times.resize(P);
  out.costs.dp_sync_s.resize(P);
  SimResult& sim = out.sim;
  sim.iteration_time_s = ev.iteration_time_s;
  sim.aggregate_bubble_ratio = ev.aggregate_bubble_ratio;
  for (int i = 0; i < P; ++i) {
    out.costs.times[i] = {st[i].fwd_s, st[i].bwd_s, st[i].send_fwd_s, st[i].send_bwd_s};
    out.costs.dp_sync_s[i] = st[i].dp_sync_s;
    sim.per_stage_busy_s.push_back(st[i].busy_s);
    sim.per_stage_compute_end_s.push_back(st[i].compute_end_s);
    sim.per_stage_bubble_ratio.push_back(st[i].bubble_ratio);
    sim.peak_in_flight.push_back(st[i].peak_in_flight);
    sim.peak_memory_bytes.push_back(st[i].peak_memory_bytes);
  }
  sim.trace.reserve(ev.n_trace);
  for (uint64_t k = 0; k < ev.n_trace; ++k)
    sim.trace.push_back({tr[k].stage, static_cast<EventKind>(tr[k].kind), tr[k].microbatch, tr[k].start_s,
                         tr[k].end_s});
  return out;
}

}  // namespace

SearchOutcome search(const ModelSpec& model, const ClusterSpec& cluster, const TrainConfig& cfg,
                     const PlannerConfig& pcfg, int jobs) {
  Flat f;
  flatten(model, cluster, cfg, pcfg, f);
  const char* lg = std::getenv("HETPLAN_B200_LOG");
  const bool want_log = !(lg && std::strcmp(lg, "0") == 0);

  std::lock_guard<std::mutex> lock(g_mu);
  hp_ctx* ctx = context();
  // jobs -> GPUs of this box (planner.cpp:612-664's thread pool); the result
  // is the same for any count, like the reference's for any jobs
  const std::vector<int32_t> devs = devices_for(jobs);
  hp_multi* mg = devs.size() > 1 ? multi(devs) : nullptr;
  auto run = [&](int32_t flags, hp_result& res) {
    if (mg) {
      hp_status st = hp_search_multi(mg, &f.prob, flags, &res, nullptr);
      if (st != HP_OK) raise_msg(st, hp_multi_last_error(mg));
      return;
    }
    hp_search_opts opts{0, 1, 0, flags, 0.0};
    hp_status st = hp_search(ctx, &f.prob, &opts, &res);
    if (st != HP_OK) raise(ctx, st);
  };
  hp_result res;
  run(want_log ? HP_FLAG_LOG : 0, res);

  SearchOutcome out;
  out.candidates_simulated = res.candidates_simulated;
  out.candidates_pruned = res.candidates_pruned;
  if (want_log || !res.has_best) {
    if (!want_log) run(HP_FLAG_LOG, res);  // infeasible: the reasons come from the log
    uint64_t n = 0, tb = 0;
    hp_status st;
    auto get_log = [&](hp_log_entry* e, uint64_t ec, char* t, uint64_t tc) {
      st = mg ? hp_multi_search_log(mg, e, ec, t, tc, &n, &tb) : hp_search_log(ctx, e, ec, t, tc, &n, &tb);
      if (st != HP_OK) raise_msg(st, mg ? hp_multi_last_error(mg) : hp_last_error(ctx));
    };
    get_log(nullptr, 0, nullptr, 0);
    std::vector<hp_log_entry> ents(n);
    std::vector<char> text(tb);
    get_log(ents.data(), n, text.data(), tb);
    out.log.reserve(n);
    for (const hp_log_entry& e : ents)
      out.log.push_back({std::string(text.data() + e.candidate), e.time_s, std::string(text.data() + e.reason)});
  }
  if (!res.has_best) {
    std::vector<std::string> reasons;
    std::set<std::string> seen;
    for (const SearchLogEntry& e : out.log) {
      if (e.prune_reason.empty()) continue;
      std::string line = e.candidate + " -> " + e.prune_reason;
      if (seen.insert(line).second && reasons.size() < 200) reasons.push_back(line);
    }
    if (res.tasks == 0)
      reasons.push_back(
          "no usable pipeline degree: candidates must lie in [1, num_layers] and fit the "
          "cluster's node counts");
    throw InfeasibleError("no feasible plan found", std::move(reasons));
  }
  if (!want_log) out.log.clear();
  out.plan = unflatten(res.best_plan, cluster);
  // the winner's full evaluation with trace, on the GPU
  out.eval = evaluate_winner(ctx, f.prob, res.best_plan);
  return out;
}

}  // namespace hetplan
