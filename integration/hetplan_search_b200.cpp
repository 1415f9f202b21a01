// hetplan_search_b200.cpp — drop-in hetplan::search over the B200 engine.
//
// Defines the reference's own entry point
//   SearchOutcome hetplan::search(const ModelSpec&, const ClusterSpec&,
//                                 const TrainConfig&, const PlannerConfig&, int jobs)
// (planner.hpp:115-116; reference body planner.cpp:579-685) by flattening the
// specs into the C ABI of include/hetplan_b200.h, running hp_search on the
// GPU and rebuilding SearchOutcome: the winner plan (make_plan,
// planner.cpp:553-575), its full evaluation with trace (planner.cpp:681-684,
// the reference's own evaluate_plan_unchecked — cold, once per search), the
// candidate counts and the search log (hp_search_log). Errors keep the
// reference's exception types: ConfigError for spec/planner problems,
// InfeasibleError with the first 200 distinct "candidate -> reason" lines
// (planner.cpp:666-678).
//
// A maintainer links this file in place of planner.cpp's search() (see
// INTEGRATION.md); integration/Makefile does exactly that against the
// unmodified reference sources to run the reference's callers on the GPU.
//
// Environment: HETPLAN_B200_DEVICE (CUDA device, default 0);
// HETPLAN_B200_LOG=0 skips the search log for callers that never read it.
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
    if (g.name.size() >= HP_NAME_LEN)
      throw ConfigError("cluster: group name '" + g.name + "' longer than " +
                        std::to_string(HP_NAME_LEN - 1) + " bytes");
    std::memcpy(h.name, g.name.data(), g.name.size());
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

// One engine context per process (the reference's search is re-entrant per
// call; calls here are serialised on the context).
std::mutex g_mu;
hp_ctx* g_ctx = nullptr;

hp_ctx* context() {
  if (!g_ctx) {
    const char* dev = std::getenv("HETPLAN_B200_DEVICE");
    if (hp_create(&g_ctx, dev ? std::atoi(dev) : 0) != HP_OK)
      throw std::runtime_error("hetplan_b200: no usable CUDA device");
  }
  return g_ctx;
}

[[noreturn]] void raise(hp_ctx* ctx, hp_status st) {
  std::string msg = hp_last_error(ctx);
  if (st == HP_BAD_CONFIG) throw ConfigError(msg);
  if (st == HP_INFEASIBLE) throw InfeasibleError(msg);
  throw std::runtime_error("hetplan_b200: " + msg);
}

}  // namespace

SearchOutcome search(const ModelSpec& model, const ClusterSpec& cluster, const TrainConfig& cfg,
                     const PlannerConfig& pcfg, int jobs) {
  (void)jobs;  // the GPU replaces the thread pool; results never depended on it
  Flat f;
  flatten(model, cluster, cfg, pcfg, f);
  const char* lg = std::getenv("HETPLAN_B200_LOG");
  const bool want_log = !(lg && std::strcmp(lg, "0") == 0);

  std::lock_guard<std::mutex> lock(g_mu);
  hp_ctx* ctx = context();
  hp_search_opts opts{0, 1, 0, want_log ? HP_FLAG_LOG : 0, 0.0};
  hp_result res;
  hp_status st = hp_search(ctx, &f.prob, &opts, &res);
  if (st != HP_OK) raise(ctx, st);

  SearchOutcome out;
  out.candidates_simulated = res.candidates_simulated;
  out.candidates_pruned = res.candidates_pruned;
  if (want_log || !res.has_best) {
    if (!want_log) {  // infeasible: the reasons come from the log
      opts.flags = HP_FLAG_LOG;
      st = hp_search(ctx, &f.prob, &opts, &res);
      if (st != HP_OK) raise(ctx, st);
    }
    uint64_t n = 0, tb = 0;
    if ((st = hp_search_log(ctx, nullptr, 0, nullptr, 0, &n, &tb)) != HP_OK) raise(ctx, st);
    std::vector<hp_log_entry> ents(n);
    std::vector<char> text(tb);
    if ((st = hp_search_log(ctx, ents.data(), n, text.data(), tb, &n, &tb)) != HP_OK) raise(ctx, st);
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
  // The inner loop simulates without traces; give the winner a full one.
  out.eval = evaluate_plan_unchecked(out.plan, model, cluster, cfg);
  return out;
}

}  // namespace hetplan
