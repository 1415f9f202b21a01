// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI driver around the UNMODIFIED reference planner (hetplan, compiled
// from /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).
// It parses the reference's own JSON documents with the reference's own
// parsers (json_io.cpp:83-219), calls hetplan::search()
// (planner.cpp:579-685) and reports the outcome as JSON with the iteration
// time's exact bit pattern, so tests can compare the CUDA path bit-exactly.
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs load this library.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "json.hpp"

#include "hetplan/errors.hpp"
#include "hetplan/evaluate.hpp"
#include "hetplan/json_io.hpp"
#include "hetplan/planner.hpp"
#include "hetplan/profile.hpp"

using nlohmann::json;

namespace {

std::string hex_bits(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, sizeof u);
  char buf[19];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(u));
  return buf;
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

json eval_json(const hetplan::PlanEvaluation& e) {
  json stages = json::array();
  for (std::size_t i = 0; i < e.costs.times.size(); ++i) {
    const auto& t = e.costs.times[i];
    stages.push_back(json{{"fwd", hex_bits(t.fwd_s)},
                          {"bwd", hex_bits(t.bwd_s)},
                          {"send_fwd", hex_bits(t.send_fwd_s)},
                          {"send_bwd", hex_bits(t.send_bwd_s)},
                          {"dp_sync", hex_bits(e.costs.dp_sync_s[i])},
                          {"compute_end", hex_bits(e.sim.per_stage_compute_end_s[i])},
                          {"peak_in_flight", e.sim.peak_in_flight[i]},
                          {"peak_memory", hex_bits(e.sim.peak_memory_bytes[i])}});
  }
  return json{{"iteration_time_s", e.sim.iteration_time_s},
              {"iteration_bits", hex_bits(e.sim.iteration_time_s)},
              {"pipeline_bits", hex_bits(e.pipeline_time_s)},
              {"aggregate_bubble_bits", hex_bits(e.sim.aggregate_bubble_ratio)},
              {"stages", stages}};
}

}  // namespace

extern "C" {

// Runs hetplan::search on the four JSON documents. Returns 0 on success,
// 1 ConfigError, 2 InfeasibleError/PlanError, 3 anything else (cli.hpp:25
// exit-code convention). *out receives a malloc'd JSON string either way.
int ref_search_json(const char* model, const char* cluster, const char* train,
                    const char* planner, int jobs, int want_log, char** out) {
  json result;
  int status = 0;
  try {
    hetplan::ModelSpec m = hetplan::model_from_json(json::parse(model));
    hetplan::ClusterSpec c = hetplan::cluster_from_json(json::parse(cluster));
    hetplan::TrainConfig t = hetplan::train_from_json(json::parse(train));
    hetplan::PlannerConfig p = hetplan::planner_from_json(json::parse(planner));
    auto t0 = std::chrono::steady_clock::now();
    hetplan::SearchOutcome o = hetplan::search(m, c, t, p, jobs);
    auto t1 = std::chrono::steady_clock::now();
    result["plan"] = hetplan::to_json(o.plan);
    result["eval"] = eval_json(o.eval);
    result["candidates_simulated"] = o.candidates_simulated;
    result["candidates_pruned"] = o.candidates_pruned;
    result["wall_s"] = std::chrono::duration<double>(t1 - t0).count();
    if (want_log) {
      json log = json::array();
      for (const auto& e : o.log)
        log.push_back(json{{"candidate", e.candidate},
                           {"time_bits", hex_bits(e.time_s)},
                           {"reason", e.prune_reason}});
      result["log"] = std::move(log);
    }
  } catch (const hetplan::ConfigError& e) {
    status = 1;
    result["error"] = e.what();
  } catch (const hetplan::InfeasibleError& e) {
    status = 2;
    result["error"] = e.what();
    result["reasons"] = e.reasons;
  } catch (const hetplan::PlanError& e) {
    status = 2;
    result["error"] = e.what();
    result["reasons"] = e.violations;
  } catch (const std::exception& e) {
    status = 3;
    result["error"] = e.what();
  }
  result["status"] = status;
  *out = dup_string(result.dump());
  return status;
}

// evaluate_plan_unchecked (evaluate.cpp:78-107) on one explicit plan.
int ref_evaluate_json(const char* model, const char* cluster, const char* train,
                      const char* plan, char** out) {
  json result;
  int status = 0;
  try {
    hetplan::ModelSpec m = hetplan::model_from_json(json::parse(model));
    hetplan::ClusterSpec c = hetplan::cluster_from_json(json::parse(cluster));
    hetplan::TrainConfig t = hetplan::train_from_json(json::parse(train));
    hetplan::ParallelPlan p = hetplan::plan_from_json(json::parse(plan));
    hetplan::PlanEvaluation e = hetplan::evaluate_plan_unchecked(p, m, c, t, false);
    result["eval"] = eval_json(e);
  } catch (const std::exception& e) {
    status = 3;
    result["error"] = e.what();
  }
  result["status"] = status;
  *out = dup_string(result.dump());
  return status;
}

// evaluate_plan_unchecked(record_trace = true) on one explicit plan: every
// field of PlanEvaluation (evaluate.hpp:38-44) as bit patterns, plus the
// sorted trace (sim.hpp:34-42) as [stage, kind, microbatch, start, end].
int ref_evaluate_trace_json(const char* model, const char* cluster, const char* train,
                            const char* plan, char** out) {
  json result;
  int status = 0;
  try {
    hetplan::ModelSpec m = hetplan::model_from_json(json::parse(model));
    hetplan::ClusterSpec c = hetplan::cluster_from_json(json::parse(cluster));
    hetplan::TrainConfig t = hetplan::train_from_json(json::parse(train));
    hetplan::ParallelPlan p = hetplan::plan_from_json(json::parse(plan));
    hetplan::PlanEvaluation e = hetplan::evaluate_plan_unchecked(p, m, c, t, true);
    json ev = eval_json(e);
    for (std::size_t i = 0; i < e.costs.times.size(); ++i) {
      ev["stages"][i]["busy"] = hex_bits(e.sim.per_stage_busy_s[i]);
      ev["stages"][i]["bubble"] = hex_bits(e.sim.per_stage_bubble_ratio[i]);
    }
    ev["micro_batches"] = e.micro_batches;
    ev["total_devices"] = e.total_devices;
    json tr = json::array();
    for (const auto& x : e.sim.trace)
      tr.push_back(json::array({x.stage, static_cast<int>(x.kind), x.microbatch, hex_bits(x.start_s),
                                hex_bits(x.end_s)}));
    ev["trace"] = std::move(tr);
    result["eval"] = std::move(ev);
  } catch (const std::exception& e) {
    status = 3;
    result["error"] = e.what();
  }
  result["status"] = status;
  *out = dup_string(result.dump());
  return status;
}

// simulate() (sim.cpp:63-195) on raw stage times: times is P x 4 doubles
// (fwd, bwd, send_fwd, send_bwd). Writes the makespan and compute ends.
int ref_simulate(int schedule_gpipe, const double* times, int P, long long M,
                 double* iteration, double* compute_end) {
  try {
    std::vector<hetplan::StageTimes> st(P);
    for (int i = 0; i < P; ++i)
      st[i] = {times[4 * i], times[4 * i + 1], times[4 * i + 2], times[4 * i + 3]};
    hetplan::SimResult r = hetplan::simulate(
        schedule_gpipe ? hetplan::Schedule::GPipe : hetplan::Schedule::OneFOneB, st, M, false);
    *iteration = r.iteration_time_s;
    for (int i = 0; i < P; ++i) compute_end[i] = r.per_stage_compute_end_s[i];
    return 0;
  } catch (const std::exception&) {
    return 3;
  }
}

// parse_profiles + calibrate (profile.cpp:63-135), as cli.cpp:107-114 runs
// them: the calibrated cluster, its per-group scalars as bit patterns, and
// the diagnostics in CLI order (parse first, then calibration).
int ref_calibrate_json(const char* model, const char* cluster, const char* profiles, char** out) {
  json result;
  int status = 0;
  try {
    hetplan::ModelSpec m = hetplan::model_from_json(json::parse(model));
    hetplan::ClusterSpec c = hetplan::cluster_from_json(json::parse(cluster));
    hetplan::ParsedProfiles parsed = hetplan::parse_profiles(std::string(profiles));
    hetplan::CalibrationResult cal = hetplan::calibrate(parsed.records, m, c);
    json diags = json::array();
    for (const auto& d : parsed.diagnostics) diags.push_back("profiles: " + d);
    for (const auto& d : cal.diagnostics) diags.push_back("calibration: " + d);
    json groups = json::array();
    for (const auto& g : cal.cluster.groups)
      groups.push_back(json{{"name", g.name},
                            {"compute_efficiency_bits", hex_bits(g.compute_efficiency)},
                            {"bwd_fwd_ratio_bits", hex_bits(g.bwd_fwd_ratio)}});
    result["cluster"] = hetplan::to_json(cal.cluster);
    result["groups"] = groups;
    result["diagnostics"] = diags;
  } catch (const hetplan::ConfigError& e) {
    status = 1;
    result["error"] = e.what();
  } catch (const std::exception& e) {
    status = 3;
    result["error"] = e.what();
  }
  result["status"] = status;
  *out = dup_string(result.dump());
  return status;
}

// split_layers (planner.cpp:42-84). Returns 0, 1 ConfigError, 2 InfeasibleError.
int ref_split_layers(int total, const double* w, int parts, int* out) {
  try {
    std::vector<int> r = hetplan::split_layers(total, std::vector<double>(w, w + parts));
    for (int i = 0; i < parts; ++i) out[i] = r[i];
    return 0;
  } catch (const hetplan::ConfigError&) {
    return 1;
  } catch (const hetplan::InfeasibleError&) {
    return 2;
  }
}

void ref_free(char* p) { std::free(p); }

}  // extern "C"
