// hp_capi.cpp — the C ABI (include/hetplan_b200.h) over the host model and
// the sm_100a kernels. No exception crosses this boundary.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>

#include "../../include/hetplan_b200.h"
#include "hp_device.hpp"
#include "hp_eval.hpp"
#include "hp_host.hpp"
#include "hp_log.hpp"

struct hp_ctx {
  hpd::Arena arena;
  std::string err;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  hpl::Log log;  // of the last hp_search with HP_FLAG_LOG
  // The enumerated problem of the last hp_probe, handed to the next
  // hp_search of the same problem (a sharded default-mode search calls both
  // per search); one-shot, so every search still enumerates once.
  std::unique_ptr<hph::Problem> probed;
  std::string probed_key;
};

namespace {

thread_local std::string g_err;  // last error of calls made without a context

hp_status fail(hp_ctx* ctx, const hph::Status& s) {
  if (ctx) ctx->err = s.msg;
  else g_err = s.msg;
  return s.code;
}

hp_status fail(hp_ctx* ctx, hp_status code, const std::string& m) {
  return fail(ctx, hph::Status{code, m});
}

// The inputs of a problem, byte for byte (struct fields, arrays and names).
std::string problem_key(const hp_problem* in) {
  std::string k;
  auto put = [&k](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
  put(&in->model, sizeof in->model);
  put(&in->train, sizeof in->train);
  for (int g = 0; g < in->cluster.n_groups; ++g) {
    hp_group x = in->cluster.groups[g];
    const char* nm = x.name ? x.name : "";
    x.name = nullptr;
    put(&x, sizeof x);
    k.append(nm);
    k.push_back('\0');
  }
  for (int l = 0; l < in->cluster.n_links; ++l) {
    hp_link x = in->cluster.links[l];
    x.group_a_name = x.group_b_name = nullptr;
    put(&x, sizeof x);
  }
  hp_planner pl = in->planner;
  pl.pipeline_degrees = nullptr;
  pl.micro_batch_candidates = nullptr;
  put(&pl, sizeof pl);
  if (in->planner.n_pipeline_degrees > 0)
    put(in->planner.pipeline_degrees, sizeof(int32_t) * in->planner.n_pipeline_degrees);
  if (in->planner.n_micro_batch_candidates > 0)
    put(in->planner.micro_batch_candidates, sizeof(int64_t) * in->planner.n_micro_batch_candidates);
  return k;
}

hp_status prepare(hp_ctx* ctx, const hp_problem* problem, hph::Problem& p) {
  hph::Status s = hph::load_problem(problem, p);
  if (!s.ok()) return fail(ctx, s);
  hph::enumerate(p);
  for (const hph::LeafHost& lf : p.leaves)
    if (lf.M > 5000000) return fail(ctx, HP_INTERNAL, "simulate: micro_batches too large");
  return HP_OK;
}

// The plans hp_evaluate_plans / hp_evaluate_plan_full accept: the shapes
// evaluate_plan_unchecked (evaluate.cpp:23-107) gives a meaning, checked so
// the device's stage-index edge test (hp_core.cuh stage_compute) is the
// reference's layer_range test (begin == 0 / end == num_layers): stages
// cover [0, num_layers) contiguously, each non-empty (an empty or inverted
// range is what makes simulate reject negative stage times, sim.cpp:66-73).
hph::Status check_plan_shape(const hph::Problem& p, const hp_plan& pl) {
  auto bad = [](const std::string& m) { return hph::Status{HP_BAD_CONFIG, m}; };
  if (pl.n_stages < 1 || pl.n_stages > HP_MAX_STAGES) return bad("plan: bad stage count");
  if (pl.schedule != HP_GPIPE && pl.schedule != HP_1F1B) return bad("plan: unknown schedule");
  if (pl.micro_batches_per_dp_replica < 1) return bad("simulate: micro_batches must be >= 1");
  if (pl.micro_batches_per_dp_replica > 5000000) return bad("simulate: micro_batches too large");
  int next = 0;
  for (int i = 0; i < pl.n_stages; ++i) {
    const hp_stage& st = pl.stages[i];
    if (st.layer_begin != next || st.layer_end <= st.layer_begin)
      return bad("plan: stage " + std::to_string(i) + " layer range [" + std::to_string(st.layer_begin) + ", " +
                 std::to_string(st.layer_end) + ") does not continue the previous stage");
    next = st.layer_end;
    if (st.group < 0 || st.group >= static_cast<int>(p.groups.size())) return bad("plan: unknown device group");
    if (st.tp_degree < 1) return bad("compute_time: tp_degree must be >= 1");
    if (st.dp_degree < 1) return bad("plan: dp_degree must be >= 1");
    if (i + 1 < pl.n_stages && st.group != pl.stages[i + 1].group &&
        p.pair[st.group][pl.stages[i + 1].group] < 0)
      return bad("no link between stages " + std::to_string(i) + " and " + std::to_string(i + 1));
  }
  if (next != p.model.num_layers)
    return bad("plan: stages cover " + std::to_string(next) + " of " + std::to_string(p.model.num_layers) +
               " layers");
  return hph::Status{};
}

}  // namespace

extern "C" {

int hp_abi_version(void) { return HP_ABI_VERSION; }

hp_status hp_create(hp_ctx** out, int device) {
  if (!out) return HP_INTERNAL;
  *out = nullptr;
  hp_ctx* ctx = new hp_ctx();
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->arena.sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->arena.stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
  if (e == cudaSuccess && !hpd::reserve_local_memory().ok()) e = cudaErrorMemoryAllocation;
  if (e != cudaSuccess) {
    delete ctx;
    return HP_CUDA;
  }
  ctx->arena.device = device;
  *out = ctx;
  return HP_OK;
}

void hp_destroy(hp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->arena.device);
  ctx->arena.release();
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->arena.stream) cudaStreamDestroy(ctx->arena.stream);
  delete ctx;
}

const char* hp_last_error(const hp_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

hp_status hp_validate(hp_ctx* ctx, const hp_problem* problem) {
  hph::Problem p;
  hph::Status s = hph::load_problem(problem, p);
  return s.ok() ? HP_OK : fail(ctx, s);
}

hp_status hp_probe(hp_ctx* ctx, const hp_problem* problem, const hp_search_opts* opts,
                   double* bound) {
  if (!ctx || !bound) return HP_INTERNAL;
  cudaSetDevice(ctx->arena.device);
  *bound = std::numeric_limits<double>::infinity();
  ctx->probed.reset();
  auto pp = std::make_unique<hph::Problem>();
  hph::Problem& p = *pp;
  hp_status st = prepare(ctx, problem, p);
  if (st != HP_OK) return st;
  int shard = opts ? opts->shard_index : 0;
  int nshard = opts && opts->shard_count > 0 ? opts->shard_count : 1;
  if (shard < 0 || shard >= nshard) return fail(ctx, HP_BAD_CONFIG, "bad shard index");
  if (!p.pruning) return HP_OK;  // no probe pass when pruning is off
  hpd::SearchOut out;
  hph::Status s = hpd::search_default(ctx->arena, p, hph::shard_tasks(p, shard, nshard), false, 0.0,
                                      true, out);
  if (!s.ok()) return fail(ctx, s);
  *bound = out.global_bound;
  ctx->probed_key = problem_key(problem);
  ctx->probed = std::move(pp);
  return HP_OK;
}

hp_status hp_search(hp_ctx* ctx, const hp_problem* problem, const hp_search_opts* opts,
                    hp_result* result) {
  if (!ctx || !result) return HP_INTERNAL;
  cudaSetDevice(ctx->arena.device);
  std::memset(result, 0, sizeof(*result));
  auto h0 = std::chrono::steady_clock::now();
  std::unique_ptr<hph::Problem> probed = std::move(ctx->probed);
  if (probed && ctx->probed_key != problem_key(problem)) probed.reset();
  std::unique_ptr<hph::Problem> own;
  if (!probed) {
    own = std::make_unique<hph::Problem>();
    hp_status st = prepare(ctx, problem, *own);
    if (st != HP_OK) return st;
  }
  hph::Problem& p = probed ? *probed : *own;
  const auto h_prep = std::chrono::steady_clock::now();
  int shard = opts ? opts->shard_index : 0;
  int nshard = opts && opts->shard_count > 0 ? opts->shard_count : 1;
  if (shard < 0 || shard >= nshard) return fail(ctx, HP_BAD_CONFIG, "bad shard index");
  if (nshard > 1 && p.pruning && !(opts && opts->have_global_bound))
    return fail(ctx, HP_BAD_CONFIG,
                "sharded default-mode search needs the all-shard probe bound (hp_probe)");
  result->tasks = static_cast<int64_t>(p.tasks.size());
  result->global_bound = std::numeric_limits<double>::infinity();

  // Task-level prunes (planner.cpp:317-327, 395-400) are host decisions;
  // shard 0 reports them.
  if (shard == 0) {
    for (const hph::Task& t : p.tasks) {
      if (t.no_link) {
        result->candidates_pruned++;
        result->reason_counts[HP_REASON_NO_LINK]++;
      } else if (t.leaf_begin == t.leaf_end) {
        result->candidates_pruned++;
        result->reason_counts[HP_REASON_NO_ASSIGNMENT]++;
      }
    }
  }
  std::vector<int> mine;
  if (p.pruning) mine = hph::shard_tasks(p, shard, nshard);
  else mine = hph::shard_leaves(p, shard, nshard);
  result->host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  ctx->arena.time_evals = opts && (opts->flags & HP_FLAG_TIME_KERNELS);
  ctx->arena.shard_count = nshard;
  const bool want_log = opts && (opts->flags & HP_FLAG_LOG);
  ctx->log.clear();
  ctx->arena.log.reset();
  ctx->arena.log.on = want_log;
  hpd::SearchOut out;
  hph::Status s;
  for (int attempt = 0;; ++attempt) {
    out = hpd::SearchOut{};
    cudaEventRecord(ctx->ev0, ctx->arena.stream);
    if (p.pruning) {
      bool have = opts && opts->have_global_bound;
      s = hpd::search_default(ctx->arena, p, mine, have, have ? opts->global_bound : 0.0, false, out);
    } else {
      s = hpd::search_full(ctx->arena, p, mine, out);
    }
    if (!s.ok()) {
      ctx->arena.log.on = false;
      return fail(ctx, s);
    }
    // a log that outgrew its buffers: the counters sized them, run again
    if (!(want_log && ctx->arena.log.overflow) || attempt >= 2) break;
  }
  ctx->arena.log.on = false;
  if (want_log) {
    if (ctx->arena.log.overflow) return fail(ctx, HP_INTERNAL, "search log: buffers overflowed twice");
    s = hpl::build(p, ctx->arena.log, out.global_bound, shard == 0, ctx->log);
    ctx->arena.log.reset();
    if (!s.ok()) return fail(ctx, s);
  }
  cudaEventRecord(ctx->ev1, ctx->arena.stream);
  cudaEventSynchronize(ctx->ev1);
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  result->device_ms = ms;
  if (std::getenv("HP_DEBUG_TIMING")) {  // diagnostics: host phases of this call
    const auto h_end = std::chrono::steady_clock::now();
    auto dms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "hp_search: prepare %.2f ms, shard %.2f ms, search+log %.2f ms (device %.2f ms)\n",
                 dms(h0, h_prep), result->host_ms - dms(h0, h_prep), dms(h_prep, h_end) - (result->host_ms - dms(h0, h_prep)),
                 ms);
  }
  result->gpu_launches = out.launches;
  result->eval_launches = out.eval_launches;
  result->eval_ms = out.eval_ms;
  result->eval_fp64_ops = out.eval_fp64_ops;
  result->h2d_bytes = out.h2d_bytes;
  result->d2h_bytes = out.d2h_bytes + sizeof(hp_result);
  result->hill_iterations = out.hill_iterations;
  result->device_simulated = out.dev_simulated;
  result->device_aborted = out.dev_aborted;
  result->device_screened = out.dev_screened;
  result->global_bound = p.pruning ? out.global_bound : std::numeric_limits<double>::infinity();
  if (p.pruning) {
    long long nl = 0;
    for (int ti : mine) nl += p.tasks[ti].leaf_end - p.tasks[ti].leaf_begin;
    result->leaves = nl;
  } else {
    result->leaves = static_cast<int64_t>(mine.size());
  }
  result->candidates_simulated += out.simulated;
  result->candidates_pruned += out.pruned;
  if (p.pruning) {
    result->reason_counts[HP_REASON_MEMORY] += out.pruned_mem;
    result->reason_counts[HP_REASON_BOUND] += out.pruned_bound;
  } else {
    result->reason_counts[HP_REASON_MEMORY] += out.pruned;
  }
  if (want_log && (ctx->log.simulated != result->candidates_simulated ||
                   ctx->log.pruned != result->candidates_pruned)) {
    ctx->log.clear();
    return fail(ctx, HP_INTERNAL, "search log: replay counts differ from the GPU counts");
  }
  if (out.has_best) {
    result->has_best = 1;
    result->best_time_s = out.best_time;
    const hph::LeafHost& lf = p.leaves[out.best_leaf];
    result->best_pp = p.tasks[lf.task].pp;
    hph::make_plan(p, lf, out.best_split.data(), result->best_plan);
  }
  return HP_OK;
}

hp_status hp_search_log(hp_ctx* ctx, hp_log_entry* entries, uint64_t entry_cap, char* text,
                        uint64_t text_cap, uint64_t* n_entries, uint64_t* text_bytes) {
  if (!ctx) return HP_INTERNAL;
  if (!ctx->log.valid) return fail(ctx, HP_BAD_CONFIG, "no search log: run hp_search with HP_FLAG_LOG");
  const uint64_t n = ctx->log.entries.size(), tb = ctx->log.text.size();
  if (n_entries) *n_entries = n;
  if (text_bytes) *text_bytes = tb;
  if (entries) {
    if (entry_cap < n) return fail(ctx, HP_BAD_CONFIG, "search log: entry buffer too small");
    if (n) std::memcpy(entries, ctx->log.entries.data(), sizeof(hp_log_entry) * n);
  }
  if (text) {
    if (text_cap < tb) return fail(ctx, HP_BAD_CONFIG, "search log: text buffer too small");
    if (tb) std::memcpy(text, ctx->log.text.data(), tb);
  }
  return HP_OK;
}

int hp_better_than(const hp_problem* problem, double time_a, const hp_plan* plan_a, double time_b,
                   const hp_plan* plan_b) {
  hph::Problem p;
  if (!hph::load_problem(problem, p).ok() || !plan_a || !plan_b) return 0;
  return hph::compare_plans(p, time_a, *plan_a, time_b, *plan_b);
}

hp_status hp_evaluate_plans(hp_ctx* ctx, const hp_problem* problem, const hp_plan* plans,
                            int32_t n, double* iteration_time_s) {
  if (!ctx) return HP_INTERNAL;
  cudaSetDevice(ctx->arena.device);
  hph::Problem p;
  hph::Status s = hph::load_problem(problem, p);
  if (!s.ok()) return fail(ctx, s);
  if (n < 0 || (n > 0 && (!plans || !iteration_time_s))) return fail(ctx, HP_BAD_CONFIG, "bad plan array");
  for (int k = 0; k < n; ++k) {
    hph::Status c = check_plan_shape(p, plans[k]);
    if (!c.ok()) return fail(ctx, c);
  }
  s = hpd::evaluate_plans(ctx->arena, p, plans, n, iteration_time_s);
  return s.ok() ? HP_OK : fail(ctx, s);
}

hp_status hp_evaluate_plan_full(hp_ctx* ctx, const hp_problem* problem, const hp_plan* plan, hp_plan_eval* eval,
                                hp_stage_eval* stages, hp_trace_event* trace, uint64_t trace_cap) {
  if (!ctx) return HP_INTERNAL;
  cudaSetDevice(ctx->arena.device);
  hph::Problem p;
  hph::Status s = hph::load_problem(problem, p);
  if (!s.ok()) return fail(ctx, s);
  if (!plan || !eval || !stages) return fail(ctx, HP_BAD_CONFIG, "hp_evaluate_plan_full: null argument");
  s = check_plan_shape(p, *plan);
  if (!s.ok()) return fail(ctx, s);
  s = hpe::evaluate_plan_full(ctx->arena, p, *plan, eval, stages, trace, trace_cap);
  return s.ok() ? HP_OK : fail(ctx, s);
}

}  // extern "C"
