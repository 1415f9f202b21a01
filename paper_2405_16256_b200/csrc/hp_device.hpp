// hp_device.hpp — device arena and the per-shard search driver interface.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "hp_host.hpp"

namespace hpd {

// Raw search-log data of one search (HP_FLAG_LOG): the iteration times the
// GPU simulated, per stream in the reference's visit order. hp_log.cpp
// replays the reference's control flow over them to build the entries.
struct LogRaw {
  bool on = false;                      // requested for the next search
  unsigned long long val_cap = 1ULL << 22, seg_cap = 1ULL << 20;
  bool overflow = false;                // capacities grown; search must be re-run
  // full mode: key = shard leaf position; default mode: key = device task position
  std::vector<int> key_of;              // key -> global leaf (full) or global task (default)
  std::vector<std::vector<double>> streams;
  std::vector<double> tseed;            // full mode: uniform / proportional time per shard leaf
  std::vector<double> exh;              // full mode: time per bounded rank, exhaustive leaves
  std::vector<long long> exh_off;       // per shard leaf, -1 when not exhaustive
  void reset() {
    overflow = false;
    key_of.clear();
    streams.clear();
    tseed.clear();
    exh.clear();
    exh_off.clear();
  }
};

// Named, grow-only device buffers reused across searches on one context, so
// repeated searches (benchmarks, sweeps) do not pay cudaMalloc each time.
struct Arena {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::map<std::string, std::pair<void*, size_t>> bufs;
  // side streams (one per evaluator class, created on first use) and a pool
  // of ordering events
  cudaStream_t sides[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> markers;
  size_t markers_used = 0;

  cudaStream_t side(int k) {
    if (!sides[k]) cudaStreamCreateWithFlags(&sides[k], cudaStreamNonBlocking);
    return sides[k];
  }

  // An event for stream ordering; recycled after 256 uses (callers
  // synchronise long before that).
  cudaEvent_t marker() {
    if (markers.size() < 256) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      markers.push_back(e);
      return e;
    }
    return markers[markers_used++ % markers.size()];
  }

  LogRaw log;

  // Pinned staging for host->device table uploads (a pageable cudaMemcpy
  // stages through a driver buffer at a fraction of the bandwidth). A
  // bump allocator, reset per search; growing it first drains the stream.
  char* pinned = nullptr;
  size_t pinned_cap = 0, pinned_used = 0;
  char* stage(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (pinned_used + bytes > pinned_cap) {
      cudaStreamSynchronize(stream);
      if (pinned) cudaFreeHost(pinned);
      pinned = nullptr;
      size_t want = std::max(pinned_cap * 2, pinned_used + bytes + (size_t(8) << 20));
      if (cudaHostAlloc(reinterpret_cast<void**>(&pinned), want, cudaHostAllocDefault) != cudaSuccess) {
        pinned_cap = pinned_used = 0;
        return nullptr;
      }
      pinned_cap = want;
      pinned_used = 0;
    }
    char* p = pinned + pinned_used;
    pinned_used += bytes;
    return p;
  }

  // optional per-launch timing of the evaluator kernels (bench roofline)
  bool time_evals = false;
  int shard_count = 1;  // shards of the whole search (climb scheduling policy only)
  double h2d_bytes = 0.0, d2h_bytes = 0.0;  // per search
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;

  void event_pair(cudaEvent_t* e0, cudaEvent_t* e1) {
    while (ev_pool.size() < ev_used + 2) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    *e0 = ev_pool[ev_used++];
    *e1 = ev_pool[ev_used++];
  }

  // Sums the recorded pairs (caller synchronised the stream) and resets.
  double drain_events() {
    double ms = 0.0;
    for (size_t k = 0; k + 1 < ev_used; k += 2) {
      float x = 0.f;
      if (cudaEventElapsedTime(&x, ev_pool[k], ev_pool[k + 1]) == cudaSuccess) ms += x;
    }
    ev_used = 0;
    return ms;
  }

  hph::Status get(const char* name, size_t bytes, void** out) {
    auto& e = bufs[name];
    if (e.second < bytes) {
      if (e.first) cudaFree(e.first);
      e.first = nullptr;
      e.second = 0;
      size_t want = bytes + bytes / 4;
      cudaError_t err = cudaMalloc(&e.first, want);
      if (err != cudaSuccess)
        return hph::Status{HP_CUDA, std::string("cudaMalloc(") + name + "): " + cudaGetErrorString(err)};
      e.second = want;
    }
    *out = e.first;
    return hph::Status{};
  }

  void release() {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    pinned_cap = pinned_used = 0;
    for (auto& kv : bufs)
      if (kv.second.first) cudaFree(kv.second.first);
    bufs.clear();
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    ev_pool.clear();
    for (cudaEvent_t e : markers) cudaEventDestroy(e);
    markers.clear();
    for (cudaStream_t& s : sides)
      if (s) {
        cudaStreamDestroy(s);
        s = nullptr;
      }
  }
};

struct SearchOut {
  long long simulated = 0, pruned = 0, pruned_mem = 0, pruned_bound = 0;
  bool has_best = false;
  double best_time = 0.0;
  int best_leaf = -1;          // index into Problem::leaves
  std::vector<int> best_split;
  long long launches = 0;
  int hill_iterations = 0;
  double global_bound = 0.0;
  long long eval_launches = 0;
  double eval_ms = 0.0;        // summed evaluator kernel time (when timed)
  double eval_fp64_ops = 0.0;  // algorithmic FP64 add/max ops simulated
  // device work behind the counts: candidates simulated to the end, stopped
  // early by the admissible bound, and excluded by it before simulation
  // (the latter two are counted as simulated, like the reference, which
  // simulates them; their times cannot win or tie)
  long long dev_simulated = 0, dev_aborted = 0, dev_screened = 0;
  double h2d_bytes = 0.0, d2h_bytes = 0.0;
};

// Reserves the kernels' per-thread stack on the current device (once per
// context, hp_create).
hph::Status reserve_local_memory();

// Full strategy sweep (time_bound_pruning = false) over `my_leaves`.
hph::Status search_full(Arena& a, const hph::Problem& p, const std::vector<int>& my_leaves,
                        SearchOut& out);

// Time-bound-pruned (default) mode over whole tasks; runs the probe pass
// first unless have_bound (then `bound` is the all-shard probe minimum).
// probe_only stops after the probe (out.global_bound = this shard's min).
hph::Status search_default(Arena& a, const hph::Problem& p, const std::vector<int>& my_tasks,
                           bool have_bound, double bound, bool probe_only, SearchOut& out);

// Every node time of one explicit plan (winner post-processing): dur = per
// stage (f, b, sf, sb, dps); nodes = 8 arrays of P*M doubles (F start/end,
// B start/end, SendF start/end, SendB start/end at [stage * M + microbatch]);
// fin = per stage (final stage_free, forward channel end, backward channel end).
struct PlanNodes {
  int P = 0;
  long long M = 0;
  std::vector<double> dur, nodes, fin;
};
hph::Status plan_node_times(Arena& a, const hph::Problem& p, const hp_plan& plan, PlanNodes& out);

// Batched evaluate_plan_unchecked(...).sim.iteration_time_s of explicit plans.
hph::Status evaluate_plans(Arena& a, const hph::Problem& p, const hp_plan* plans, int n,
                           double* out_times);

}  // namespace hpd
