// hp_device.hpp — device arena and the per-shard search driver interface.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "hp_host.hpp"

namespace hpd {

// Named, grow-only device buffers reused across searches on one context, so
// repeated searches (benchmarks, sweeps) do not pay cudaMalloc each time.
struct Arena {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  std::map<std::string, std::pair<void*, size_t>> bufs;

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
    for (auto& kv : bufs)
      if (kv.second.first) cudaFree(kv.second.first);
    bufs.clear();
  }
};

struct SearchOut {
  long long simulated = 0, pruned = 0;
  bool has_best = false;
  double best_time = 0.0;
  int best_leaf = -1;          // index into Problem::leaves
  std::vector<int> best_split;
  long long launches = 0;
  int hill_iterations = 0;
  double global_bound = 0.0;
};

// Full strategy sweep (time_bound_pruning = false) over `my_leaves`.
hph::Status search_full(Arena& a, const hph::Problem& p, const std::vector<int>& my_leaves,
                        SearchOut& out);

// Batched evaluate_plan_unchecked(...).sim.iteration_time_s of explicit plans.
hph::Status evaluate_plans(Arena& a, const hph::Problem& p, const hp_plan* plans, int n,
                           double* out_times);

}  // namespace hpd
