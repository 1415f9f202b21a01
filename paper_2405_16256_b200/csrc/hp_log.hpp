// hp_log.hpp — the search log (SearchOutcome::log, planner.hpp:95-107).
//
// The GPU records only what the host cannot cheaply recompute: the iteration
// time of every candidate the reference simulates, in visit order
// (hpd::LogRaw). This file replays the reference's per-leaf control flow
// (planner.cpp:404-551: seeds, memo, exhaustive enumeration or steepest
// descent, memory gate, compute lower bound) over those times and formats
// the entries byte-identically to the reference's nlohmann descriptors and
// prune reasons. Host only; runs after the search, only with HP_FLAG_LOG.
#pragma once

#include <string>
#include <vector>

#include "../../include/hetplan_b200.h"
#include "hp_device.hpp"
#include "hp_host.hpp"

namespace hpl {

struct Log {
  std::vector<hp_log_entry> entries;
  std::string text;  // NUL-terminated strings referenced by entries
  long long simulated = 0, pruned = 0;
  bool valid = false;
  void clear() {
    entries.clear();
    text.clear();
    simulated = pruned = 0;
    valid = false;
  }
};

// Builds this shard's log. global_bound: the bound the search pruned against
// (default mode). task_entries: emit the task-level entries (no link / no
// assignment), which belong to shard 0. Fails with HP_INTERNAL when the GPU
// streams and the replay disagree.
hph::Status build(const hph::Problem& p, const hpd::LogRaw& raw, double global_bound,
                  bool task_entries, Log& out);

}  // namespace hpl
