// hp_host.hpp — host-side model of one search: validated inputs, the
// reference's task list and leaf list, and the split-independent cost tables
// uploaded to the GPU. Host C++ per the north star ("cluster/model config
// parsing and plan output stay in host C++"); it runs once per search.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hetplan_b200.h"
#include "hp_core.cuh"

namespace hph {

struct Status {
  hp_status code = HP_OK;
  std::string msg;
  bool ok() const { return code == HP_OK; }
};

// TaskSpec (planner.cpp:164-168) plus what run_task decides before any
// split is tried (planner.cpp:317-344, 395-400).
struct Task {
  int pp = 0;
  int spg[HP_MAX_GROUPS] = {0};  // stages per group
  std::vector<int> layout;       // stage -> group
  int layout_off = 0;
  int leaf_begin = 0, leaf_end = 0;
  bool no_link = false;          // adjacent groups without an inter-group link
};

struct LeafHost {
  int task;
  int dp;
  int64_t B;
  int B_idx;
  int64_t M;
  int tp_base;          // this leaf's tp per group: Problem::leaf_tp[tp_base + g]
  bool exhaustive;
  long long n_splits;   // C(L-1, pp-1), saturating
  double cost;          // work estimate for sharding
};

struct Problem {
  // inputs
  hp_model model{};
  std::vector<hp_group> groups;       // name pointers into `names`
  std::vector<std::string> names;     // group names (owned copies)
  std::string names_blob;             // names concatenated (Consts::names on the host)
  std::vector<int> name_off;
  std::vector<hp_link> links;
  hp_train train{};
  // normalised planner (planner.cpp:585-607)
  std::vector<int> pps;
  std::vector<int64_t> mbs;
  double headroom = 0.9;
  int beam = 24;
  int64_t limit = 2000;
  bool uniform_only = false, interleave = false, pruning = true;
  int schedule = HP_1F1B;
  // link index (first declaration wins, like types.cpp:26-56)
  int intra[HP_MAX_GROUPS], inter[HP_MAX_GROUPS], pair[HP_MAX_GROUPS][HP_MAX_GROUPS];
  // enumeration
  std::vector<Task> tasks;
  std::vector<LeafHost> leaves;
  std::vector<int32_t> leaf_tp;  // G per leaf (1 for groups the task leaves out)
  std::vector<uint8_t> layouts;  // concatenated task layouts
  int total_nodes = 0;
};

// Copies + validates (validate_spec, types.cpp:78-163; planner checks,
// planner.cpp:600-607) and normalises the planner config.
Status load_problem(const hp_problem* in, Problem& p);

// build_tasks (planner.cpp:238-304) and the leaf enumeration of run_task
// (planner.cpp:312-393), in reference order.
void enumerate(Problem& p);

// tp and nodes_used of group g in leaf h (planner.cpp:366-379: nodes =
// dp * tp / devices_per_node where the task has stages of g, else 0).
inline int leaf_tp(const Problem& p, const LeafHost& h, int g) { return p.leaf_tp[h.tp_base + g]; }
inline int leaf_nodes(const Problem& p, const LeafHost& h, int g) {
  if (p.tasks[h.task].spg[g] == 0) return 0;
  return static_cast<int>(static_cast<long long>(h.dp) * leaf_tp(p, h, g) / p.groups[g].devices_per_node);
}

// Exact-order cost terms.
double hop_time(const Problem& p, int link, int64_t B);            // cost_model.cpp:43-61
hpc::LeafGroup leaf_group(const Problem& p, int g, int tp, int64_t B, int dp, int nodes);
void fill_consts(const Problem& p, hpc::Consts& c);

// Deterministic leaf -> shard assignment (longest-processing-time first on
// the work estimate); returns the leaves of `shard` in reference order.
std::vector<int> shard_leaves(const Problem& p, int shard, int count);
// Default mode shards by task (tasks are sequential there).
std::vector<int> shard_tasks(const Problem& p, int shard, int count);

// better_than (planner.cpp:178-183) on two plans.
std::string encode_plan(const Problem& p, const hp_plan& plan);
int compare_plans(const Problem& p, double ta, const hp_plan& a, double tb, const hp_plan& b);

// Device record and per-group cost rows of leaf `li` (split_off and lg_off
// are left 0 for the caller to place). rows: n_groups entries.
hpc::Leaf device_leaf(const Problem& p, int li);
void leaf_rows(const Problem& p, int li, hpc::LeafGroup* rows);
// hop_time per (micro-batch candidate, link): [n_B][n_links]
std::vector<double> hop_table(const Problem& p);

// make_plan (planner.cpp:553-575) for a leaf and split.
void make_plan(const Problem& p, const LeafHost& lf, const int* split, hp_plan& out);

}  // namespace hph
