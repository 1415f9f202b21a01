/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference planner's
 * hot path (see hetplan_oracle.c). Uses the boundary's POD types. */
#ifndef HETPLAN_ORACLE_H_
#define HETPLAN_ORACLE_H_

#include "../include/hetplan_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One leaf (task, dp, B, tp) as visited by the search, for statistics. */
typedef struct ho_leaf_info {
  int32_t task;
  int32_t pp;
  int32_t dp;
  int32_t tp[HP_MAX_GROUPS];
  int64_t B;
  int64_t M;
  int32_t exhaustive;     /* 1 if C(L-1,pp-1) <= exhaustive_split_limit */
  int32_t hill_steps;     /* accepted hill-climb moves */
  int64_t evaluated;      /* distinct splits evaluated (memo misses) */
  int64_t simulated;
  int64_t pruned;
} ho_leaf_info;

typedef void (*ho_leaf_cb)(void* user, const ho_leaf_info* info);

/* search() (planner.cpp:579-685). Returns an hp_status. On success fills
 * result->best_plan/best_time_s/counts. `cb` may be NULL. */
int ho_search(const hp_problem* problem, hp_result* result, ho_leaf_cb cb, void* user);

/* evaluate_plan_unchecked(...).sim.iteration_time_s (evaluate.cpp:78-107). */
int ho_evaluate(const hp_problem* problem, const hp_plan* plan, double* iteration_time_s);

/* simulate() (sim.cpp:63-195): times = P x {fwd,bwd,send_fwd,send_bwd}. */
int ho_simulate(int gpipe, const double* times, int P, int64_t M, double* iteration,
                double* compute_end);

/* split_layers (planner.cpp:42-84). 0 ok, 1 ConfigError, 2 InfeasibleError. */
int ho_split_layers(int total, const double* w, int parts, int* out);

#ifdef __cplusplus
}
#endif
#endif
