/* hetplan_b200.h — C ABI of the B200-native candidate-evaluation engine.
 *
 * Drop-in boundary for the reference planner's hot path:
 *   SearchOutcome hetplan::search(const ModelSpec&, const ClusterSpec&,
 *                                 const TrainConfig&, const PlannerConfig&, int jobs)
 *   (/root/reference/proj/core/include/hetplan/planner.hpp:115-116,
 *    implementation planner.cpp:579-685).
 * The reference exposes no FFI; this header is the flat, exception-free
 * equivalent (plain structs, pointers and sizes, no C++/torch types). The C++
 * function with the reference's exact signature is implemented over these
 * entry points in integration/hetplan_search_b200.cpp.
 *
 * Every entry point returns an hp_status; on failure hp_last_error(ctx) holds a
 * message. Status codes follow the reference's exception kinds
 * (errors.hpp:26-44, mapped to CLI exit codes at tools/cli.cpp:193-212):
 *   HP_BAD_CONFIG  <- ConfigError        (exit 1)
 *   HP_INFEASIBLE  <- InfeasibleError    (exit 2)
 *   HP_CUDA/HP_NCCL/HP_INTERNAL <- anything else (exit 3)
 */
#ifndef HETPLAN_B200_H_
#define HETPLAN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_ABI_VERSION 3
#define HP_MAX_GROUPS 16     /* device groups (accelerator types) per cluster */
#define HP_MAX_STAGES 256    /* pipeline stages per plan */

typedef enum hp_status {
  HP_OK = 0,
  HP_BAD_CONFIG = 1,
  HP_INFEASIBLE = 2,
  HP_CUDA = 3,
  HP_NCCL = 4,
  HP_INTERNAL = 5,
} hp_status;

typedef enum hp_schedule { HP_GPIPE = 0, HP_1F1B = 1 } hp_schedule;         /* types.hpp:134 */
typedef enum hp_scope { HP_INTRA_NODE = 0, HP_INTER_NODE = 1, HP_INTER_GROUP = 2 } hp_scope; /* types.hpp:63 */
typedef enum hp_path { HP_GPU_DIRECT = 0, HP_CPU_STAGED = 1 } hp_path;       /* types.hpp:75 */

/* ModelSpec, types.hpp:28-44 */
typedef struct hp_model {
  int32_t num_layers;
  int32_t num_heads;
  int64_t hidden_size;
  int64_t seq_length;
  int64_t vocab_size;
  int32_t bytes_per_element;
  int32_t _pad0;
  double activation_bytes_per_token_per_hidden;
  double edge_layer_cost_multiplier;
} hp_model;

/* DeviceGroup, types.hpp:47-61 */
typedef struct hp_group {
  const char* name; /* NUL-terminated UTF-8, any length; borrowed for the call */
  double peak_tflops;
  double memory_bytes;
  int32_t node_count;
  int32_t devices_per_node;
  double compute_efficiency;
  double bwd_fwd_ratio;
} hp_group;

/* Link + LinkScope, types.hpp:67-88; groups referenced by index into
 * hp_cluster.groups (the reference stores names and resolves them by linear
 * scan, types.cpp:26-56). group_b is ignored unless scope == HP_INTER_GROUP.
 * A caller resolving names passes -1 for a name no group has and, optionally,
 * the name itself in group_a_name / group_b_name, so validation reports it
 * like the reference ("link references unknown group '<name>'",
 * types.cpp:126-135); both may be NULL. */
typedef struct hp_link {
  int32_t scope;
  int32_t path;
  int32_t group_a;
  int32_t group_b;
  double bandwidth_bits_per_s;
  double latency_s;
  double efficiency;
  double staging_copy_bytes_per_s;
  const char* group_a_name;
  const char* group_b_name;
} hp_link;

/* ClusterSpec, types.hpp:90-103 */
typedef struct hp_cluster {
  int32_t n_groups;
  int32_t n_links;
  const hp_group* groups;
  const hp_link* links;
} hp_cluster;

/* TrainConfig, types.hpp:105-113 */
typedef struct hp_train {
  int64_t global_batch_size;
  int64_t micro_batch_size;
  double optimizer_state_multiplier;
} hp_train;

/* PlannerConfig, planner.hpp:27-49. Empty lists take the reference defaults
 * (planner.cpp:586-595). */
typedef struct hp_planner {
  int32_t n_pipeline_degrees;
  int32_t n_micro_batch_candidates;
  const int32_t* pipeline_degrees;
  const int64_t* micro_batch_candidates;
  double memory_headroom;
  int64_t exhaustive_split_limit;
  int32_t stage_order_beam_width;
  int32_t uniform_split_only;
  int32_t allow_group_interleaving;
  int32_t time_bound_pruning;
  int32_t schedule; /* hp_schedule */
  int32_t _pad0;
} hp_planner;

typedef struct hp_problem {
  hp_model model;
  hp_cluster cluster;
  hp_train train;
  hp_planner planner;
} hp_problem;

/* StageAssignment, types.hpp:124-132 (group by index). */
typedef struct hp_stage {
  int32_t layer_begin;
  int32_t layer_end;
  int32_t group;
  int32_t nodes_used;
  int32_t tp_degree;
  int32_t dp_degree;
} hp_stage;

/* ParallelPlan, types.hpp:136-154 (input digests are host-side provenance). */
typedef struct hp_plan {
  int32_t n_stages;
  int32_t schedule;
  int64_t micro_batches_per_dp_replica;
  int64_t micro_batch_size;
  hp_stage stages[HP_MAX_STAGES];
} hp_plan;

/* Search options. The candidate space is the reference's task list
 * (planner.cpp:238-304) expanded into leaves (task, dp, B, tp vector;
 * planner.cpp:353-391). A shard evaluates leaves whose position in that list
 * satisfies the shard's partition (weighted, deterministic), so N shards
 * together evaluate exactly the reference's candidates.
 *
 * Default mode (time_bound_pruning) needs the global probe bound
 * (planner.cpp:640-651): a single-device search computes it itself; a
 * sharded search passes the min over shards of hp_probe() in global_bound
 * with have_global_bound = 1. */
#define HP_FLAG_TIME_KERNELS 1 /* time every evaluator launch with CUDA events */
#define HP_FLAG_LOG 2          /* record the search log (SearchOutcome::log), read it
                                  back with hp_search_log() */

typedef struct hp_search_opts {
  int32_t shard_index;
  int32_t shard_count;
  int32_t have_global_bound;
  int32_t flags;       /* HP_FLAG_* */
  double global_bound; /* used when have_global_bound */
} hp_search_opts;

/* Per-shard result. has_best = 0 when the shard simulated no candidate.
 * best_time_s is the winner's iteration time (evaluate.cpp:90-97) with the
 * exact bit pattern of the reference. Counts follow planner.cpp:425-432,513-515,
 * 529-531,546 (memo hits are not counted; probe simulations are not counted).
 * reason_counts tallies pruned candidates per reason (hp_reason). */
typedef enum hp_reason {
  HP_REASON_MEMORY = 0,       /* "stage i memory ... exceeds ..."        planner.cpp:509-515 */
  HP_REASON_BOUND = 1,        /* "compute lower bound above incumbent"    planner.cpp:529-531 */
  HP_REASON_NO_LINK = 2,      /* "no heterogeneous link between ..."      planner.cpp:317-327 */
  HP_REASON_NO_ASSIGNMENT = 3,/* "no integral dp/tp/micro-batch assignment" planner.cpp:395-400 */
  HP_REASON_COUNT = 4
} hp_reason;

typedef struct hp_result {
  int64_t candidates_simulated;
  int64_t candidates_pruned;
  int64_t reason_counts[HP_REASON_COUNT];
  int64_t leaves;          /* leaves this shard evaluated */
  int64_t tasks;           /* tasks in the whole space */
  int32_t has_best;
  int32_t best_pp;
  double best_time_s;
  double global_bound;     /* probe bound used (inf when pruning is off) */
  double device_ms;        /* device time of this call (first to last kernel), CUDA events */
  int64_t gpu_launches;    /* kernels this call launched */
  int64_t eval_launches;   /* evaluator (k_eval*) launches among them */
  double eval_ms;          /* summed evaluator kernel time (HP_FLAG_TIME_KERNELS) */
  double eval_fp64_ops;    /* algorithmic FP64 add/max ops of simulated candidates */
  double h2d_bytes;        /* host->device bytes copied by this call */
  double d2h_bytes;        /* device->host bytes copied by this call */
  double host_ms;          /* host enumeration + table build time */
  int32_t hill_iterations; /* steepest-descent rounds */
  int32_t _pad1;
  /* Device work behind candidates_simulated (which counts like the
   * reference): candidates simulated to the end on the GPU, simulations
   * stopped early by the admissible lower bound, and candidates that bound
   * excluded before any simulation. The bound only removes candidates whose
   * time can neither be the hill-climb move nor tie the leaf best, so
   * decisions, counts and the winner are the reference's. Memo hits the GPU
   * re-evaluates are included here but not in candidates_simulated. */
  int64_t device_simulated;
  int64_t device_aborted;
  int64_t device_screened;
  hp_plan best_plan;
} hp_result;

typedef struct hp_ctx hp_ctx;

/* Creates a context bound to CUDA device `device` (one context per GPU; a
 * process may hold several). */
hp_status hp_create(hp_ctx** out, int device);
void hp_destroy(hp_ctx* ctx);
const char* hp_last_error(const hp_ctx* ctx);
int hp_abi_version(void);

/* Validation of the specs (types.cpp:78-163) and planner config
 * (planner.cpp:600-607). Host only; ctx may be NULL (then hp_last_error(NULL)
 * returns this thread's last message). */
hp_status hp_validate(hp_ctx* ctx, const hp_problem* problem);

/* Probe pass for this shard (planner.cpp:640-651): min over the shard's tasks
 * of the first simulated seed candidate. *bound = +inf when none. */
hp_status hp_probe(hp_ctx* ctx, const hp_problem* problem, const hp_search_opts* opts,
                   double* bound);

/* The hot path: enumerate, score and reduce this shard's candidates on the
 * GPU. HP_INFEASIBLE is NOT returned for an empty shard (has_best = 0); the
 * caller decides infeasibility after reducing over shards. */
hp_status hp_search(hp_ctx* ctx, const hp_problem* problem, const hp_search_opts* opts,
                    hp_result* result);

/* One SearchLogEntry (planner.hpp:95-99). The reference appends one per
 * candidate it decides, in task order and, inside a task, in visit order
 * (planner.cpp:306-551, 656-660); memo hits are not logged. Strings live in
 * the text buffer of hp_search_log as NUL-terminated UTF-8 and are
 * byte-identical to the reference's: `candidate` is the compact JSON
 * descriptor (nlohmann dump, keys sorted), `reason` the prune reason ("" when
 * simulated). */
typedef struct hp_log_entry {
  uint64_t candidate;  /* byte offset of the descriptor in text */
  uint64_t reason;     /* byte offset of the prune reason in text */
  double time_s;       /* simulated iteration time; -1.0 when pruned */
  int32_t task;        /* task index in build_tasks order: merge key across shards */
  int32_t leaf;        /* leaf index inside the task (run_task order); -1 for task-level entries */
} hp_log_entry;

/* The log of the last hp_search on ctx made with HP_FLAG_LOG: this shard's
 * entries in the reference's order. Sets *n_entries and *text_bytes; copies
 * when entries/text are non-NULL and their capacities suffice (else
 * HP_BAD_CONFIG). Shards own whole tasks (default mode) or whole leaves (full
 * mode), so the global log is the stable merge of the shards' logs by
 * (task, leaf). */
hp_status hp_search_log(hp_ctx* ctx, hp_log_entry* entries, uint64_t entry_cap, char* text,
                        uint64_t text_cap, uint64_t* n_entries, uint64_t* text_bytes);

/* Argmin order of the reference (planner.cpp:178-200): returns <0 when
 * (time_a, plan_a) ranks before (time_b, plan_b), >0 after, 0 if identical.
 * Host only; used to reduce per-shard results. */
int hp_better_than(const hp_problem* problem, double time_a, const hp_plan* plan_a,
                   double time_b, const hp_plan* plan_b);

/* Batched explicit-plan evaluation on the GPU: iteration_time_s of
 * evaluate_plan_unchecked (evaluate.cpp:78-107) for n plans. Plans must be
 * structurally valid (validate_plan, types.cpp:171-272). */
hp_status hp_evaluate_plans(hp_ctx* ctx, const hp_problem* problem, const hp_plan* plans,
                            int32_t n, double* iteration_time_s);

/* Multi-GPU search inside one process (the reference's `jobs` thread pool,
 * planner.cpp:612-664, becomes one host thread per GPU): hp_multi_create
 * binds one context per listed CUDA device and one NCCL communicator per
 * device (ncclCommInitAll; NCCL is loaded at run time). hp_search_multi
 * runs shard r on device r; default mode all-reduces (MIN) the shards' probe
 * minima into the global bound (planner.cpp:640-651), and the fixed-size
 * per-shard records are all-gathered (one NCCL collective each) and reduced
 * with better_than (planner.cpp:656-664). `result` is the reduced record
 * (device_ms = the slowest shard); per_device (optional) receives each
 * shard's record. Equal, bit for bit, to hp_search on one device.
 * hp_multi_search_log merges the shards' logs (HP_FLAG_LOG) in the
 * reference's order, with hp_search_log's buffer protocol. */
typedef struct hp_multi hp_multi;
int hp_device_count(void); /* visible CUDA devices (0 without a GPU) */
hp_status hp_multi_create(hp_multi** out, const int32_t* devices, int32_t n_devices);
void hp_multi_destroy(hp_multi* multi);
const char* hp_multi_last_error(const hp_multi* multi);
hp_status hp_search_multi(hp_multi* multi, const hp_problem* problem, int32_t flags, hp_result* result,
                          hp_result* per_device);
hp_status hp_multi_search_log(hp_multi* multi, hp_log_entry* entries, uint64_t entry_cap, char* text,
                              uint64_t text_cap, uint64_t* n_entries, uint64_t* text_bytes);

/* Winner post-processing (planner.cpp:681-684): the full PlanEvaluation of
 * evaluate_plan_unchecked(plan, ..., record_trace) (evaluate.cpp:78-107,
 * evaluate.hpp:38-44), bit for bit. The simulation runs on the GPU (every
 * node time); the trace sort, busy sums, in-flight counts, bubble ratios and
 * peak memory follow on the host in the reference's order (sim.cpp:148-209). */

/* TraceEvent, sim.hpp:34-42; kind: 0 F, 1 B, 2 SendF, 3 SendB */
typedef struct hp_trace_event {
  int32_t stage;
  int32_t kind;
  int32_t microbatch;
  int32_t _pad;
  double start_s;
  double end_s;
} hp_trace_event;

/* Per stage: PlanCosts (evaluate.hpp:28-31) and SimResult's per-stage
 * vectors (sim.hpp:44-53) after evaluate_plan_unchecked's DP-sync pass. */
typedef struct hp_stage_eval {
  double fwd_s;
  double bwd_s;
  double send_fwd_s;
  double send_bwd_s;
  double dp_sync_s;
  double busy_s;            /* per_stage_busy_s (compute + DP sync) */
  double compute_end_s;     /* per_stage_compute_end_s */
  double bubble_ratio;      /* per_stage_bubble_ratio */
  double peak_memory_bytes; /* peak_memory_bytes */
  int32_t peak_in_flight;   /* peak_in_flight */
  int32_t _pad;
} hp_stage_eval;

typedef struct hp_plan_eval {
  double iteration_time_s;       /* sim.iteration_time_s (incl. DP sync) */
  double pipeline_time_s;        /* flush time before gradient sync */
  double aggregate_bubble_ratio;
  int64_t micro_batches;
  int64_t total_devices;         /* ParallelPlan::total_devices, types.cpp:71-76 */
  int32_t n_stages;
  int32_t _pad;
  uint64_t n_trace;              /* trace events (4PM - 2M; written when trace != NULL) */
} hp_plan_eval;

/* stages: n_stages entries (caller-allocated). trace: NULL for no trace,
 * else trace_cap >= 4*P*M - 2*M entries, sorted by (start, stage, kind,
 * microbatch) like sim.cpp:162-167. Plan shape as hp_evaluate_plans. */
hp_status hp_evaluate_plan_full(hp_ctx* ctx, const hp_problem* problem, const hp_plan* plan,
                                hp_plan_eval* eval, hp_stage_eval* stages, hp_trace_event* trace,
                                uint64_t trace_cap);

#ifdef __cplusplus
}
#endif

#endif /* HETPLAN_B200_H_ */
