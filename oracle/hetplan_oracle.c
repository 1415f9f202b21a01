/* TEST INFRASTRUCTURE ONLY — NOT part of the product.
 *
 * Plain-C restatement of the reference planner's hot path, used by tests/ as
 * the parity checker and by bench.py's cpu_baseline leg ("port"). It follows
 * the reference line by line (citations are to /root/reference/proj/...),
 * including its floating-point association order, so results are
 * bit-identical to the compiled reference (oracle/_ref); tests pin that.
 *
 * The product path (paper_2405_16256_b200/csrc) never links or calls this.
 */
#include "hetplan_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define INF_D (1.0 / 0.0)

/* ---------------- cost model (core/src/cost_model.cpp) ------------------ */

/* p2p_activation_volume, cost_model.cpp:23-27 */
static double p2p_volume(int64_t B, int64_t seq, int64_t H, int bytes) {
  return (double)B * (double)seq * (double)H * bytes;
}

/* layer_flops forward, cost_model.cpp:29-35 */
static double layer_flops_fwd(const hp_model* m, int64_t micro_batch) {
  const double B = (double)micro_batch, L = (double)m->seq_length, H = (double)m->hidden_size;
  return 24.0 * B * L * H * H + 4.0 * B * L * L * H;
}

/* compute_time, cost_model.cpp:37-41 */
static double compute_time(double flops, const hp_group* g, int tp) {
  return flops / (tp * g->peak_tflops * 1e12 * g->compute_efficiency);
}

/* hop_time(...).time_s, cost_model.cpp:43-61 */
static double hop_time(double vol, const hp_link* l) {
  double wire = vol * 8.0 / (l->bandwidth_bits_per_s * l->efficiency);
  double t = l->latency_s;
  if (l->path == HP_CPU_STAGED) {
    double copy = vol / l->staging_copy_bytes_per_s;
    t += copy;
    t += wire;
    t += copy;
  } else {
    t += wire;
  }
  return t;
}

/* collective_time AllReduce, cost_model.cpp:63-73 */
static double allreduce_time(double vol, int ranks, const hp_link* l) {
  if (ranks == 1) return 0.0;
  double factor = 2.0;
  double steps = factor * (ranks - 1);
  double moved = factor * (ranks - 1) / (double)ranks * vol;
  return steps * l->latency_s + moved * 8.0 / (l->bandwidth_bits_per_s * l->efficiency);
}

/* stage_memory, cost_model.cpp:75-86 */
static double stage_memory(int count, int tp, const hp_model* m, const hp_train* t, int64_t B,
                           int in_flight) {
  const double layers = count;
  if (layers <= 0) return 0.0;
  const double H = (double)m->hidden_size;
  double weight_bytes = layers * 12.0 * H * H * m->bytes_per_element;
  double param_state = weight_bytes / tp * t->optimizer_state_multiplier;
  double Bd = (double)B;
  double act_per_mb = layers * Bd * (double)m->seq_length * H * m->activation_bytes_per_token_per_hidden;
  return param_state + in_flight * act_per_mb / tp;
}

typedef struct layer_cost_t { double fwd, bwd, param_bytes; } layer_cost_t;

/* layer_cost, cost_model.cpp:88-107 */
static layer_cost_t layer_cost(const hp_model* m, const hp_group* g, const hp_link* intra, int tp,
                               int64_t B) {
  layer_cost_t c;
  double fwd_flops = layer_flops_fwd(m, B);
  double fwd_compute = compute_time(fwd_flops, g, tp);
  double tp_volume = p2p_volume(B, m->seq_length, m->hidden_size, m->bytes_per_element);
  double tp_sync = 2.0 * allreduce_time(tp_volume, tp, intra);
  c.fwd = fwd_compute + tp_sync;
  c.bwd = fwd_compute * g->bwd_fwd_ratio + tp_sync;
  c.param_bytes = 12.0 * (double)m->hidden_size * (double)m->hidden_size * m->bytes_per_element;
  return c;
}

/* ---------------- links (core/src/types.cpp:26-56) ---------------------- */

typedef struct links_t {
  int intra[HP_MAX_GROUPS];
  int inter[HP_MAX_GROUPS];
  int pair[HP_MAX_GROUPS][HP_MAX_GROUPS];
} links_t;

static void index_links(const hp_cluster* c, links_t* lk) {
  for (int a = 0; a < HP_MAX_GROUPS; ++a) {
    lk->intra[a] = lk->inter[a] = -1;
    for (int b = 0; b < HP_MAX_GROUPS; ++b) lk->pair[a][b] = -1;
  }
  /* First match in declaration order, like the linear scans. */
  for (int i = c->n_links - 1; i >= 0; --i) {
    const hp_link* l = &c->links[i];
    if (l->scope == HP_INTRA_NODE) lk->intra[l->group_a] = i;
    else if (l->scope == HP_INTER_NODE) lk->inter[l->group_a] = i;
    else {
      lk->pair[l->group_a][l->group_b] = i;
      lk->pair[l->group_b][l->group_a] = i;
    }
  }
}

/* ---------------- simulator (core/src/sim.cpp) -------------------------- */

typedef struct stage_times { double fwd, bwd, sf, sb; } stage_times;

/* one_f_one_b_in_flight, sim.hpp:81-84 */
static int in_flight_1f1b(int stage, int P, int64_t M) {
  int64_t bound = P - stage;
  return (int)(bound < M ? bound : M);
}

/* simulate(), sim.cpp:63-195 — iteration time and per-stage compute end
 * (trace/in-flight bookkeeping is not needed for candidate selection). */
static int simulate(int gpipe, const stage_times* t, int P, int64_t M64, double* iteration,
                    double* compute_end) {
  if (P < 1 || M64 < 1 || M64 > 5000000) return -1;
  const int M = (int)M64;
  for (int i = 0; i < P; ++i)
    if (t[i].fwd < 0 || t[i].bwd < 0 || t[i].sf < 0 || t[i].sb < 0) return -1;
  size_t PM = (size_t)P * M;
  double* sendf = malloc(PM * sizeof(double));
  double* sendb = malloc(PM * sizeof(double));
  double* stage_free = calloc(P, sizeof(double));
  double* chan_f = calloc(P, sizeof(double));
  double* chan_b = calloc(P, sizeof(double));
  int* nf = calloc(P, sizeof(int)); /* forwards issued */
  int* nb = calloc(P, sizeof(int)); /* backwards issued */
  int* pos = calloc(P, sizeof(int));
  for (size_t k = 0; k < PM; ++k) sendf[k] = sendb[k] = -1.0;
  double max_end = 0.0;
  size_t done = 0, total = 2 * PM;
  /* stage_ops, sim.cpp:43-59: op k of stage i is F or B of some mb. */
  while (done < total) {
    int progressed = 0;
    for (int i = 0; i < P; ++i) {
      for (;;) {
        if (pos[i] >= 2 * M) break;
        int is_f, mb;
        if (gpipe) {
          is_f = pos[i] < M;
          mb = is_f ? pos[i] : pos[i] - M;
        } else {
          int w = in_flight_1f1b(i, P, M);
          /* F while warming up; then B,F alternation; trailing Bs. */
          if (nf[i] < w) is_f = 1;
          else if (nf[i] < M && nb[i] > nf[i] - w) is_f = 1;
          else is_f = 0;
          mb = is_f ? nf[i] : nb[i];
        }
        /* ready, sim.cpp:101-104 */
        if (is_f) {
          if (!(i == 0 || sendf[(size_t)(i - 1) * M + mb] >= 0)) break;
        } else {
          if (!(i == P - 1 || sendb[(size_t)(i + 1) * M + mb] >= 0)) break;
        }
        /* run, sim.cpp:106-146 */
        double data_ready = 0.0, dur;
        if (is_f) {
          if (i > 0) data_ready = sendf[(size_t)(i - 1) * M + mb];
          dur = t[i].fwd;
        } else {
          if (i < P - 1) data_ready = sendb[(size_t)(i + 1) * M + mb];
          dur = t[i].bwd;
        }
        double start = stage_free[i] < data_ready ? data_ready : stage_free[i];
        double end = start + dur;
        stage_free[i] = end;
        if (max_end < end) max_end = end;
        if (is_f) {
          if (i < P - 1) {
            double s = end < chan_f[i] ? chan_f[i] : end;
            double e = s + t[i].sf;
            chan_f[i] = e;
            sendf[(size_t)i * M + mb] = e;
            if (max_end < e) max_end = e;
          }
          nf[i]++;
        } else {
          if (i > 0) {
            double s = end < chan_b[i] ? chan_b[i] : end;
            double e = s + t[i].sb;
            chan_b[i] = e;
            sendb[(size_t)i * M + mb] = e;
            if (max_end < e) max_end = e;
          }
          nb[i]++;
        }
        pos[i]++;
        done++;
        progressed = 1;
      }
    }
    if (!progressed) break; /* cannot happen: the schedules are deadlock-free */
  }
  *iteration = max_end;
  for (int i = 0; i < P; ++i) compute_end[i] = stage_free[i];
  free(sendf); free(sendb); free(stage_free); free(chan_f); free(chan_b);
  free(nf); free(nb); free(pos);
  return done == total ? 0 : -2;
}

int ho_simulate(int gpipe, const double* times, int P, int64_t M, double* iteration,
                double* compute_end) {
  stage_times* t = malloc(sizeof(stage_times) * (P > 0 ? P : 1));
  for (int i = 0; i < P; ++i) {
    t[i].fwd = times[4 * i]; t[i].bwd = times[4 * i + 1];
    t[i].sf = times[4 * i + 2]; t[i].sb = times[4 * i + 3];
  }
  int rc = simulate(gpipe, t, P, M, iteration, compute_end);
  free(t);
  return rc;
}

/* ---------------- plan evaluation (core/src/evaluate.cpp) --------------- */

static int64_t eff_B(const hp_plan* p, const hp_train* t) {
  return p->micro_batch_size > 0 ? p->micro_batch_size : t->micro_batch_size;
}

/* plan_stage_times, evaluate.cpp:23-76 */
static void plan_stage_times(const hp_problem* pr, const links_t* lk, const hp_plan* plan,
                             stage_times* st, double* dp_sync) {
  const hp_model* m = &pr->model;
  const int P = plan->n_stages;
  const int64_t B = eff_B(plan, &pr->train);
  for (int i = 0; i < P; ++i) { st[i].fwd = st[i].bwd = st[i].sf = st[i].sb = 0.0; dp_sync[i] = 0.0; }
  double vol = p2p_volume(B, m->seq_length, m->hidden_size, m->bytes_per_element);
  for (int i = 0; i < P; ++i) {
    const hp_stage* s = &plan->stages[i];
    const hp_group* g = &pr->cluster.groups[s->group];
    const hp_link* intra = &pr->cluster.links[lk->intra[s->group]];
    layer_cost_t pl = layer_cost(m, g, intra, s->tp_degree, B);
    double layers = s->layer_end - s->layer_begin;
    if (s->layer_begin == 0) layers += m->edge_layer_cost_multiplier;
    if (s->layer_end == m->num_layers) layers += m->edge_layer_cost_multiplier;
    st[i].fwd = layers * pl.fwd;
    st[i].bwd = layers * pl.bwd;
    if (i + 1 < P) {
      const hp_stage* n = &plan->stages[i + 1];
      int li = s->group == n->group ? lk->inter[s->group] : lk->pair[s->group][n->group];
      double t = hop_time(vol, &pr->cluster.links[li]);
      st[i].sf = t;
      st[i + 1].sb = hop_time(vol, &pr->cluster.links[li]);
    }
    if (s->dp_degree > 1) {
      double grad_bytes = (double)(s->layer_end - s->layer_begin) * pl.param_bytes / s->tp_degree;
      const hp_link* dl = s->nodes_used > 1 ? &pr->cluster.links[lk->inter[s->group]] : intra;
      dp_sync[i] = allreduce_time(grad_bytes, s->dp_degree, dl);
    }
  }
}

/* evaluate_plan_unchecked(...).sim.iteration_time_s, evaluate.cpp:78-107 */
static int evaluate_plan(const hp_problem* pr, const links_t* lk, const hp_plan* plan,
                         double* out) {
  const int P = plan->n_stages;
  stage_times* st = malloc(sizeof(stage_times) * P);
  double* dps = malloc(sizeof(double) * P);
  double* ce = malloc(sizeof(double) * P);
  plan_stage_times(pr, lk, plan, st, dps);
  double pipeline;
  int rc = simulate(plan->schedule == HP_GPIPE, st, P, plan->micro_batches_per_dp_replica,
                    &pipeline, ce);
  double iteration = 0.0;
  for (int i = 0; i < P; ++i) {
    double v = ce[i] + dps[i];
    if (iteration < v) iteration = v;
  }
  *out = pipeline < iteration ? iteration : pipeline;
  free(st); free(dps); free(ce);
  return rc;
}

int ho_evaluate(const hp_problem* problem, const hp_plan* plan, double* iteration_time_s) {
  links_t lk;
  index_links(&problem->cluster, &lk);
  return evaluate_plan(problem, &lk, plan, iteration_time_s);
}

/* ---------------- planner (core/src/planner.cpp) ------------------------ */

/* split_layers, planner.cpp:42-84 */
int ho_split_layers(int total, const double* w, int parts, int* counts) {
  if (parts < 1) return 2;
  if (total < parts) return 2;
  double weight_sum = 0.0;
  for (int i = 0; i < parts; ++i) {
    if (!(w[i] > 0)) return 1;
    weight_sum += w[i];
  }
  double* fraction = malloc(sizeof(double) * parts);
  int* order = malloc(sizeof(int) * parts);
  int assigned = 0;
  for (int i = 0; i < parts; ++i) {
    double quota = total * w[i] / weight_sum;
    counts[i] = (int)floor(quota);
    fraction[i] = quota - counts[i];
    assigned += counts[i];
  }
  int remainder = total - assigned;
  /* std::stable_sort by fraction descending == stable insertion sort */
  for (int i = 0; i < parts; ++i) {
    int j = i;
    order[j] = i;
    while (j > 0 && fraction[order[j - 1]] < fraction[i]) { order[j] = order[j - 1]; --j; }
    order[j] = i;
  }
  for (int r = 0; r < remainder; ++r) ++counts[order[r % parts]];
  for (int i = 0; i < parts; ++i) {
    while (counts[i] == 0) {
      int donor = 0;
      for (int j = 1; j < parts; ++j) if (counts[j] > counts[donor]) donor = j;
      --counts[donor];
      ++counts[i];
    }
  }
  free(fraction); free(order);
  return 0;
}

/* contiguous_split_count, planner.cpp:134-147 */
static long long contiguous_split_count(int layers, int parts) {
  const long long kSat = 1LL << 40;
  if (parts < 1 || layers < parts) return 0;
  long long n = layers - 1, k = parts - 1;
  if (k > n - k) k = n - k;
  long long c = 1;
  for (long long i = 1; i <= k; ++i) {
    c = c * (n - k + i) / i;
    if (c > kSat) return kSat;
  }
  return c;
}

/* TaskSpec, planner.cpp:164-168 */
typedef struct task_t {
  int pp;
  int spg[HP_MAX_GROUPS];
  int* stage_group;
} task_t;

typedef struct norm_t {
  int n_pp;
  int* pps;
  int n_mb;
  int64_t* mbs;
} norm_t;

typedef struct ctx_t {
  const hp_problem* pr;
  links_t lk;
  norm_t nm;
  task_t* tasks;
  int n_tasks, cap_tasks;
  ho_leaf_cb cb;
  void* user;
} ctx_t;

static void push_task(ctx_t* c, int pp, const int* comp, const int* layout) {
  if (c->n_tasks == c->cap_tasks) {
    c->cap_tasks = c->cap_tasks ? 2 * c->cap_tasks : 64;
    c->tasks = realloc(c->tasks, sizeof(task_t) * c->cap_tasks);
  }
  task_t* t = &c->tasks[c->n_tasks++];
  t->pp = pp;
  for (int g = 0; g < HP_MAX_GROUPS; ++g) t->spg[g] = g < c->pr->cluster.n_groups ? comp[g] : 0;
  t->stage_group = malloc(sizeof(int) * pp);
  memcpy(t->stage_group, layout, sizeof(int) * pp);
}

/* std::next_permutation on an int array */
static int next_perm(int* a, int n) {
  int i = n - 2;
  while (i >= 0 && !(a[i] < a[i + 1])) --i;
  if (i < 0) {
    for (int l = 0, r = n - 1; l < r; ++l, --r) { int x = a[l]; a[l] = a[r]; a[r] = x; }
    return 0;
  }
  int j = n - 1;
  while (!(a[i] < a[j])) --j;
  int x = a[i]; a[i] = a[j]; a[j] = x;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) { x = a[l]; a[l] = a[r]; a[r] = x; }
  return 1;
}

static void layouts_for(ctx_t* c, int pp, const int* comp) {
  const hp_planner* pc = &c->pr->planner;
  const int G = c->pr->cluster.n_groups;
  int* layout = malloc(sizeof(int) * pp);
  int seen = 0;
  if (pc->allow_group_interleaving) {
    int* labels = malloc(sizeof(int) * pp);
    int k = 0;
    for (int g = 0; g < G; ++g) for (int s = 0; s < comp[g]; ++s) labels[k++] = g;
    do {
      push_task(c, pp, comp, labels);
      if (pc->stage_order_beam_width > 0 && ++seen >= pc->stage_order_beam_width) break;
    } while (next_perm(labels, pp));
    free(labels);
  } else {
    int part[HP_MAX_GROUPS], np = 0, perm[HP_MAX_GROUPS];
    for (int g = 0; g < G; ++g) if (comp[g] > 0) part[np++] = g;
    for (int b = 0; b < np; ++b) perm[b] = b;
    do {
      int k = 0;
      for (int b = 0; b < np; ++b) {
        int g = part[perm[b]];
        for (int s = 0; s < comp[g]; ++s) layout[k++] = g;
      }
      push_task(c, pp, comp, layout);
      if (pc->stage_order_beam_width > 0 && ++seen >= pc->stage_order_beam_width) break;
    } while (next_perm(perm, np));
  }
  free(layout);
}

static void comp_rec(ctx_t* c, int pp, int g, int remaining, int* cur) {
  const int G = c->pr->cluster.n_groups;
  if (g == G) {
    if (remaining == 0) layouts_for(c, pp, cur);
    return;
  }
  int cap = remaining < c->pr->cluster.groups[g].node_count ? remaining
                                                              : c->pr->cluster.groups[g].node_count;
  for (int s = 0; s <= cap; ++s) {
    cur[g] = s;
    comp_rec(c, pp, g + 1, remaining - s, cur);
  }
  cur[g] = 0;
}

/* build_tasks, planner.cpp:238-304 */
static void build_tasks(ctx_t* c) {
  int cur[HP_MAX_GROUPS] = {0};
  for (int k = 0; k < c->nm.n_pp; ++k) {
    int pp = c->nm.pps[k];
    if (pp < 1 || pp > c->pr->model.num_layers) continue;
    comp_rec(c, pp, 0, pp, cur);
  }
}

/* ---- per-task search state ---- */

typedef struct best_t {
  int has;
  double time;
  int pp;
  char* enc;
  hp_plan plan;
} best_t;

typedef struct task_result {
  best_t best;
  long long simulated, pruned;
  long long reasons[HP_REASON_COUNT];
  int log_nonempty;
} task_result;

/* encode_plan, planner.cpp:192-200 */
static char* encode_plan(const hp_problem* pr, const hp_plan* p) {
  size_t longest = 0;
  for (int g = 0; g < pr->cluster.n_groups; ++g)
    if (strlen(pr->cluster.groups[g].name) > longest) longest = strlen(pr->cluster.groups[g].name);
  size_t cap = 64 + (size_t)p->n_stages * (longest + 64);
  char* s = malloc(cap);
  size_t n = (size_t)snprintf(s, cap, "%s|%lld|%lld", p->schedule == HP_GPIPE ? "gpipe" : "1f1b",
                              (long long)p->micro_batches_per_dp_replica,
                              (long long)p->micro_batch_size);
  for (int i = 0; i < p->n_stages; ++i) {
    const hp_stage* st = &p->stages[i];
    n += (size_t)snprintf(s + n, cap - n, "|%s:%d-%d:%d:%d:%d", pr->cluster.groups[st->group].name,
                          st->layer_begin, st->layer_end, st->nodes_used, st->tp_degree,
                          st->dp_degree);
  }
  return s;
}

/* better_than, planner.cpp:178-183 */
static int better_than(double ta, int ppa, const char* ea, double tb, int ppb, const char* eb) {
  if (ta != tb) return ta < tb;
  if (ppa != ppb) return ppa < ppb;
  return strcmp(ea, eb) < 0;
}

/* memo: std::map<vector<int>, optional<double>> (planner.cpp:425-432) */
typedef struct memo_t {
  int pp;
  size_t cap, n;
  int* keys;     /* cap * pp */
  uint8_t* used;
  uint8_t* has;  /* optional engaged */
  double* val;
} memo_t;

static uint64_t hash_split(const int* s, int pp) {
  uint64_t h = 1469598103934665603ULL;
  for (int i = 0; i < pp; ++i) { h ^= (uint64_t)(uint32_t)s[i]; h *= 1099511628211ULL; }
  return h;
}

static void memo_init(memo_t* m, int pp) {
  m->pp = pp; m->cap = 64; m->n = 0;
  m->keys = malloc(sizeof(int) * m->cap * pp);
  m->used = calloc(m->cap, 1);
  m->has = calloc(m->cap, 1);
  m->val = malloc(sizeof(double) * m->cap);
}
static void memo_free(memo_t* m) { free(m->keys); free(m->used); free(m->has); free(m->val); }

static long memo_find(const memo_t* m, const int* s) {
  size_t i = hash_split(s, m->pp) & (m->cap - 1);
  while (m->used[i]) {
    if (memcmp(&m->keys[i * m->pp], s, sizeof(int) * m->pp) == 0) return (long)i;
    i = (i + 1) & (m->cap - 1);
  }
  return -1 - (long)i;
}

static void memo_put(memo_t* m, const int* s, int has, double v);
static void memo_grow(memo_t* m) {
  memo_t o = *m;
  m->cap *= 2; m->n = 0;
  m->keys = malloc(sizeof(int) * m->cap * m->pp);
  m->used = calloc(m->cap, 1);
  m->has = calloc(m->cap, 1);
  m->val = malloc(sizeof(double) * m->cap);
  for (size_t i = 0; i < o.cap; ++i)
    if (o.used[i]) memo_put(m, &o.keys[i * o.pp], o.has[i], o.val[i]);
  memo_free(&o);
}
static void memo_put(memo_t* m, const int* s, int has, double v) {
  if (2 * (m->n + 1) > m->cap) memo_grow(m);
  long f = memo_find(m, s);
  size_t i = (size_t)(-1 - f);
  m->used[i] = 1; m->has[i] = (uint8_t)has; m->val[i] = v;
  memcpy(&m->keys[i * m->pp], s, sizeof(int) * m->pp);
  m->n++;
}

typedef struct leaf_t {
  int dp;
  int64_t B;
  int tp[HP_MAX_GROUPS];
} leaf_t;

/* make_plan, planner.cpp:553-575 */
static void make_plan(const ctx_t* c, const task_t* task, const leaf_t* lf, const int* split,
                      hp_plan* plan) {
  plan->schedule = c->pr->planner.schedule;
  plan->micro_batch_size = lf->B;
  plan->micro_batches_per_dp_replica = c->pr->train.global_batch_size / ((int64_t)lf->dp * lf->B);
  plan->n_stages = task->pp;
  int begin = 0;
  for (int i = 0; i < task->pp; ++i) {
    int g = task->stage_group[i];
    hp_stage* s = &plan->stages[i];
    s->layer_begin = begin;
    s->layer_end = begin + split[i];
    begin += split[i];
    s->group = g;
    s->tp_degree = lf->tp[g];
    s->dp_degree = lf->dp;
    s->nodes_used = (int)((int64_t)lf->dp * s->tp_degree / c->pr->cluster.groups[g].devices_per_node);
  }
}

/* evaluate_split, planner.cpp:492-551. Returns 1 and *t when simulated. */
static int evaluate_split(const ctx_t* c, const task_t* task, const leaf_t* lf, const int* split,
                          double global_bound, task_result* out, double* t_out,
                          ho_leaf_info* li) {
  const hp_problem* pr = c->pr;
  hp_plan* plan = malloc(sizeof(hp_plan));
  make_plan(c, task, lf, split, plan);
  const int P = plan->n_stages;
  const int64_t M = plan->micro_batches_per_dp_replica;
  li->evaluated++;
  for (int i = 0; i < P; ++i) {
    int inf = plan->schedule == HP_GPIPE ? (int)M : in_flight_1f1b(i, P, M);
    const hp_stage* s = &plan->stages[i];
    double need = stage_memory(s->layer_end - s->layer_begin, s->tp_degree, &pr->model, &pr->train,
                               eff_B(plan, &pr->train), inf);
    double budget = pr->cluster.groups[s->group].memory_bytes * pr->planner.memory_headroom;
    if (need > budget) {
      out->log_nonempty = 1;
      out->pruned++;
      out->reasons[HP_REASON_MEMORY]++;
      li->pruned++;
      free(plan);
      return 0;
    }
  }
  double incumbent = global_bound;
  if (out->best.has && out->best.time < incumbent) incumbent = out->best.time;
  if (pr->planner.time_bound_pruning && incumbent < INF_D) {
    stage_times* st = malloc(sizeof(stage_times) * P);
    double* dps = malloc(sizeof(double) * P);
    plan_stage_times(pr, &c->lk, plan, st, dps);
    double lower = 0.0;
    for (int i = 0; i < P; ++i) {
      double v = M * (st[i].fwd + st[i].bwd);
      if (lower < v) lower = v;
    }
    free(st); free(dps);
    if (lower > incumbent) {
      out->log_nonempty = 1;
      out->pruned++;
      out->reasons[HP_REASON_BOUND]++;
      li->pruned++;
      free(plan);
      return 0;
    }
  }
  double t;
  evaluate_plan(pr, &c->lk, plan, &t);
  out->log_nonempty = 1;
  out->simulated++;
  li->simulated++;
  char* enc = encode_plan(pr, plan);
  if (!out->best.has || better_than(t, task->pp, enc, out->best.time, out->best.pp, out->best.enc)) {
    free(out->best.enc);
    out->best.has = 1;
    out->best.time = t;
    out->best.pp = task->pp;
    out->best.enc = enc;
    out->best.plan = *plan;
  } else {
    free(enc);
  }
  free(plan);
  *t_out = t;
  return 1;
}

typedef struct leaf_run {
  const ctx_t* c;
  const task_t* task;
  const leaf_t* lf;
  double global_bound;
  task_result* out;
  memo_t memo;
  ho_leaf_info* li;
} leaf_run;

/* try_split, planner.cpp:426-432 */
static int try_split(leaf_run* r, const int* split, double* t) {
  long f = memo_find(&r->memo, split);
  if (f >= 0) {
    *t = r->memo.val[f];
    return r->memo.has[f];
  }
  int has = evaluate_split(r->c, r->task, r->lf, split, r->global_bound, r->out, t, r->li);
  memo_put(&r->memo, split, has, has ? *t : 0.0);
  return has;
}

static void enum_rec(leaf_run* r, int remaining, int parts, int* cur, int depth) {
  double t;
  if (parts == 1) {
    cur[depth] = remaining;
    try_split(r, cur, &t);
    return;
  }
  for (int v = 1; remaining - v >= parts - 1; ++v) {
    cur[depth] = v;
    enum_rec(r, remaining - v, parts - 1, cur, depth + 1);
  }
}

/* leaf_splits, planner.cpp:404-490 */
static void leaf_splits(const ctx_t* c, const task_t* task, const leaf_t* lf, double global_bound,
                        int probe, task_result* out, ho_leaf_info* li) {
  const int pp = task->pp;
  const int L = c->pr->model.num_layers;
  if (L < pp) {
    out->log_nonempty = 1;
    out->pruned++;
    return;
  }
  leaf_run r = {c, task, lf, global_bound, out, {0}, li};
  memo_init(&r.memo, pp);
  int* uniform = malloc(sizeof(int) * pp);
  int* prop = malloc(sizeof(int) * pp);
  double* w = malloc(sizeof(double) * pp);
  double t;
  for (int i = 0; i < pp; ++i) w[i] = 1.0;
  ho_split_layers(L, w, pp, uniform);
  try_split(&r, uniform, &t);
  if (c->pr->planner.uniform_split_only) goto done;
  {
    /* stage_weights over merged blocks, planner.cpp:86-104 / :440-449 */
    double sum = 0.0;
    for (int i = 0; i < pp; ++i) {
      const hp_group* g = &c->pr->cluster.groups[task->stage_group[i]];
      double eff = g->peak_tflops * g->compute_efficiency * lf->tp[task->stage_group[i]];
      w[i] = eff;
      sum += eff;
    }
    for (int i = 0; i < pp; ++i) w[i] /= sum;
    ho_split_layers(L, w, pp, prop);
  }
  try_split(&r, prop, &t);
  if (probe) goto done;
  if (contiguous_split_count(L, pp) <= c->pr->planner.exhaustive_split_limit) {
    int* cur = malloc(sizeof(int) * pp);
    li->exhaustive = 1;
    enum_rec(&r, L, pp, cur, 0);
    free(cur);
    goto done;
  }
  {
    int* cur = malloc(sizeof(int) * pp);
    int* nb = malloc(sizeof(int) * pp);
    int* bestn = malloc(sizeof(int) * pp);
    memcpy(cur, prop, sizeof(int) * pp);
    double cur_t;
    int has = try_split(&r, cur, &cur_t);
    if (!has) {
      memcpy(cur, uniform, sizeof(int) * pp);
      has = try_split(&r, cur, &cur_t);
    }
    int max_steps = 4 * L;
    for (int step = 0; step < max_steps && has; ++step) {
      int bn_has = 0;
      double bn_t = 0.0;
      for (int i = 0; i + 1 < pp; ++i) {
        for (int d = 1; d >= -1; d -= 2) {
          memcpy(nb, cur, sizeof(int) * pp);
          nb[i] += d;
          nb[i + 1] -= d;
          if (nb[i] < 1 || nb[i + 1] < 1) continue;
          double tn;
          int h = try_split(&r, nb, &tn);
          if (h && (!bn_has || tn < bn_t)) {
            bn_has = 1;
            bn_t = tn;
            memcpy(bestn, nb, sizeof(int) * pp);
          }
        }
      }
      if (!bn_has || bn_t >= cur_t) break;
      memcpy(cur, bestn, sizeof(int) * pp);
      cur_t = bn_t;
      li->hill_steps++;
    }
    free(cur); free(nb); free(bestn);
  }
done:
  free(uniform); free(prop); free(w);
  memo_free(&r.memo);
}

static void ascending_divisors(int n, int* out, int* k) {
  *k = 0;
  for (int i = 1; i <= n; ++i) if (n % i == 0) out[(*k)++] = i;
}

/* run_task, planner.cpp:312-402 */
static void run_task(const ctx_t* c, int ti, double global_bound, int probe, task_result* out) {
  const task_t* task = &c->tasks[ti];
  const hp_problem* pr = c->pr;
  const int G = pr->cluster.n_groups;
  memset(out, 0, sizeof(*out));
  for (int i = 0; i + 1 < task->pp; ++i) {
    int a = task->stage_group[i], b = task->stage_group[i + 1];
    if (a != b && c->lk.pair[a][b] < 0) {
      out->log_nonempty = 1;
      out->pruned++;
      out->reasons[HP_REASON_NO_LINK]++;
      return;
    }
  }
  long long dp_max = INT64_MAX;
  for (int g = 0; g < G; ++g) {
    if (task->spg[g] == 0) continue;
    const hp_group* grp = &pr->cluster.groups[g];
    long long nps = grp->node_count / task->spg[g];
    long long v = nps * grp->devices_per_node;
    if (v < dp_max) dp_max = v;
  }
  int tpo[HP_MAX_GROUPS][64], ntp[HP_MAX_GROUPS];
  for (int g = 0; g < G; ++g) {
    if (task->spg[g] > 0) ascending_divisors(pr->cluster.groups[g].devices_per_node, tpo[g], &ntp[g]);
    else { tpo[g][0] = 1; ntp[g] = 1; }
  }
  for (long long dp = dp_max; dp >= 1; --dp) {
    for (int bi = 0; bi < c->nm.n_mb; ++bi) {
      int64_t B = c->nm.mbs[bi];
      if (pr->train.global_batch_size % (dp * B) != 0) continue;
      int idx[HP_MAX_GROUPS] = {0};
      for (;;) {
        leaf_t lf;
        lf.dp = (int)dp;
        lf.B = B;
        for (int g = 0; g < HP_MAX_GROUPS; ++g) lf.tp[g] = g < G ? tpo[g][idx[g]] : 1;
        int ok = 1;
        for (int g = 0; g < G && ok; ++g) {
          if (task->spg[g] == 0) continue;
          const hp_group* grp = &pr->cluster.groups[g];
          long long devices = dp * lf.tp[g];
          if (devices % grp->devices_per_node != 0) { ok = 0; break; }
          long long nodes_used = devices / grp->devices_per_node;
          if (nodes_used < 1 || nodes_used * task->spg[g] > grp->node_count) ok = 0;
        }
        if (ok) {
          ho_leaf_info li;
          memset(&li, 0, sizeof li);
          li.task = ti; li.pp = task->pp; li.dp = (int)dp; li.B = B;
          li.M = pr->train.global_batch_size / (dp * B);
          for (int g = 0; g < HP_MAX_GROUPS; ++g) li.tp[g] = lf.tp[g];
          leaf_splits(c, task, &lf, global_bound, probe, out, &li);
          if (c->cb && !probe) c->cb(c->user, &li);
          if (probe && out->simulated > 0) return;
        }
        int g = 0;
        while (g < G && ++idx[g] == ntp[g]) idx[g++] = 0;
        if (g == G) break;
      }
    }
  }
  if (!probe && out->simulated == 0 && !out->log_nonempty) {
    out->pruned++;
    out->reasons[HP_REASON_NO_ASSIGNMENT]++;
  }
}

static int cmp_int(const void* a, const void* b) { int x = *(const int*)a, y = *(const int*)b; return (x > y) - (x < y); }
static int cmp_i64(const void* a, const void* b) { int64_t x = *(const int64_t*)a, y = *(const int64_t*)b; return (x > y) - (x < y); }

/* search(), planner.cpp:579-685 (validation is left to the reference / the
 * product's host layer; the oracle assumes valid specs). */
int ho_search(const hp_problem* pr, hp_result* res, ho_leaf_cb cb, void* user) {
  ctx_t c;
  memset(&c, 0, sizeof c);
  c.pr = pr;
  c.cb = cb;
  c.user = user;
  index_links(&pr->cluster, &c.lk);
  memset(res, 0, sizeof(*res));
  /* normalise, planner.cpp:585-599 */
  const hp_planner* pc = &pr->planner;
  int total_nodes = 0;
  for (int g = 0; g < pr->cluster.n_groups; ++g) total_nodes += pr->cluster.groups[g].node_count;
  if (pc->n_pipeline_degrees == 0) {
    int cap = pr->model.num_layers < total_nodes ? pr->model.num_layers : total_nodes;
    c.nm.pps = malloc(sizeof(int) * (cap > 0 ? cap : 1));
    for (int p = 1; p <= cap; ++p) c.nm.pps[c.nm.n_pp++] = p;
  } else {
    c.nm.pps = malloc(sizeof(int) * pc->n_pipeline_degrees);
    memcpy(c.nm.pps, pc->pipeline_degrees, sizeof(int) * pc->n_pipeline_degrees);
    qsort(c.nm.pps, pc->n_pipeline_degrees, sizeof(int), cmp_int);
    int k = 0;
    for (int i = 0; i < pc->n_pipeline_degrees; ++i)
      if (k == 0 || c.nm.pps[k - 1] != c.nm.pps[i]) c.nm.pps[k++] = c.nm.pps[i];
    c.nm.n_pp = k;
  }
  if (pc->n_micro_batch_candidates == 0) {
    c.nm.mbs = malloc(sizeof(int64_t));
    c.nm.mbs[0] = pr->train.micro_batch_size;
    c.nm.n_mb = 1;
  } else {
    c.nm.mbs = malloc(sizeof(int64_t) * pc->n_micro_batch_candidates);
    memcpy(c.nm.mbs, pc->micro_batch_candidates, sizeof(int64_t) * pc->n_micro_batch_candidates);
    qsort(c.nm.mbs, pc->n_micro_batch_candidates, sizeof(int64_t), cmp_i64);
    int k = 0;
    for (int i = 0; i < pc->n_micro_batch_candidates; ++i)
      if (k == 0 || c.nm.mbs[k - 1] != c.nm.mbs[i]) c.nm.mbs[k++] = c.nm.mbs[i];
    c.nm.n_mb = k;
  }
  build_tasks(&c);
  res->tasks = c.n_tasks;

  double global_bound = INF_D;
  if (pc->time_bound_pruning) {
    for (int i = 0; i < c.n_tasks; ++i) {
      task_result pr_out;
      run_task(&c, i, INF_D, 1, &pr_out);
      if (pr_out.best.has && pr_out.best.time < global_bound) global_bound = pr_out.best.time;
      free(pr_out.best.enc);
    }
  }
  res->global_bound = global_bound;

  best_t best;
  memset(&best, 0, sizeof best);
  for (int i = 0; i < c.n_tasks; ++i) {
    task_result out;
    run_task(&c, i, global_bound, 0, &out);
    res->candidates_simulated += out.simulated;
    res->candidates_pruned += out.pruned;
    for (int k = 0; k < HP_REASON_COUNT; ++k) res->reason_counts[k] += out.reasons[k];
    if (out.best.has && (!best.has || better_than(out.best.time, out.best.pp, out.best.enc,
                                                  best.time, best.pp, best.enc))) {
      free(best.enc);
      best = out.best;
    } else {
      free(out.best.enc);
    }
  }
  int status = HP_OK;
  if (!best.has) {
    status = HP_INFEASIBLE;
  } else {
    res->has_best = 1;
    res->best_time_s = best.time;
    res->best_pp = best.pp;
    res->best_plan = best.plan;
  }
  free(best.enc);
  for (int i = 0; i < c.n_tasks; ++i) free(c.tasks[i].stage_group);
  free(c.tasks);
  free(c.nm.pps);
  free(c.nm.mbs);
  return status;
}
