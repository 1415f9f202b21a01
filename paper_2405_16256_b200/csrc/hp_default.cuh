// hp_default.cuh — time-bound-pruned ("default") search mode on the GPU.
// Included by hp_kernels.cu inside namespace hpk (shares c_consts, Bufs,
// Work and the evaluator device functions).
//
// With time_bound_pruning the reference prunes a candidate whose serial
// compute lower bound max_i M*(f_i+b_i) exceeds the incumbent
// min(global_bound, best-so-far-in-this-task) (planner.cpp:519-534). The
// incumbent evolves along the task's candidate sequence, so every task is a
// sequential process (path-dependent; SURVEY.md finding 1). One warp runs
// one task: each batch (seed, hill-climb neighbourhood, chunk of exhaustive
// compositions) is decided speculatively — memory gate and lower bound for all
// candidates in parallel, simulation of every candidate the batch-start
// incumbent does not already exclude — and then replayed in the reference's
// order by lane 0, which applies the evolving incumbent exactly. The
// incumbent only decreases, so the speculative set always contains every
// candidate the replay simulates.

struct TaskDev {
  int leaf_begin, leaf_end;  // this shard's leaves of the task, reference order
  int pp;
  int best_off;              // task best split row
};

struct TaskRes {
  double best_time;
  double probe_time;  // +inf when the probe simulated nothing
  long long simulated, pruned_mem, pruned_bound;
  int has_best, best_leaf;
};

// Per-block scratch (global memory): CH entries each for the candidates of
// one batch; 2*SC entries (SC = most leaves in a task) for the seeds of
// every leaf of the task.
struct DefScratch {
  long long* ids;
  double* lower;
  double* times;
  unsigned char* flag;  // bit0 valid, bit1 mem_ok, bit2 old
  double* dec;          // per-slot decision of a hill step (time or -1)
  int CH;
};

// Per-leaf seed state (indexed by leaf; computed once per search, by the
// probe pass when there is one, else by the main pass).
struct DefSeeds {
  unsigned char* flag;  // [2*leaf + s]: gate bits, bit3 = proportional equals uniform (memo hit)
  double* low;          // [2*leaf + s]: lower bounds
  unsigned char* done;  // [2*leaf + s]: tseed holds its simulated time already
  // exhaustive leaves: compositions the memory gate prunes, feasible ones,
  // and the least lower bound among the feasible (seeds, memo hits,
  // excluded) — a leaf whose least bound is above the incumbent is decided
  // without being enumerated again
  long long* xmem;
  long long* xfeas;
  double* xmin;
};

constexpr int DEF_CH = 1024;
#ifndef HP_DEF_WARPS
#define HP_DEF_WARPS 4  // warps per task (tuning)
#endif
constexpr int DEF_WARPS = HP_DEF_WARPS;
constexpr int DEF_THREADS = 32 * DEF_WARPS;

// Lower bound and memory gate of one candidate (serial over stages).
// Returns flag bits (valid | mem_ok) and the bound.
__device__ inline unsigned char cand_gate(const Consts& c, const Leaf& lf, const LeafGroup* lg,
                                          const uint8_t* slots, const double* hop, const int* split,
                                          double* lower) {
  const int P = lf.P;
  double lo = 0.0;
  bool mem_ok = true;
  for (int i = 0; i < P; ++i)
    if (split[i] < 1) return 0;
  for (int i = 0; i < P; ++i) {
    StageDur d;
    if (!stage_setup(c, lf, lg, slots, hop, i, split[i], d)) {
      mem_ok = false;  // planner.cpp:509: first failing stage prunes
      break;
    }
    lo = dmax(lo, (double)lf.M * (d.f + d.b));  // planner.cpp:526-528
  }
  *lower = lo;
  return (unsigned char)(1 | (mem_ok ? 2 : 0));
}

// composition rank in enumerate_splits order (inverse of unrank_composition)
__device__ inline long long rank_composition(const int* c, int total, int parts) {
  long long rank = 0;
  int rem = total;
  for (int j = 0; j < parts - 1; ++j) {
    int left = parts - j;
    for (int v = 1; v < c[j]; ++v) rank += binom(rem - v - 1, left - 2);
    rem -= c[j];
  }
  return rank;
}

__device__ __forceinline__ void eval_dispatch(int cls, const Bufs& b, const Work& w, int lane) {
  switch (cls) {
    case 0: eval_item<2, true>(b, w, lane); break;
    case 1: eval_item<4, true>(b, w, lane); break;
    case 2: eval_item<6, true>(b, w, lane); break;
    case 3: eval_item<8, true>(b, w, lane); break;
    case 4: eval_item<1, false>(b, w, lane); break;
    case 5: eval_item<2, false>(b, w, lane); break;
    case 6: eval_item<3, false>(b, w, lane); break;
    default: eval_item<8, false>(b, w, lane); break;
  }
}

struct TaskState {
  double best_t;
  int has_best;
  int best_leaf;
  long long sim, pmem, pbound;
};

// Lane 0: apply one decided, simulated candidate to the task best.
__device__ inline void take_best(const Bufs& b, TaskState& ts, int* tbest, int li, const int* split,
                                 double t) {
  bool better = !ts.has_best || t < ts.best_t;
  if (!better && t == ts.best_t) {
    const Leaf la = b.leaves[li];
    if (li == ts.best_leaf) {
      // same leaf: the encodings differ first at the first differing stage
      // end (split_enc_less, hp_search_core.cuh) — exact ties are common
      // between identical stages, so this is the hot case
      better = split_enc_less(la.P, split, tbest);
    } else {
      const Leaf lb = b.leaves[ts.best_leaf];
      better = cand_less(c_consts, t, la, b.lg + la.lg_off, b.layouts + la.layout_off, split, ts.best_t,
                         lb, b.lg + lb.lg_off, b.layouts + lb.layout_off, tbest);
    }
  }
  if (better) {
    ts.has_best = 1;
    ts.best_t = t;
    ts.best_leaf = li;
    const int P = b.leaves[li].P;
    for (int i = 0; i < P; ++i) tbest[i] = split[i];
  }
}

__device__ inline double incumbent(const TaskState& ts, double gb) {
  return ts.has_best && ts.best_t < gb ? ts.best_t : gb;
}

// Simulates the candidates ids[0..n) of kind `kind` for leaf li (any order)
// on the block's warps, cpw per warp pass. Results land where eval_item
// writes them; the caller syncs the block before and after.
__device__ inline void simulate_list(const Bufs& b, int li, int kind, const long long* ids, int n,
                                     int out_base, int warp, int lane) {
  const Leaf lf = b.leaves[li];
  const int cls = eval_class(lf.P, lf.M, lf.sched == 0);
  const int cpw = class_cpw(cls, lf.P);
  for (int g = warp * cpw; g < n; g += DEF_WARPS * cpw) {
    Work w;
    w.leaf = li;
    w.kind = kind;
    w.first = g;
    w.n = min(cpw, n - g);
    w.out = out_base + g;
    w.ids = ids;
    eval_dispatch(cls, b, w, lane);
  }
}

// HP_DEBUG_TASKS phase accounting: cycles since the last mark go to `acc`.
#define DBG_MARK(acc)                  \
  if (b.trace) {                       \
    const long long now_ = clock64();  \
    acc += now_ - dbg_c;               \
    dbg_c = now_;                      \
  }

// One block of DEF_WARPS warps per task, tasks pulled in `order` (longest
// expected first). The task's leaves run in reference order; per leaf every
// batch (the seeds, a hill-climb neighbourhood, a chunk of exhaustive
// compositions) is gated by all threads and the candidates the batch-start
// incumbent does not exclude are simulated by all warps (speculatively: the
// incumbent only decreases, so this is a superset of what the reference
// simulates), then thread 0 replays the batch in the reference's order with
// the evolving incumbent (planner.cpp:425-551). The seeds of every leaf and
// their gates are incumbent-free and computed for the whole task at once.
// probe: the probe pass (planner.cpp:640-651): stop a task at its first
// simulated seed and fold its time into *gb_bits (atomic min of the bit
// patterns of non-negative doubles); otherwise *gb_bits is the global bound.
__global__ void __launch_bounds__(DEF_THREADS) k_default(Bufs bg, const TaskDev* tasks, const int* order, int n_tasks,
                                                        int* next_task, TaskRes* res, int* tbest_rows, DefScratch sc,
                                                        DefSeeds sd, int seeds_ready, unsigned long long* gb_bits,
                                                        int probe, int uniform_only, StagedTables tt) {
  extern __shared__ __align__(128) unsigned char smem_tables[];
  __shared__ __align__(8) unsigned long long tables_bar;
  const Bufs b = stage_tables(bg, tt, smem_tables, &tables_bar);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  long long* ids = sc.ids + (size_t)blockIdx.x * sc.CH;  // global: the evaluators read it
  // batch decisions in shared memory: thread 0's in-order replay reads them
  // back serially, so they must be a few cycles away, not an L2 round trip
  __shared__ double lower[DEF_CH];
  __shared__ double dec[DEF_CH];
  __shared__ unsigned char flag[DEF_CH];
  Bufs bx = b;
  bx.xbuf = sc.times;
  const int xbase = blockIdx.x * sc.CH;
  const bool pruning = c_consts.pruning != 0;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  __shared__ int s_task, s_cnt, s_stop, s_moved;
  __shared__ double s_inc, s_dseed[2], s_cur_t;

  for (;;) {
    if (tid == 0) s_task = atomicAdd(next_task, 1);
    __syncthreads();
    const int kpos = s_task;
    if (kpos >= n_tasks) return;
    const int task = order[kpos];
    const TaskDev td = tasks[task];
    int* tbest = tbest_rows + td.best_off;
    TaskState ts{0.0, 0, -1, 0, 0, 0};  // meaningful in thread 0
    const double gb = probe ? INF : __longlong_as_double(*(volatile long long*)gb_bits);
    int lseq = 0;  // search-log segment counter of this task (thread 0)
    const bool logging = b.log.vals != nullptr && !probe;
    // HP_DEBUG_TASKS (thread 0's view): per task total cycles, leaves, hill
    // steps, simulations, and cycles per phase (seeds, simulation, gates,
    // replay, memo marks), accumulated at the block's sync points
    const long long dbg_t0 = b.trace ? clock64() : 0;
    long long dbg_steps = 0;
    long long dbg_sim = 0, dbg_gate = 0, dbg_rep = 0, dbg_seed = 0, dbg_c = 0, dbg_mo = 0;
    if (b.trace) dbg_c = clock64();

    // ---- seeds of every leaf and their gates (incumbent-free)
    const int nl = td.leaf_end - td.leaf_begin;
    for (int j = seeds_ready ? nl : tid; j < nl; j += DEF_THREADS) {
      const int li = td.leaf_begin + j;
      const Leaf lf = b.leaves[li];
      const LeafGroup* lg = b.lg + lf.lg_off;
      const uint8_t* slots = b.layouts + lf.layout_off;
      const double* hop = b.hop + lf.B_idx * c_consts.n_links;
      int* uni = b.uni + lf.split_off;
      int* prop = b.prop + lf.split_off;
      double w[HP_MAX_STAGES], frac[HP_MAX_STAGES];
      int ord[HP_MAX_STAGES];
      seed_splits(c_consts, lf, lg, slots, uni, prop, w, frac, ord);
      double lo = 0.0;
      sd.flag[2 * li] = cand_gate(c_consts, lf, lg, slots, hop, uni, &lo);
      sd.low[2 * li] = lo;
      if (same_split(uni, prop, lf.P)) {
        sd.flag[2 * li + 1] = 8;
        sd.low[2 * li + 1] = 0.0;
      } else {
        sd.flag[2 * li + 1] = cand_gate(c_consts, lf, lg, slots, hop, prop, &lo);
        sd.low[2 * li + 1] = lo;
      }
      sd.done[2 * li] = sd.done[2 * li + 1] = 0;
      if (lf.mode == 1 && !uniform_only) {
        const long long total = contiguous_split_count(c_consts.L, lf.P);
        const long long ru = rank_composition(uni, c_consts.L, lf.P);
        const long long rp = rank_composition(prop, c_consts.L, lf.P);
        int comp[HP_MAX_STAGES];
        long long nmem = 0, nfeas = 0;
        double mn = INF;
        unrank_composition(0, c_consts.L, lf.P, comp);
        for (long long r = 0; r < total; ++r) {
          if (r) next_composition(comp, lf.P);
          if (r == ru || r == rp) continue;
          double l;
          const unsigned char f = cand_gate(c_consts, lf, lg, slots, hop, comp, &l);
          if (!(f & 2)) {
            ++nmem;
          } else {
            ++nfeas;
            if (l < mn) mn = l;
          }
        }
        sd.xmem[li] = nmem;
        sd.xfeas[li] = nfeas;
        sd.xmin[li] = mn;
      }
    }
    __syncthreads();
    DBG_MARK(dbg_seed)

    for (int j = 0; j < nl; ++j) {
      const int li = td.leaf_begin + j;
      const Leaf lf = b.leaves[li];
      const int P = lf.P;
      const LeafGroup* lg = b.lg + lf.lg_off;
      const uint8_t* slots = b.layouts + lf.layout_off;
      const double* hop = b.hop + lf.B_idx * c_consts.n_links;
      int* uni = b.uni + lf.split_off;
      int* prop = b.prop + lf.split_off;
      const int nseed = uniform_only ? 1 : 2;

      // ---- seeds (planner.cpp:435-451): simulate those the incumbent at the
      // leaf's start admits, then decide them one at a time
      if (tid == 0) {
        const double inc0 = incumbent(ts, gb);
        int n = 0;
        for (int s = 0; s < nseed; ++s) {
          const unsigned char f = sd.flag[2 * li + s];
          if ((f & 8) || sd.done[2 * li + s]) continue;
          if ((f & 2) && !(pruning && inc0 < INF && sd.low[2 * li + s] > inc0)) {
            ids[n++] = s;
            sd.done[2 * li + s] = 1;  // (the time lands in tseed below)
          }
        }
        s_cnt = n;
      }
      __syncthreads();
      DBG_MARK(dbg_rep)
      if (s_cnt > 0) simulate_list(bx, li, 0, ids, s_cnt, xbase, warp, lane);
      __syncthreads();
      DBG_MARK(dbg_sim)
      if (tid == 0) {
        double dseed[2] = {-1.0, -1.0};
        for (int s = 0; s < nseed; ++s) {
          const unsigned char f = sd.flag[2 * li + s];
          if (f & 8) {  // memo hit (planner.cpp:425-432)
            dseed[1] = dseed[0];
            continue;
          }
          const double inc = incumbent(ts, gb);
          if (!(f & 2)) {
            ts.pmem++;
          } else if (pruning && inc < INF && sd.low[2 * li + s] > inc) {
            ts.pbound++;
          } else {
            const double t = b.tseed[2 * li + s];
            dseed[s] = t;
            ts.sim++;
            take_best(b, ts, tbest, li, s == 0 ? uni : prop, t);
            if (logging) {
              const long long off = log_reserve(b.log, task, lseq++, 1);
              if (off >= 0) b.log.vals[off] = t;
            }
          }
        }
        s_dseed[0] = dseed[0];
        s_dseed[1] = dseed[1];
        s_stop = probe && ts.sim > 0;
      }
      __syncthreads();
      DBG_MARK(dbg_seed)
      if (probe) {
        if (s_stop) break;
        continue;
      }
      if (uniform_only) continue;

      if (lf.mode == 1) {
        // ---- exhaustive, in rank order (planner.cpp:454-459)
        if (tid == 0) {
          // every feasible composition's bound above the incumbent: all
          // bound-pruned, nothing simulated, no need to enumerate again
          const double inc = incumbent(ts, gb);
          const double mn = sd.xmin[li];
          s_stop = pruning && inc < INF && mn > inc;
          if (s_stop) {
            ts.pmem += sd.xmem[li];
            ts.pbound += sd.xfeas[li];
          }
        }
        __syncthreads();
        if (s_stop) continue;
        const long long total = contiguous_split_count(c_consts.L, P);
        long long ru = 0, rp = 0;
        ru = rank_composition(uni, c_consts.L, P);
        rp = rank_composition(prop, c_consts.L, P);
        for (long long base = 0; base < total; base += sc.CH) {
          const int n = (int)min((long long)sc.CH, total - base);
          if (tid == 0) {
            s_inc = incumbent(ts, gb);
            s_cnt = 0;
          }
          __syncthreads();
          const double inc0 = s_inc;
          // gate: thread-contiguous rank ranges; survivors get a result slot
          const int per = (n + DEF_THREADS - 1) / DEF_THREADS;
          const int lo_k = tid * per, hi_k = min(n, lo_k + per);
          if (lo_k < hi_k) {
            int comp[HP_MAX_STAGES];
            unrank_composition(base + lo_k, c_consts.L, P, comp);
            for (int k = lo_k; k < hi_k; ++k) {
              if (k > lo_k) next_composition(comp, P);
              double l;
              unsigned char f = cand_gate(c_consts, lf, lg, slots, hop, comp, &l);
              const long long r = base + k;
              if (r == ru || r == rp) f |= 4;  // memo: seeds already decided
              flag[k] = f;
              lower[k] = l;
              if ((f & 1) && (f & 2) && !(f & 4) && !(pruning && inc0 < INF && l > inc0)) {
                const int pos = atomicAdd(&s_cnt, 1);
                ids[pos] = r;
                dec[k] = (double)pos;  // where its time will land
              }
            }
          }
          __syncthreads();
          const int cnt = s_cnt;
          if (cnt > 0) simulate_list(bx, li, 2, ids, cnt, xbase, warp, lane);
          __syncthreads();
          if (tid == 0) {
            int comp[HP_MAX_STAGES];
            int nv = 0;  // simulated times, compacted into dec[0..nv) (nv <= k: not yet read)
            for (int k = 0; k < n; ++k) {
              const unsigned char f = flag[k];
              if (f & 4) continue;  // memo hit
              if (!(f & 2)) {
                ts.pmem++;
                continue;
              }
              const double inc = incumbent(ts, gb);
              if (pruning && inc < INF && lower[k] > inc) {
                ts.pbound++;
                continue;
              }
              const double t = sc.times[xbase + (int)dec[k]];
              dec[nv++] = t;
              ts.sim++;
              if (!ts.has_best || t <= ts.best_t) {
                unrank_composition(base + k, c_consts.L, P, comp);
                take_best(b, ts, tbest, li, comp, t);
              }
            }
            if (logging) {
              const long long off = log_reserve(b.log, task, lseq++, nv);
              if (off >= 0)
                for (int q = 0; q < nv; ++q) b.log.vals[off + q] = dec[q];
            }
          }
          __syncthreads();
        }
        continue;
      }

      // ---- steepest descent (planner.cpp:461-489)
      int* cur = b.cur + lf.split_off;
      short* hist = b.hist + b.hist_off[li];
      const double ds0 = s_dseed[0], ds1 = s_dseed[1];
      double cur_t = 0.0;
      int start = 0;
      if (ds1 >= 0) {
        start = 1;
        cur_t = ds1;
      } else if (ds0 >= 0) {
        start = 2;
        cur_t = ds0;
      }
      if (start == 0) continue;
      for (int i = tid; i < P; i += DEF_THREADS) cur[i] = start == 1 ? prop[i] : uni[i];
      const int nslots = 2 * (P - 1);
      const int max_steps = 4 * c_consts.L;
      for (int step = 0; step < max_steps; ++step) {
        __syncthreads();
        // old flags (memo) by thread 0
        if (tid == 0) {
          int delta[HP_MAX_STAGES];
          for (int i = 0; i < P; ++i) delta[i] = 0;
          unsigned char old[2 * HP_MAX_STAGES];
          mark_old(lf, cur, uni, prop, hist, step, delta, old);
          for (int q = 0; q < nslots; ++q) flag[q] = old[q] ? 4 : 0;
          s_inc = incumbent(ts, gb);
          s_cnt = 0;
        }
        __syncthreads();
        DBG_MARK(dbg_mo)
        const double inc0 = s_inc;
        // gate every neighbour; list the ones to simulate
        for (int q = tid; q < nslots; q += DEF_THREADS) {
          int nbs[HP_MAX_STAGES];
          const int bb = q >> 1, d = (q & 1) ? -1 : 1;
          for (int i = 0; i < P; ++i) nbs[i] = cur[i];
          nbs[bb] += d;
          nbs[bb + 1] -= d;
          double l = 0.0;
          const unsigned char f0 = (nbs[bb] >= 1 && nbs[bb + 1] >= 1)
                                       ? cand_gate(c_consts, lf, lg, slots, hop, nbs, &l) : 0;
          const unsigned char f = flag[q] | f0;
          flag[q] = f;
          lower[q] = l;
          if ((f & 1) && (f & 2) && !(f & 4) && !(pruning && inc0 < INF && l > inc0)) ids[atomicAdd(&s_cnt, 1)] = q;
        }
        __syncthreads();
        DBG_MARK(dbg_gate)
        const int cnt = s_cnt;
        if (cnt > 0) simulate_list(bx, li, 1, ids, cnt, xbase, warp, lane);
        __syncthreads();
        DBG_MARK(dbg_sim)
        if (tid == 0) {
          const double* nbt = b.nb + b.nb_off[li];
          int nbs[HP_MAX_STAGES];
          int bq = -1;
          double bt = 0.0;
          int nv = 0;
          int moved = 0;
          for (int q = 0; q < nslots; ++q) {
            const unsigned char f = flag[q];
            if (!(f & 1)) continue;  // count < 1: skipped by the reference (:478)
            double t = -1.0;
            const int bb = q >> 1, d = (q & 1) ? -1 : 1;
            if (f & 4) {
              // memo hit: only the seeds can still matter for the argmin
              for (int i = 0; i < P; ++i) nbs[i] = cur[i];
              nbs[bb] += d;
              nbs[bb + 1] -= d;
              if (same_split(nbs, uni, P)) t = ds0;
              else if (same_split(nbs, prop, P)) t = ds1;
            } else if (!(f & 2)) {
              ts.pmem++;
            } else {
              const double inc = incumbent(ts, gb);
              if (pruning && inc < INF && lower[q] > inc) {
                ts.pbound++;
              } else {
                t = nbt[q];
                dec[nv++] = t;
                ts.sim++;
                if (!ts.has_best || t <= ts.best_t) {
                  for (int i = 0; i < P; ++i) nbs[i] = cur[i];
                  nbs[bb] += d;
                  nbs[bb + 1] -= d;
                  take_best(b, ts, tbest, li, nbs, t);
                }
              }
            }
            if (t >= 0 && (bq < 0 || t < bt)) {
              bq = q;
              bt = t;
            }
          }
          if (logging) {
            const long long off = log_reserve(b.log, task, lseq++, nv);
            if (off >= 0)
              for (int q = 0; q < nv; ++q) b.log.vals[off + q] = dec[q];
          }
          if (bq >= 0 && bt < cur_t) {
            const int bb = bq >> 1, d = (bq & 1) ? -1 : 1;
            cur[bb] += d;
            cur[bb + 1] -= d;
            hist[step] = (short)bq;
            cur_t = bt;
            moved = 1;
          }
          s_moved = moved;
          s_cur_t = cur_t;
        }
        __syncthreads();
        DBG_MARK(dbg_rep)
        ++dbg_steps;
        cur_t = s_cur_t;
        if (!s_moved) break;
      }
    }
    if (tid == 0) {
      TaskRes r;
      r.best_time = ts.best_t;
      r.probe_time = ts.has_best ? ts.best_t : INF;
      r.simulated = ts.sim;
      r.pruned_mem = ts.pmem;
      r.pruned_bound = ts.pbound;
      r.has_best = ts.has_best;
      r.best_leaf = ts.best_leaf;
      res[task] = r;
      if (probe && ts.has_best) atomicMin(gb_bits, (unsigned long long)__double_as_longlong(ts.best_t));
      if (b.trace) {
        unsigned long long* rec = b.trace + 8 * (size_t)(task + (probe ? n_tasks : 0));
        rec[0] = (unsigned long long)(clock64() - dbg_t0);
        rec[1] = (unsigned long long)(td.leaf_end - td.leaf_begin);
        rec[2] = (unsigned long long)dbg_steps | ((unsigned long long)(dbg_mo >> 10) << 20);
        rec[3] = (unsigned long long)ts.sim;
        rec[4] = (unsigned long long)dbg_seed;
        rec[5] = (unsigned long long)dbg_sim;
        rec[6] = (unsigned long long)dbg_gate;
        rec[7] = (unsigned long long)dbg_rep;
      }
    }
    __syncthreads();
  }
}

#undef DBG_MARK
