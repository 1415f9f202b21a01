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

// Per-warp scratch (global memory), CH entries each.
struct DefScratch {
  long long* ids;
  double* lower;
  double* times;
  unsigned char* flag;  // bit0 valid, bit1 mem_ok, bit2 old
  double* dec;          // per-slot decision of a hill step (time or -1)
  int CH;
};

constexpr int DEF_CH = 1024;

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
    const Leaf la = b.leaves[li], lb = b.leaves[ts.best_leaf];
    better = cand_less(c_consts, t, la, b.lg + la.lg_off, b.layouts + la.layout_off, split, ts.best_t,
                       lb, b.lg + lb.lg_off, b.layouts + lb.layout_off, tbest);
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

// Simulates the candidates ids[0..n) of kind `kind` for leaf li (any order),
// cpw per warp pass. Results land where eval_item writes them.
__device__ inline void simulate_list(const Bufs& b, int li, int kind, const long long* ids, int n,
                                     int out_base, int lane) {
  const Leaf lf = b.leaves[li];
  const int cls = eval_class(lf.P, lf.M, lf.sched == 0);
  const int cpw = class_cpw(cls, lf.P);
  for (int g = 0; g < n; g += cpw) {
    Work w;
    w.leaf = li;
    w.kind = kind;
    w.first = g;
    w.n = min(cpw, n - g);
    w.out = out_base + g;
    w.ids = ids;
    eval_dispatch(cls, b, w, lane);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(128) k_default(Bufs b, const TaskDev* tasks, int n_tasks,
                                                 int* next_task, TaskRes* res, int* tbest_rows,
                                                 DefScratch sc, double global_bound, int probe,
                                                 int uniform_only) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long long* ids = sc.ids + (size_t)gw * sc.CH;
  double* lower = sc.lower + (size_t)gw * sc.CH;
  unsigned char* flag = sc.flag + (size_t)gw * sc.CH;
  double* dec = sc.dec + (size_t)gw * sc.CH;
  Bufs bx = b;
  bx.xbuf = sc.times;
  const int xbase = gw * sc.CH;
  const bool pruning = c_consts.pruning != 0;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);

  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(next_task, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= n_tasks) return;
    const TaskDev td = tasks[task];
    int* tbest = tbest_rows + td.best_off;
    TaskState ts{0.0, 0, -1, 0, 0, 0};
    const double gb = probe ? INF : global_bound;
    int lseq = 0;  // search-log segment counter of this task (lane 0)
    const bool logging = b.log.vals != nullptr && !probe;

    for (int li = td.leaf_begin; li < td.leaf_end; ++li) {
      const Leaf lf = b.leaves[li];
      const int P = lf.P;
      const LeafGroup* lg = b.lg + lf.lg_off;
      const uint8_t* slots = b.layouts + lf.layout_off;
      const double* hop = b.hop + lf.B_idx * c_consts.n_links;
      int* uni = b.uni + lf.split_off;
      int* prop = b.prop + lf.split_off;
      if (lane == 0) {
        double w[HP_MAX_STAGES], frac[HP_MAX_STAGES];
        int order[HP_MAX_STAGES];
        seed_splits(c_consts, lf, lg, slots, uni, prop, w, frac, order);
      }
      __syncwarp();

      // ---- seeds, decided one at a time (planner.cpp:435-451)
      double dseed[2] = {-1.0, -1.0};
      const bool prop_same = same_split(uni, prop, P);
      const int nseed = uniform_only ? 1 : 2;
      for (int s = 0; s < nseed; ++s) {
        if (s == 1 && prop_same) {  // memo hit
          dseed[1] = dseed[0];
          continue;
        }
        const int* split = s == 0 ? uni : prop;
        double lo = 0.0;
        unsigned char fl = 0;
        if (lane == 0) fl = cand_gate(c_consts, lf, lg, slots, hop, split, &lo);
        fl = __shfl_sync(0xffffffffu, fl, 0);
        lo = __shfl_sync(0xffffffffu, lo, 0);
        double inc = incumbent(ts, gb);
        int act;  // 0 mem, 1 bound, 2 simulate
        if (!(fl & 2)) act = 0;
        else if (pruning && inc < INF && lo > inc) act = 1;
        else act = 2;
        if (act == 2) {
          long long id = s;
          if (lane == 0) ids[0] = id;
          __syncwarp();
          simulate_list(bx, li, 0, ids, 1, xbase, lane);
          double t = b.tseed[2 * li + s];
          dseed[s] = t;
          if (lane == 0) {
            ts.sim++;
            take_best(b, ts, tbest, li, split, t);
            if (logging) {
              const long long off = log_reserve(b.log, task, lseq++, 1);
              if (off >= 0) b.log.vals[off] = t;
            }
          }
        } else if (lane == 0) {
          if (act == 0) ts.pmem++;
          else ts.pbound++;
        }
        ts.best_t = __shfl_sync(0xffffffffu, ts.best_t, 0);
        ts.has_best = __shfl_sync(0xffffffffu, ts.has_best, 0);
        ts.best_leaf = __shfl_sync(0xffffffffu, ts.best_leaf, 0);
      }
      if (probe) {
        if (__shfl_sync(0xffffffffu, (int)(ts.sim > 0), 0)) break;
        continue;
      }
      if (uniform_only) continue;

      if (lf.mode == 1) {
        // ---- exhaustive, in rank order (planner.cpp:454-459)
        const long long total = contiguous_split_count(c_consts.L, P);
        long long ru = 0, rp = 0;
        if (lane == 0) {
          ru = rank_composition(uni, c_consts.L, P);
          rp = rank_composition(prop, c_consts.L, P);
        }
        ru = __shfl_sync(0xffffffffu, ru, 0);
        rp = __shfl_sync(0xffffffffu, rp, 0);
        for (long long base = 0; base < total; base += sc.CH) {
          const int n = (int)min((long long)sc.CH, total - base);
          const double inc0 = incumbent(ts, gb);
          // gate all candidates of the chunk: lane-contiguous rank ranges
          const int per = (n + 31) / 32;
          const int lo_k = lane * per, hi_k = min(n, lo_k + per);
          if (lo_k < hi_k) {
            int comp[HP_MAX_STAGES];
            unrank_composition(base + lo_k, c_consts.L, P, comp);
            for (int k = lo_k; k < hi_k; ++k) {
              if (k > lo_k) next_composition(comp, P);
              double l;
              unsigned char f = cand_gate(c_consts, lf, lg, slots, hop, comp, &l);
              long long r = base + k;
              if (r == ru || r == rp) f |= 4;  // memo: seeds already decided
              flag[k] = f;
              lower[k] = l;
            }
          }
          __syncwarp();
          // survivors (ordered compaction not needed: results are indexed)
          int cnt = 0;
          for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            bool surv = false;
            if (k < n) {
              unsigned char f = flag[k];
              surv = (f & 1) && (f & 2) && !(f & 4) && !(pruning && inc0 < INF && lower[k] > inc0);
            }
            unsigned m = __ballot_sync(0xffffffffu, surv);
            if (surv) {
              int pos = cnt + __popc(m & ((1u << lane) - 1u));
              ids[pos] = base + k;
              dec[k] = (double)pos;  // where its time will land
            }
            cnt += __popc(m);
          }
          __syncwarp();
          if (cnt > 0) simulate_list(bx, li, 2, ids, cnt, xbase, lane);
          if (lane == 0) {
            int comp[HP_MAX_STAGES];
            bool have_comp = false;
            int nv = 0;  // simulated times, compacted into dec[0..nv) (nv <= k: not yet read)
            for (int k = 0; k < n; ++k) {
              unsigned char f = flag[k];
              if (f & 4) continue;  // memo hit
              if (!(f & 2)) {
                ts.pmem++;
                continue;
              }
              double inc = incumbent(ts, gb);
              if (pruning && inc < INF && lower[k] > inc) {
                ts.pbound++;
                continue;
              }
              double t = sc.times[xbase + (int)dec[k]];
              dec[nv++] = t;
              ts.sim++;
              if (!ts.has_best || t <= ts.best_t) {
                unrank_composition(base + k, c_consts.L, P, comp);
                have_comp = true;
                take_best(b, ts, tbest, li, comp, t);
              }
            }
            (void)have_comp;
            if (logging) {
              long long off = log_reserve(b.log, task, lseq++, nv);
              if (off >= 0)
                for (int j = 0; j < nv; ++j) b.log.vals[off + j] = dec[j];
            }
          }
          ts.best_t = __shfl_sync(0xffffffffu, ts.best_t, 0);
          ts.has_best = __shfl_sync(0xffffffffu, ts.has_best, 0);
          ts.best_leaf = __shfl_sync(0xffffffffu, ts.best_leaf, 0);
          __syncwarp();
        }
        continue;
      }

      // ---- steepest descent (planner.cpp:461-489)
      int* cur = b.cur + lf.split_off;
      short* hist = b.hist + b.hist_off[li];
      double cur_t;
      int start = 0;
      if (dseed[1] >= 0) {
        start = 1;
        cur_t = dseed[1];
      } else if (dseed[0] >= 0) {
        start = 2;
        cur_t = dseed[0];
      }
      if (start == 0) continue;
      if (lane == 0)
        for (int i = 0; i < P; ++i) cur[i] = start == 1 ? prop[i] : uni[i];
      __syncwarp();
      const int nslots = 2 * (P - 1);
      const int max_steps = 4 * c_consts.L;
      for (int step = 0; step < max_steps; ++step) {
        const double inc0 = incumbent(ts, gb);
        // old flags (memo) by lane 0
        if (lane == 0) {
          int delta[HP_MAX_STAGES];
          for (int i = 0; i < P; ++i) delta[i] = 0;
          unsigned char old[2 * HP_MAX_STAGES];
          mark_old(lf, cur, uni, prop, hist, step, delta, old);
          for (int q = 0; q < nslots; ++q) flag[q] = old[q] ? 4 : 0;
        }
        __syncwarp();
        // gate every neighbour
        for (int q = lane; q < nslots; q += 32) {
          int nbs[HP_MAX_STAGES];
          const int bb = q >> 1, d = (q & 1) ? -1 : 1;
          for (int i = 0; i < P; ++i) nbs[i] = cur[i];
          nbs[bb] += d;
          nbs[bb + 1] -= d;
          double l = 0.0;
          unsigned char f = (nbs[bb] >= 1 && nbs[bb + 1] >= 1)
                                ? cand_gate(c_consts, lf, lg, slots, hop, nbs, &l) : 0;
          flag[q] |= f;
          lower[q] = l;
        }
        __syncwarp();
        int cnt = 0;
        for (int q0 = 0; q0 < nslots; q0 += 32) {
          const int q = q0 + lane;
          bool surv = false;
          if (q < nslots) {
            unsigned char f = flag[q];
            surv = (f & 1) && (f & 2) && !(f & 4) && !(pruning && inc0 < INF && lower[q] > inc0);
          }
          unsigned m = __ballot_sync(0xffffffffu, surv);
          if (surv) ids[cnt + __popc(m & ((1u << lane) - 1u))] = q;
          cnt += __popc(m);
        }
        __syncwarp();
        if (cnt > 0) simulate_list(bx, li, 1, ids, cnt, xbase, lane);
        int moved = 0;
        if (lane == 0) {
          const double* nbt = b.nb + b.nb_off[li];
          int nbs[HP_MAX_STAGES];
          int bq = -1;
          double bt = 0.0;
          int nv = 0;
          // memo values of neighbours equal to the seeds
          for (int q = 0; q < nslots; ++q) {
            unsigned char f = flag[q];
            if (!(f & 1)) continue;  // count < 1: skipped by the reference (:478)
            double t = -1.0;
            const int bb = q >> 1, d = (q & 1) ? -1 : 1;
            if (f & 4) {
              // memo hit: only the seeds can still matter for the argmin
              for (int i = 0; i < P; ++i) nbs[i] = cur[i];
              nbs[bb] += d;
              nbs[bb + 1] -= d;
              if (same_split(nbs, uni, P)) t = dseed[0];
              else if (same_split(nbs, prop, P)) t = dseed[1];
            } else if (!(f & 2)) {
              ts.pmem++;
            } else {
              double inc = incumbent(ts, gb);
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
            long long off = log_reserve(b.log, task, lseq++, nv);
            if (off >= 0)
              for (int j = 0; j < nv; ++j) b.log.vals[off + j] = dec[j];
          }
          if (bq >= 0 && bt < cur_t) {
            const int bb = bq >> 1, d = (bq & 1) ? -1 : 1;
            cur[bb] += d;
            cur[bb + 1] -= d;
            hist[step] = (short)bq;
            cur_t = bt;
            moved = 1;
          }
        }
        moved = __shfl_sync(0xffffffffu, moved, 0);
        cur_t = __shfl_sync(0xffffffffu, cur_t, 0);
        ts.best_t = __shfl_sync(0xffffffffu, ts.best_t, 0);
        ts.has_best = __shfl_sync(0xffffffffu, ts.has_best, 0);
        ts.best_leaf = __shfl_sync(0xffffffffu, ts.best_leaf, 0);
        __syncwarp();
        if (!moved) break;
      }
    }
    if (lane == 0) {
      TaskRes r;
      r.best_time = ts.best_t;
      r.probe_time = ts.has_best ? ts.best_t : INF;
      r.simulated = ts.sim;
      r.pruned_mem = ts.pmem;
      r.pruned_bound = ts.pbound;
      r.has_best = ts.has_best;
      r.best_leaf = ts.best_leaf;
      res[task] = r;
    }
    __syncwarp();
  }
}
