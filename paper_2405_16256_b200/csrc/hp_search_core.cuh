// hp_search_core.cuh — per-candidate and per-leaf search logic, shared by
// the sm_100a kernels (hp_kernels.cu) and the CPU emulation test harness
// (tests/emu). Pure functions of their arguments; no CUDA intrinsics.
#pragma once

#include <cstddef>

#include "hp_core.cuh"

namespace hpc {

// Result codes stored per candidate slot.
constexpr double T_INVALID = -2.0;   // neighbour with a count < 1 (planner.cpp:478)
constexpr double T_MEMORY = -1.0;    // memory-pruned (planner.cpp:509-515)
constexpr double T_SKIP = __builtin_huge_val();  // feasible, bound above the current time (nb_screen)

// ------------------------------------------------------------ candidate setup

// Per-stage setup of one candidate (make_plan + memory gate + plan_stage_times,
// planner.cpp:499-517, evaluate.cpp:23-76). Returns false when the stage's
// memory exceeds the budget. hop[] is this leaf's row of hop times per link.
HPD bool stage_setup(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                     const double* hop, int i, int count, StageDur& d) {
  const LeafGroup& row = lg[slots[i]];
  const int g = row.group;
  const int P = lf.P;
  stage_compute(c, row, i, P, count, d);
  d.sf = 0.0;
  d.sb = 0.0;
  if (i + 1 < P) {
    int h = lg[slots[i + 1]].group;
    d.sf = hop[c.link_pair[g][h]];
  }
  if (i > 0) {
    int h = lg[slots[i - 1]].group;
    d.sb = hop[c.link_pair[h][g]];
  }
  d.dps = dp_sync(row, count);
  if (lf.mode == 3) return true;  // evaluate_plan_unchecked has no memory gate
  double need = stage_memory(c, count, row.tp, (double)lf.B, in_flight(c, i, P, lf.M));
  return !(need > c.budget[g]);
}

// Serial level-synchronous simulation of one candidate (all stages in one
// thread). Used by the small-P thread-per-candidate kernel and the tests.
// st/dur are caller scratch of P entries. Returns iteration_time_s
// (evaluate.cpp:90-97).
HPD double simulate_serial(bool gpipe, int P, int M, const StageDur* dur, StageState* st) {
  for (int i = 0; i < P; ++i) stage_init(st[i]);
  double max_end = 0.0;
  int done = 0;
  while (done < P) {
    // previous-level snapshot of the neighbours: process stages in
    // descending order so stage i-1 is still at its previous level when
    // stage i reads it; stage i+1's previous values are kept in (pchb, pnb).
    double pchb = 0.0;
    int pnb = 0;
    done = 0;
    for (int i = P - 1; i >= 0; --i) {
      double my_chb = st[i].chb;
      int my_nb = st[i].nb;
      int w = gpipe ? M : (P - i < M ? P - i : M);
      double lchf = i > 0 ? st[i - 1].chf : 0.0;
      int lnf = i > 0 ? st[i - 1].nf : 0;
      stage_level(gpipe, i, P, M, w, dur[i], st[i], lchf, lnf, pchb, pnb, max_end);
      pchb = my_chb;
      pnb = my_nb;
      done += stage_done(st[i], M) ? 1 : 0;
    }
  }
  double iteration = 0.0;
  for (int i = 0; i < P; ++i) iteration = dmax(iteration, st[i].free_t + dur[i].dps);
  return dmax(max_end, iteration);
}

// ------------------------------------------------------------ seeds

// Uniform and proportional seed splits of one leaf (planner.cpp:435-451):
// split_layers(L, 1...1) and split_layers(L, stage_weights(blocks)).
// w/frac: P doubles, order: P ints scratch.
HPD void seed_splits(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                     int* uni, int* prop, double* w, double* frac, int* order) {
  const int P = lf.P;
  for (int i = 0; i < P; ++i) w[i] = 1.0;
  split_layers(c.L, w, P, uni, frac, order);
  double sum = 0.0;
  for (int i = 0; i < P; ++i) {
    w[i] = lg[slots[i]].weight;
    sum += w[i];
  }
  for (int i = 0; i < P; ++i) w[i] /= sum;
  split_layers(c.L, w, P, prop, frac, order);
}

HPD bool same_split(const int* a, const int* b, int P) {
  for (int i = 0; i < P; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

// better_than within/between leaves: (time, pp, encoding).
HPD bool cand_less(const Consts& c, double ta, const Leaf& la, const LeafGroup* lga,
                   const uint8_t* sa, const int* ca, double tb, const Leaf& lb,
                   const LeafGroup* lgb, const uint8_t* sb, const int* cb) {
  if (ta != tb) return ta < tb;
  if (la.P != lb.P) return la.P < lb.P;
  EncStream ea{&c, sa, lga, ca, la.P, (long long)la.M, la.B, la.dp, 0, 0, 0, 0, {0}, 0};
  EncStream eb{&c, sb, lgb, cb, lb.P, (long long)lb.M, lb.B, lb.dp, 0, 0, 0, 0, {0}, 0};
  return enc_less(ea, eb);
}

// encode_plan order of two splits of the SAME leaf: the strings agree up to
// the first stage whose layer count differs; there the "end" fields differ
// and are compared as decimal strings followed by ':' (which sorts after
// every digit). Equivalent to cand_less for equal (time, pp, leaf).
HPD bool split_enc_less(int P, const int* a, const int* b) {
  int s = 0;
  for (int i = 0; i < P; ++i) {
    if (a[i] != b[i]) {
      char da[24], db[24];
      int na = fmt_ll(s + a[i], da), nb = fmt_ll(s + b[i], db);
      for (int k = 0;; ++k) {
        int x = k < na ? (unsigned char)da[k] : ':';
        int y = k < nb ? (unsigned char)db[k] : ':';
        if (x != y) return x < y;
        if (k >= na && k >= nb) return false;
      }
    }
    s += a[i];
  }
  return false;
}

// ------------------------------------------------------------ exhaustive
//
// stage_memory (cost_model.cpp:75-86) is non-decreasing in the layer count
// (every operation is monotone under round-to-nearest), so the memory gate
// of evaluate_split (planner.cpp:502-517) accepts exactly the compositions
// with count_i <= cap_i. The exhaustive regime therefore enumerates only the
// bounded compositions, in the reference's lexicographic order restricted to
// them, and counts the rest as memory-pruned analytically.

// cap_i = largest count in [1, L] that passes stage i's memory gate, 0 if none.
HPD void exh_caps(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                  int* caps) {
  const int P = lf.P;
  for (int i = 0; i < P; ++i) {
    const LeafGroup& row = lg[slots[i]];
    const double budget = c.budget[row.group];
    const int inf = in_flight(c, i, P, lf.M);
    int lo = 0, hi = c.L;  // invariant: lo passes (or 0), hi+1 fails
    while (lo < hi) {
      int mid = (lo + hi + 1) / 2;
      double need = stage_memory(c, mid, row.tp, (double)lf.B, inf);
      if (need > budget) hi = mid - 1;
      else lo = mid;
    }
    caps[i] = lo;
  }
}

// tbl[j*(L+1)+s] = number of compositions of s into stages j..P-1 with
// 1 <= count_i <= cap_i (tbl[P][0] = 1). Returns tbl[0][L].
HPD long long exh_table(int L, int P, const int* caps, long long* tbl) {
  const int W = L + 1;
  for (int s = 0; s <= L; ++s) tbl[P * W + s] = s == 0 ? 1 : 0;
  for (int j = P - 1; j >= 0; --j) {
    // tbl[j][s] = sum_{v=1..cap_j} tbl[j+1][s-v]  (sliding window)
    long long run = 0;
    for (int s = 0; s <= L; ++s) {
      if (s - 1 >= 0) run += tbl[(j + 1) * W + s - 1];
      if (s - 1 - caps[j] >= 0) run -= tbl[(j + 1) * W + s - 1 - caps[j]];
      tbl[j * W + s] = caps[j] >= 1 ? run : 0;
    }
  }
  return tbl[L];
}

// Bounded composition with lexicographic rank `rank` among the bounded ones.
HPD void unrank_bounded(long long rank, int L, int P, const int* caps, const long long* tbl,
                        int* out) {
  const int W = L + 1;
  int rem = L;
  for (int j = 0; j < P - 1; ++j) {
    for (int v = 1;; ++v) {
      long long cnt = (v <= caps[j] && rem - v >= 0) ? tbl[(j + 1) * W + rem - v] : 0;
      if (rank < cnt) {
        out[j] = v;
        rem -= v;
        break;
      }
      rank -= cnt;
    }
  }
  out[P - 1] = rem;
}

// Successor among the bounded compositions (false after the last one).
// sufcap[j] = sum_{k>=j} caps[k].
HPD bool next_bounded(int* c, int P, const int* caps, const int* sufcap) {
  int suffix = c[P - 1];
  for (int j = P - 2; j >= 0; --j) {
    // parts j+1..P-1 sum to `suffix`; try c[j]+1 with suffix-1 left for them
    const int rest = suffix - 1;
    if (c[j] + 1 <= caps[j] && rest >= P - 1 - j && rest <= sufcap[j + 1]) {
      c[j] += 1;
      int r = rest;
      for (int k = j + 1; k < P - 1; ++k) {
        int need_after = sufcap[k + 1];  // most the later parts can take
        int v = r - need_after;
        if (v < 1) v = 1;
        c[k] = v;
        r -= v;
      }
      c[P - 1] = r;
      return true;
    }
    suffix += c[j];
  }
  return false;
}

// ------------------------------------------------------------ neighbour screen
//
// An admissible lower bound on a candidate's iteration time, from one path
// of the simulation DAG: F(0,0) -> F(1,0) -> ... -> F(k,0) (forward sends),
// every op of stage k in order (2M ops), B(k,M-1) -> ... -> B(0,M-1)
// (backward sends), then stage 0's DP sync; or stage k's own DP sync after
// its last op. Each simulated node is max(predecessors) + duration and
// rounding is monotone, so the simulated value of any node is >= the path
// sum taken in path order, and the iteration time (a max over such nodes,
// evaluate.cpp:90-97) is >= every path bound. Summation order here differs
// from path order by far less than kScreenMargin (relative).
//
// A hill-climb neighbour whose bound exceeds the current point's time
// (times (1 + margin)) can neither be the improving move (planner.cpp:
// 479-487 needs t < current) nor tie the leaf best (best <= current), so it
// need not be simulated: it is recorded as T_SKIP (+inf: feasible, counted as
// simulated, never chosen). Decisions, counts and the winner are unchanged;
// only the search log needs every time and turns the screen off.
constexpr double kScreenMargin = 1e-6;

// Per-stage terms of the current split (X_k, Y_k of the bound and their
// prefix / suffix maxima).
struct StageLB {
  double f, b, sf, dps;  // durations of the current split
  double A, Bt;          // sum_{i<k} (f_i + sf_i), sum_{i<k} (sf_i + b_i)
  double PX, PY;         // max_{j<k} X_j, max_{j<k} Y_j
  double SX, SY;         // max_{j>=k} X_j, max_{j>=k} Y_j
  double PG, PGY;        // max_{j<k} GX_j, max_{j<k} GY_j (pair circuits, pair_gain)
  double SG, SGY;        // max_{j>=k} GX_j, max_{j>=k} GY_j
};
// (the device writes the pairs A/Bt, PX/PY, SX/SY, PG/PGY, SG/SGY as one
// 16-byte store each)
static_assert(sizeof(StageLB) % 16 == 0 && offsetof(StageLB, A) % 16 == 0 && offsetof(StageLB, PX) % 16 == 0 &&
                  offsetof(StageLB, SX) % 16 == 0 && offsetof(StageLB, PG) % 16 == 0 &&
                  offsetof(StageLB, SG) % 16 == 0,
              "StageLB pair layout");

// Durations of stage i of the current split at counts cur-1 ([0]) and
// cur+1 ([1]), the only counts a neighbour gives a stage, with their status:
// 0 count < 1 (planner.cpp:478), 1 memory-pruned, 2 feasible. Lets the
// screen (nb_screen_pre) and the neighbour evaluation skip stage_setup.
struct StageNb {
  double f[2], b[2], dps[2];
  int st[2];
};

HPD double neg_inf() { return -__builtin_huge_val(); }

// Pair-circuit term of the 1F1B bound. On stage k the op after B(k, m) is
// F(k, m + w_k) (w_k = P - k in-flight, M >= P - k); that forward reaches
// stage k+1 as F(k+1, (m + 1) + w_{k+1}), which stage k+1 runs right before
// B(k+1, m + 2). So B(k+1, m) -> B(k, m) -> F(k, m + w_k) -> F(k+1, ...) ->
// B(k+1, m + 2) is a circuit of length
//   cyc = f_k + b_k + f_{k+1} + b_{k+1} + 2 sf_k
// per two microbatches (the link k <-> k+1 carries both sends), taken n
// times from B(k+1, 0) while F(k, m + w_k) exists. B(k+1, 0) cannot start
// before microbatch 0's round trip (all forwards, then the backwards of the
// stages after k+1), and the remaining backwards of stage k+1 and the
// backward chain to stage 0 follow. Written against T0 = sum of all f, b and
// sends, the bound of pair k is
//   T0 + G_k + dps_0            (GX_k = G_k)
//   T0 + G_k - Bt_{k+1} + dps_{k+1}   (GY_k, the stage's own DP sync)
// with G_k = n cyc + (M - 1 - 2n) b_{k+1} returned here; -inf when the
// circuit does not exist (M < P - k). Slow links between two stages make
// this the binding bound: the per-stage bound misses 2 sf_k / 2 per
// microbatch of send time the 1F1B alternation cannot overlap.
HPD double pair_gain(long long M, int P, int k, double cyc, double b_e) {
  const long long w = P - k;
  if (M < w) return neg_inf();
  const long long n = (M - 1 >= w) ? (M - 1 - w) / 2 + 1 : 0;
  return (double)n * cyc + (double)(M - 1 - 2 * n) * b_e;
}

HPD double pair_cyc(double fk, double bk, double fe, double be, double sfk) {
  return ((fk + bk) + (fe + be)) + 2.0 * sfk;
}

// durations of stage i of the current split (feasible by construction)
HPD void lb_stage(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                  const double* hop, int i, int count, StageLB& s) {
  StageDur d;
  stage_setup(c, lf, lg, slots, hop, i, count, d);
  s.f = d.f;
  s.b = d.b;
  s.sf = d.sf;
  s.dps = d.dps;
}

// X_k = A_k + M (f_k + b_k) + Bt_k (then + dps_0), Y_k = A_k + M (f_k + b_k) + dps_k
HPD void lb_scan(const Leaf& lf, StageLB* s) {
  const int P = lf.P;
  const double M = (double)lf.M;
  double A = 0.0, Bt = 0.0, px = neg_inf(), py = neg_inf();
  for (int k = 0; k < P; ++k) {
    s[k].A = A;
    s[k].Bt = Bt;
    s[k].PX = px;
    s[k].PY = py;
    const double core = A + M * (s[k].f + s[k].b);
    const double X = core + Bt, Y = core + s[k].dps;
    s[k].SX = X;
    s[k].SY = Y;
    px = dmax(px, X);
    py = dmax(py, Y);
    A = A + s[k].f + s[k].sf;
    Bt = Bt + s[k].sf + s[k].b;
  }
  double sx = neg_inf(), sy = neg_inf();
  for (int k = P - 1; k >= 0; --k) {
    sx = dmax(sx, s[k].SX);
    sy = dmax(sy, s[k].SY);
    s[k].SX = sx;
    s[k].SY = sy;
  }
  // pair circuits (pair_gain): GX_k, GY_k for pairs k = 0 .. P-2
  double pg = neg_inf(), pgy = neg_inf();
  for (int k = 0; k < P; ++k) {
    s[k].PG = pg;
    s[k].PGY = pgy;
    double gx = neg_inf(), gy = neg_inf();
    if (k + 1 < P && lf.sched == 1) {
      gx = pair_gain(lf.M, P, k, pair_cyc(s[k].f, s[k].b, s[k + 1].f, s[k + 1].b, s[k].sf), s[k + 1].b);
      gy = gx - s[k + 1].Bt + s[k + 1].dps;
    }
    s[k].SG = gx;
    s[k].SGY = gy;
    pg = dmax(pg, gx);
    pgy = dmax(pgy, gy);
  }
  double sg = neg_inf(), sgy = neg_inf();
  for (int k = P - 1; k >= 0; --k) {
    sg = dmax(sg, s[k].SG);
    sgy = dmax(sgy, s[k].SGY);
    s[k].SG = sg;
    s[k].SGY = sgy;
  }
}

// T0 = sum of every f, b and send of the current split (pair_gain).
HPD double lb_total(const Leaf& lf, const StageLB* s) {
  const int k = lf.P - 1;
  return (HP_LDX(&s[k].A) + HP_LDX(&s[k].f)) + (HP_LDX(&s[k].Bt) + HP_LDX(&s[k].b));
}

// Pair-circuit part of the bound of the neighbour that gives stages bb and
// bb+1 the durations (f0, b0, p0) and (f1, b1, p1): the three pairs that
// contain a changed stage explicitly, the others through the prefix /
// suffix maxima shifted by the changed sums (T0 by dA + dB, Bt_{k+1} by dB
// for k > bb).
// The current split's row values the bounds of boundary bb's two
// neighbours read (stages bb-1 .. bb+2 of StageLB, stages bb, bb+1 of
// StageNb). nb_rows_load reads every one of them unconditionally (indices
// clamped; the unused ones are ignored), so the device issues them as one
// batch of independent loads.
struct NbRows {
  double nf[2][2], nbw[2][2], nd[2][2];  // [stage bb, bb+1][count -1, +1]
  int st[2][2];
  double PX, PY, A, Bt, sf, f, b;        // stage bb
  double f1, b1, sf1;                    // stage bb+1
  double SX2, SY2, SG2, SGY2, f2, b2, Bt2, d2;  // stage bb+2 (bb + 2 < P)
  double PGm, PGYm, fm, bm, sfm;         // stage bb-1 (bb >= 1)
  double dps0, T0;                       // stage 0's DP sync, lb_total
};

// (StageLB part)
HPD void lb_rows_load(const Leaf& lf, const StageLB* s, int bb, NbRows& r) {
  const int P = lf.P;
  const int b2 = bb + 2 < P ? bb + 2 : bb + 1, bm = bb >= 1 ? bb - 1 : bb;
  r.PX = HP_LDX(&s[bb].PX);
  r.PY = HP_LDX(&s[bb].PY);
  r.A = HP_LDX(&s[bb].A);
  r.Bt = HP_LDX(&s[bb].Bt);
  r.sf = HP_LDX(&s[bb].sf);
  r.f = HP_LDX(&s[bb].f);
  r.b = HP_LDX(&s[bb].b);
  r.f1 = HP_LDX(&s[bb + 1].f);
  r.b1 = HP_LDX(&s[bb + 1].b);
  r.sf1 = HP_LDX(&s[bb + 1].sf);
  r.SX2 = HP_LDX(&s[b2].SX);
  r.SY2 = HP_LDX(&s[b2].SY);
  r.SG2 = HP_LDX(&s[b2].SG);
  r.SGY2 = HP_LDX(&s[b2].SGY);
  r.f2 = HP_LDX(&s[b2].f);
  r.b2 = HP_LDX(&s[b2].b);
  r.Bt2 = HP_LDX(&s[b2].Bt);
  r.d2 = HP_LDX(&s[b2].dps);
  r.PGm = HP_LDX(&s[bm].PG);
  r.PGYm = HP_LDX(&s[bm].PGY);
  r.fm = HP_LDX(&s[bm].f);
  r.bm = HP_LDX(&s[bm].b);
  r.sfm = HP_LDX(&s[bm].sf);
  r.dps0 = HP_LDX(&s[0].dps);
  r.T0 = lb_total(lf, s);
}

HPD void nb_rows_load(const Leaf& lf, const StageLB* s, const StageNb* nbs, int bb, NbRows& r) {
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      r.nf[u][k] = HP_LDX(&nbs[bb + u].f[k]);
      r.nbw[u][k] = HP_LDX(&nbs[bb + u].b[k]);
      r.nd[u][k] = HP_LDX(&nbs[bb + u].dps[k]);
      r.st[u][k] = HP_LDX(&nbs[bb + u].st[k]);
    }
  lb_rows_load(lf, s, bb, r);
}

// Pair-circuit part of the bound of the neighbour that gives stages bb and
// bb+1 the durations (f0, b0, p0) and (f1, b1, p1): the three pairs that
// contain a changed stage explicitly, the others through the prefix /
// suffix maxima shifted by the changed sums (T0 by dA + dB, Bt_{k+1} by dB
// for k > bb).
HPD double pair_lb_rows(const Leaf& lf, const NbRows& r, int bb, double f0, double b0, double p0,
                        double f1, double b1, double p1, double dps0, double dA, double dB) {
#ifdef HP_NO_PAIR_LB
  return neg_inf();  // tuning / A-B: per-stage bound only
#endif
  if (lf.sched != 1) return neg_inf();
  const int P = lf.P;
  const long long M = lf.M;
  const double T = r.T0 + (dA + dB);
  double g = neg_inf(), gy = neg_inf();
  if (bb >= 1) {
    g = r.PGm;
    gy = r.PGYm;
    // pair (bb-1, bb)
    const double G = pair_gain(M, P, bb - 1, pair_cyc(r.fm, r.bm, f0, b0, r.sfm), b0);
    g = dmax(g, G);
    gy = dmax(gy, G - r.Bt + p0);
  }
  const double Bt1 = r.Bt + r.sf + b0;  // the neighbour's Bt_{bb+1}
  {
    // pair (bb, bb+1)
    const double G = pair_gain(M, P, bb, pair_cyc(f0, b0, f1, b1, r.sf), b1);
    g = dmax(g, G);
    gy = dmax(gy, G - Bt1 + p1);
  }
  if (bb + 2 < P) {
    // pair (bb+1, bb+2)
    const double G = pair_gain(M, P, bb + 1, pair_cyc(f1, b1, r.f2, r.b2, r.sf1), r.b2);
    g = dmax(g, G);
    gy = dmax(gy, G - (r.Bt2 + dB) + r.d2);
    // pairs bb+2 .. P-2
    g = dmax(g, r.SG2);
    gy = dmax(gy, r.SGY2 - dB);
  }
  return dmax(T + g + dps0, T + gy);
}

HPD double pair_lb_nb(const Leaf& lf, const StageLB* s, int bb, double f0, double b0, double p0,
                      double f1, double b1, double p1, double dps0, double dA, double dB) {
  NbRows r;
  lb_rows_load(lf, s, bb, r);
  return pair_lb_rows(lf, r, bb, f0, b0, p0, f1, b1, p1, dps0, dA, dB);
}

// Screens neighbour slot q of `cur` (boundary q >> 1, +1 for even q):
// T_INVALID (a count < 1, planner.cpp:478), T_MEMORY (a changed stage fails
// the memory gate; the others are the current split's), T_SKIP (bound above
// cur_t), or 0.0 (must be simulated).
HPD double nb_screen(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                     const double* hop, const int* cur, const StageLB* s, int q, double cur_t) {
  const int P = lf.P;
  const int bb = q >> 1;
  const int dir = (q & 1) ? -1 : 1;
  const int c0 = cur[bb] + dir, c1 = cur[bb + 1] - dir;
  if (c0 < 1 || c1 < 1) return T_INVALID;
  StageDur d0, d1;
  const bool ok0 = stage_setup(c, lf, lg, slots, hop, bb, c0, d0);
  const bool ok1 = stage_setup(c, lf, lg, slots, hop, bb + 1, c1, d1);
  if (!ok0 || !ok1) return T_MEMORY;
  const double M = (double)lf.M;
  const double dps0 = bb == 0 ? d0.dps : s[0].dps;
  double lb = dmax(s[bb].PX + dps0, s[bb].PY);  // k < bb (both -inf when bb == 0)
  const double A0 = s[bb].A, B0 = s[bb].Bt;
  lb = dmax(lb, A0 + M * (d0.f + d0.b) + dmax(B0 + dps0, d0.dps));
  const double A1 = A0 + d0.f + s[bb].sf, B1 = B0 + s[bb].sf + d0.b;
  lb = dmax(lb, A1 + M * (d1.f + d1.b) + dmax(B1 + dps0, d1.dps));
  const double dA = (d0.f - s[bb].f) + (d1.f - s[bb + 1].f);
  const double dB = (d0.b - s[bb].b) + (d1.b - s[bb + 1].b);
  if (bb + 2 < P) lb = dmax(lb, dmax(s[bb + 2].SX + dA + dB + dps0, s[bb + 2].SY + dA));
  lb = dmax(lb, pair_lb_nb(lf, s, bb, d0.f, d0.b, d0.dps, d1.f, d1.b, d1.dps, dps0, dA, dB));
  return lb > cur_t * (1.0 + kScreenMargin) ? T_SKIP : 0.0;
}

HPD void lb_stage_nb(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                     const double* hop, int i, int count, StageNb& n) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int cc = count + (k ? 1 : -1);
    StageDur d;
    d.f = d.b = d.dps = 0.0;
    int st = 0;
    if (cc >= 1) st = stage_setup(c, lf, lg, slots, hop, i, cc, d) ? 2 : 1;
    n.f[k] = d.f;
    n.b[k] = d.b;
    n.dps[k] = d.dps;
    n.st[k] = st;
  }
}

// nb_screen's path lower bound of neighbour slot q = 2 bb + odd with the
// changed stages' durations taken from the StageNb rows in r (same value for
// every slot). Returns T_INVALID / T_MEMORY for an infeasible neighbour,
// else the bound (>= 0).
HPD double nb_lb_rows(const Leaf& lf, const NbRows& r, int bb, int odd) {
  const int P = lf.P;
  const int k0 = odd ? 0 : 1;  // +1 moves a layer into stage bb, out of bb+1
  const int k1 = 1 - k0;
  const int st0 = r.st[0][k0], st1 = r.st[1][k1];
  if (st0 == 0 || st1 == 0) return T_INVALID;
  if (st0 == 1 || st1 == 1) return T_MEMORY;
  const double f0 = r.nf[0][k0], b0 = r.nbw[0][k0], p0 = r.nd[0][k0];
  const double f1 = r.nf[1][k1], b1 = r.nbw[1][k1], p1 = r.nd[1][k1];
  const double M = (double)lf.M;
  const double dps0 = bb == 0 ? p0 : r.dps0;
  double lb = dmax(r.PX + dps0, r.PY);
  const double A0 = r.A, B0 = r.Bt, sf0 = r.sf;
  lb = dmax(lb, A0 + M * (f0 + b0) + dmax(B0 + dps0, p0));
  const double A1 = A0 + f0 + sf0, B1 = B0 + sf0 + b0;
  lb = dmax(lb, A1 + M * (f1 + b1) + dmax(B1 + dps0, p1));
  const double dA = (f0 - r.f) + (f1 - r.f1);
  const double dB = (b0 - r.b) + (b1 - r.b1);
  if (bb + 2 < P) lb = dmax(lb, dmax(r.SX2 + dA + dB + dps0, r.SY2 + dA));
  lb = dmax(lb, pair_lb_rows(lf, r, bb, f0, b0, p0, f1, b1, p1, dps0, dA, dB));
  return dmax(lb, 0.0);
}

HPD double nb_lb_pre(const Leaf& lf, const StageLB* s, const StageNb* nbs, int q) {
  NbRows r;
  nb_rows_load(lf, s, nbs, q >> 1, r);
  return nb_lb_rows(lf, r, q >> 1, q & 1);
}

// Screen decision from nb_lb_pre: T_INVALID / T_MEMORY, T_SKIP when the
// bound is above cur_t (with the margin), else 0.0 (simulate).
HPD double screen_of(double lb, double cur_t) {
  if (lb < 0) return lb;
  return lb > cur_t * (1.0 + kScreenMargin) ? T_SKIP : 0.0;
}

HPD double nb_screen_pre(const Leaf& lf, const StageLB* s, const StageNb* nbs, int q, double cur_t) {
  return screen_of(nb_lb_pre(lf, s, nbs, q), cur_t);
}

// ------------------------------------------------------------ hill climb

// Per-leaf state of the steepest-descent search (planner.cpp:461-489) plus
// the leaf's best candidate and its memo-equivalent counts.
struct HillState {
  double cur_time;
  double best_time;
  long long simulated;
  long long pruned;
  int steps;        // accepted moves (== path length)
  int active;       // still climbing
  int has_best;
  int start;        // 0 none, 1 proportional, 2 uniform
};

// Move code of neighbour slot q: boundary b = q >> 1, d = +1 for even q,
// -1 for odd q (planner.cpp:473-474 order: i ascending, +1 before -1).
HPD int slot_of(int b, int d) { return 2 * b + (d > 0 ? 0 : 1); }

// Seeds evaluated: init counts, best and the start point
// (planner.cpp:434-468). t_uni/t_prop < 0 when memory-pruned.
HPD void hill_init(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                   const int* uni, const int* prop, double t_uni, double t_prop, int* cur,
                   int* best_split, HillState& hs, bool uniform_only) {
  const int P = lf.P;
  hs.simulated = 0;
  hs.pruned = 0;
  hs.steps = 0;
  hs.has_best = 0;
  hs.active = 0;
  hs.start = 0;
  hs.cur_time = 0.0;
  hs.best_time = 0.0;
  if (t_uni >= 0) {
    hs.simulated++;
    hs.has_best = 1;
    hs.best_time = t_uni;
    for (int i = 0; i < P; ++i) best_split[i] = uni[i];
  } else {
    hs.pruned++;
  }
  if (uniform_only) return;
  bool prop_new = !same_split(uni, prop, P);
  if (prop_new) {
    if (t_prop >= 0) {
      hs.simulated++;
      if (!hs.has_best || t_prop < hs.best_time ||
          (t_prop == hs.best_time && split_enc_less(P, prop, best_split))) {
        hs.has_best = 1;
        hs.best_time = t_prop;
        for (int i = 0; i < P; ++i) best_split[i] = prop[i];
      }
    } else {
      hs.pruned++;
    }
  }
  if (lf.mode != 0) return;  // exhaustive leaves enumerate everything instead
  if (t_prop >= 0) {
    hs.start = 1;
    hs.cur_time = t_prop;
    for (int i = 0; i < P; ++i) cur[i] = prop[i];
  } else if (t_uni >= 0) {
    hs.start = 2;
    hs.cur_time = t_uni;
    for (int i = 0; i < P; ++i) cur[i] = uni[i];
  }
  // a single stage has no neighbours: the loop body finds none and stops
  hs.active = hs.start != 0 && P > 1 && 4 * c.L > 0;
}

// Marks old[q] for neighbours of cur that the reference's memo already holds
// (planner.cpp:425-432): the seeds, path points and neighbourhoods of earlier
// path points. Along a strictly improving path a neighbour of c_k can only be
// within distance 1 of c_j (j < k) in prefix-sum space when
// ||S_k - S_j||_1 <= 2, found by scanning the move history backwards.
// delta: P ints scratch (zeroed on entry and exit).
HPD void mark_old(const Leaf& lf, const int* cur, const int* uni, const int* prop,
                  const short* hist, int steps, int* delta, unsigned char* old) {
  const int P = lf.P;
  const int nslots = 2 * (P - 1);
  for (int q = 0; q < nslots; ++q) old[q] = 0;
  // history scan: after applying moves t..k-1, delta = S_k - S_t
  int D = 0;
  for (int t = steps - 1; t >= 0; --t) {
    int code = hist[t];
    int b = code >> 1;
    int d = (code & 1) ? -1 : 1;
    int before = delta[b] < 0 ? -delta[b] : delta[b];
    delta[b] += d;
    int after = delta[b] < 0 ? -delta[b] : delta[b];
    D += after - before;
    if (D <= 2) {
      if (D == 0) {
        for (int q = 0; q < nslots; ++q) old[q] = 1;
      } else {
        for (int bb = 0; bb + 1 < P; ++bb) {
          if (delta[bb] == 0) continue;
          // moving boundary bb toward c_t: d' = -sign(delta)
          old[slot_of(bb, delta[bb] > 0 ? -1 : 1)] = 1;
        }
      }
    }
  }
  for (int t = 0; t < steps; ++t) delta[hist[t] >> 1] = 0;
  // seeds: a neighbour equal to uniform / proportional
  for (int s = 0; s < 2; ++s) {
    const int* ref = s == 0 ? uni : prop;
    int dist = 0, cb = -1, cd = 0;
    int sc = 0, sr = 0;
    for (int bb = 0; bb + 1 < P; ++bb) {
      sc += cur[bb];
      sr += ref[bb];
      int dd = sc - sr;
      if (dd != 0) {
        dist += dd < 0 ? -dd : dd;
        cb = bb;
        cd = dd;
      }
    }
    if (dist == 1) old[slot_of(cb, cd > 0 ? -1 : 1)] = 1;
  }
}

// One steepest-descent step of a leaf given its neighbours' times
// (planner.cpp:470-489). nb[q]: time, T_MEMORY or T_INVALID. Updates
// counts, the leaf best, the current point and the history.
HPD void hill_step(const Consts& c, const Leaf& lf, const LeafGroup* lg, const uint8_t* slots,
                   int* cur, const int* uni, const int* prop, int* best_split, short* hist,
                   HillState& hs, const double* nb, int* delta, unsigned char* old, int* tmp) {
  const int P = lf.P;
  const int nslots = 2 * (P - 1);
  mark_old(lf, cur, uni, prop, hist, hs.steps, delta, old);
  int bq = -1;
  double bt = 0.0;
  for (int q = 0; q < nslots; ++q) {
    double t = nb[q];
    if (t == T_INVALID) continue;
    if (!old[q]) {
      if (t >= 0) hs.simulated++;
      else hs.pruned++;
    }
    if (t < 0) continue;
    if (bq < 0 || t < bt) {
      bq = q;
      bt = t;
    }
    if (!old[q]) {
      bool better = !hs.has_best || t < hs.best_time;
      if (!better && t == hs.best_time) {
        int b = q >> 1, d = (q & 1) ? -1 : 1;
        for (int i = 0; i < P; ++i) tmp[i] = cur[i];
        tmp[b] += d;
        tmp[b + 1] -= d;
        better = split_enc_less(P, tmp, best_split);
      }
      if (better) {
        int b = q >> 1, d = (q & 1) ? -1 : 1;
        hs.has_best = 1;
        hs.best_time = t;
        for (int i = 0; i < P; ++i) best_split[i] = cur[i];
        best_split[b] += d;
        best_split[b + 1] -= d;
      }
    }
  }
  if (bq < 0 || !(bt < hs.cur_time)) {
    hs.active = 0;
    return;
  }
  int b = bq >> 1, d = (bq & 1) ? -1 : 1;
  cur[b] += d;
  cur[b + 1] -= d;
  hist[hs.steps] = (short)bq;
  hs.steps++;
  hs.cur_time = bt;
  if (hs.steps >= 4 * c.L) hs.active = 0;
}

}  // namespace hpc
