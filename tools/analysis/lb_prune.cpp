// Analysis (dev tool): how many hill-climb neighbours an admissible path
// lower bound would exclude from simulation. For each sampled C3 leaf the
// steepest descent runs on the CPU (hp_search_core.cuh); every non-memo,
// memory-feasible neighbour q with LB_q > cur_t * (1 + 1e-9) cannot be the
// step's improving move nor tie the leaf best, so its simulation could be
// skipped. Prints the fraction of simulated stage-ops (P*M weighted) saved.
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "../../paper_2405_16256_b200/csrc/hp_host.hpp"
#include "../../paper_2405_16256_b200/csrc/hp_search_core.cuh"

using namespace hpc;

static double lower_bound(const Consts& c, const Leaf& lf, const StageDur* d) {
  const int P = lf.P;
  double A = 0.0, Bt = 0.0, lb = 0.0;
  for (int k = 0; k < P; ++k) {
    double core = A + (double)lf.M * (d[k].f + d[k].b);
    double tail = Bt + d[0].dps;
    double v = core + (tail > d[k].dps ? tail : d[k].dps);
    if (v > lb) lb = v;
    A += d[k].f + d[k].sf;
    if (k + 1 < P) Bt += d[k + 1].sb + d[k].b;
  }
  return lb;
}

// Round-trip bound (1F1B and GPipe): B(k,0) cannot start before microbatch 0
// went forward through every stage and back to k (R_k); after it stage k
// still runs M backwards and the forwards it has not issued yet, then the
// backward chain to stage 0 (or its own DP sync).
static double lower_bound_rt(const Consts& c, const Leaf& lf, const StageDur* d, bool gpipe) {
  const int P = lf.P;
  const double M = (double)lf.M;
  double fall = 0.0;  // sum_j f_j + sf_j (j < P-1) + f_{P-1}
  for (int k = 0; k < P; ++k) fall += d[k].f + (k + 1 < P ? d[k].sf : 0.0);
  std::vector<double> suf(P + 1, 0.0);  // sum_{j>k} (b_j + sb_j)
  for (int k = P - 1; k >= 0; --k) suf[k] = (k + 1 < P ? suf[k + 1] + d[k + 1].b + d[k + 1].sb : 0.0);
  double Bt = 0.0, lb = 0.0;
  for (int k = 0; k < P; ++k) {
    const double R = fall + suf[k];
    const double w = gpipe ? M : std::min((double)(P - k), M);
    const double core = R + M * d[k].b + (M - w) * d[k].f;
    const double tail = Bt + d[0].dps;
    const double v = core + (tail > d[k].dps ? tail : d[k].dps);
    if (v > lb) lb = v;
    if (k + 1 < P) Bt += d[k + 1].sb + d[k].b;
  }
  return lb;
}

// Cycle bound (1F1B): on stage k, F(k, m+w) follows B(k, m) (w = P-k
// in-flight), and B(k, m+w) needs microbatch m+w's round trip through the
// downstream stages: the circuit length C_k = sum_{j>=k} (f_j + b_j) + the
// sends between them. So B(k, n w) ends >= R_k + b_k + n C_k.
static double lower_bound_cyc(const Consts& c, const Leaf& lf, const StageDur* d) {
  const int P = lf.P;
  const long long M = lf.M;
  double fall = 0.0;
  for (int k = 0; k < P; ++k) fall += d[k].f + (k + 1 < P ? d[k].sf : 0.0);
  std::vector<double> suf(P + 1, 0.0), cyc(P + 1, 0.0);
  for (int k = P - 1; k >= 0; --k) {
    suf[k] = (k + 1 < P ? suf[k + 1] + d[k + 1].b + d[k + 1].sb : 0.0);
    cyc[k] = d[k].f + d[k].b + (k + 1 < P ? cyc[k + 1] + d[k].sf + d[k + 1].sb : 0.0);
  }
  double Bt = 0.0, lb = 0.0;
  for (int k = 0; k < P; ++k) {
    const long long w = std::min((long long)(P - k), M);
    const long long n = (M - 1) / w;
    const double R = fall + suf[k];
    const double core = R + d[k].b + (double)n * cyc[k] + (double)(M - 1 - n * w) * d[k].b;
    const double tail = Bt + d[0].dps;
    const double v = core + (tail > d[k].dps ? tail : d[k].dps);
    if (v > lb) lb = v;
    if (k + 1 < P) Bt += d[k + 1].sb + d[k].b;
  }
  return lb;
}

// Window-cycle bound (1F1B): for stages k..k+j, B(k+j, m) -> B(k, m) ->
// F(k, m + w_k) -> F(k+j, m + w_k) -> B(k+j, m + j + 1) is a circuit of
// length C = sum_{i=k}^{k+j} (f_i + b_i) + the sends between them, taken
// once per j+1 microbatches (w_k = w_{k+j} + j while M >= P - k).
static int g_J = 1;
static long g_rank[9], g_prank[9];
static double lower_bound_win(const Consts& c, const Leaf& lf, const StageDur* d) {
  const int P = lf.P;
  const long long M = lf.M;
  double fall = 0.0;
  for (int k = 0; k < P; ++k) fall += d[k].f + (k + 1 < P ? d[k].sf : 0.0);
  std::vector<double> suf(P + 1, 0.0), Bt(P, 0.0);
  for (int k = P - 1; k >= 0; --k) suf[k] = (k + 1 < P ? suf[k + 1] + d[k + 1].b + d[k + 1].sb : 0.0);
  for (int k = 1; k < P; ++k) Bt[k] = Bt[k - 1] + d[k].sb + d[k - 1].b;
  double lb = 0.0;
  for (int k = 0; k < P; ++k) {
    double cyc = d[k].f + d[k].b;
    for (int j = 1; j <= g_J && k + j < P; ++j) {
      const int e = k + j;
      cyc += d[e].f + d[e].b + d[e - 1].sf + d[e].sb;
      const long long wk = std::min((long long)(P - k), M);
      if (wk != std::min((long long)(P - e), M) + j) continue;
      const long long n = (M - 1 >= wk) ? (M - 1 - wk) / (j + 1) + 1 : 0;
      const double core = fall + suf[e] + d[e].b + (double)n * cyc + (double)(M - 1 - n * (j + 1)) * d[e].b;
      const double tail = Bt[e] + d[0].dps;
      const double v = core + (tail > d[e].dps ? tail : d[e].dps);
      if (v > lb) lb = v;
    }
  }
  return lb;
}

extern "C" int lb_analysis(const hp_problem* in, int sample_every, int max_pm) {
  hph::Problem p;
  if (!hph::load_problem(in, p).ok()) return 1;
  hph::enumerate(p);
  Consts c;
  hph::fill_consts(p, c);
  std::vector<double> hop = hph::hop_table(p);
  double work_all = 0, work_skip = 0, n_all = 0, n_skip = 0;
  double lb_gap_sum = 0; long gap_n = 0;
  static int surv_dumped = 0;
  double work_skip2 = 0, n_skip2 = 0, work_worse = 0, n_worse = 0;
  printf("leaves %zu\n", p.leaves.size());
  if (getenv("LBP_J")) g_J = atoi(getenv("LBP_J"));
  for (size_t li = 0; li < p.leaves.size(); li += sample_every) {
    Leaf lf = hph::device_leaf(p, (int)li);
    if (lf.mode != 0) continue;
    if ((long)lf.P * lf.M > max_pm) continue;
    std::vector<LeafGroup> lg(p.groups.size());
    hph::leaf_rows(p, (int)li, lg.data());
    const uint8_t* slots = &p.layouts[lf.layout_off];
    const double* hp = &hop[lf.B_idx * p.links.size()];
    const int P = lf.P;
    std::vector<int> uni(P), prop(P), cur(P), bs(P), order(P), delta(P, 0), tmp(P);
    std::vector<double> w(P), frac(P), nb(2 * P);
    std::vector<short> hist(4 * c.L + 1);
    std::vector<unsigned char> old(2 * P);
    std::vector<StageDur> d(P);
    std::vector<StageState> st(P);
    std::vector<double> lbs2(2 * P);
    double* lb2o = nullptr;
    auto eval = [&](const int* s, double* lbo) -> double {
      for (int i = 0; i < P; ++i) if (s[i] < 1) return T_INVALID;
      for (int i = 0; i < P; ++i) if (!stage_setup(c, lf, lg.data(), slots, hp, i, s[i], d[i])) return T_MEMORY;
      if (lbo) *lbo = lower_bound(c, lf, d.data());
      if (lb2o) *lb2o = std::max(*lbo, c.schedule == 0 ? lower_bound_rt(c, lf, d.data(), true)
                                                         : lower_bound_win(c, lf, d.data()));
      return simulate_serial(c.schedule == 0, P, lf.M, d.data(), st.data());
    };
    seed_splits(c, lf, lg.data(), slots, uni.data(), prop.data(), w.data(), frac.data(), order.data());
    HillState hs;
    double tu = eval(uni.data(), nullptr), tp = eval(prop.data(), nullptr);
    hill_init(c, lf, lg.data(), slots, uni.data(), prop.data(), tu, tp, cur.data(), bs.data(), hs, false);
    std::vector<double> lbs(2 * P);
    std::vector<double> prev_t;
    int prev_move = -1;
    static int dumped = 0;
    if (getenv("LBP_STAGES") && hs.active && lf.M >= 1000 && !dumped++) {
      eval(cur.data(), nullptr);
      FILE* fo = fopen(getenv("LBP_STAGES"), "w");
      fprintf(fo, "%d %lld %.17g\n", P, (long long)lf.M, hs.cur_time);
      for (int i = 0; i < P; ++i) fprintf(fo, "%.17g %.17g %.17g %.17g %.17g\n", d[i].f, d[i].b, d[i].sf, d[i].sb, d[i].dps);
      fclose(fo);
    }
    while (hs.active) {
      for (int q = 0; q < 2 * (P - 1); ++q) {
        int b = q >> 1, dd = (q & 1) ? -1 : 1;
        tmp = cur; tmp[b] += dd; tmp[b + 1] -= dd;
        lbs[q] = -1;
        lbs2[q] = -1;
        lb2o = &lbs2[q];
        nb[q] = eval(tmp.data(), &lbs[q]);
        lb2o = nullptr;
      }
      // old marks as the step will compute them
      std::vector<int> dl(P, 0);
      mark_old(lf, cur.data(), uni.data(), prop.data(), hist.data(), hs.steps, dl.data(), old.data());
      const double ct = hs.cur_time;
      for (int q = 0; q < 2 * (P - 1); ++q) {
        if (nb[q] < 0 || old[q]) continue;
        double wk = (double)P * lf.M;
        work_all += wk; n_all += 1;
        if (lbs[q] > ct * (1 + 1e-9)) { work_skip += wk; n_skip += 1; }
        if (lbs2[q] > ct * (1 + 1e-9)) { work_skip2 += wk; n_skip2 += 1; }
        if (nb[q] > ct * (1 + 1e-9)) { work_worse += wk; n_worse += 1; }
        if (getenv("LBP_SURV") && nb[q] > ct * (1 + 1e-9) && !(lbs2[q] > ct * (1 + 1e-9)) &&
            (nb[q] - lbs2[q]) / nb[q] > 0.015 && !surv_dumped++) {
          tmp = cur; tmp[q >> 1] += (q & 1) ? -1 : 1; tmp[(q >> 1) + 1] -= (q & 1) ? -1 : 1;
          eval(tmp.data(), nullptr);
          FILE* fo = fopen(getenv("LBP_SURV"), "w");
          fprintf(fo, "%d %lld %.17g %.17g %.17g\n", P, (long long)lf.M, ct, nb[q], lbs2[q]);
          for (int i = 0; i < P; ++i) fprintf(fo, "%.17g %.17g %.17g %.17g %.17g\n", d[i].f, d[i].b, d[i].sf, d[i].sb, d[i].dps);
          fclose(fo);
        }
        if (getenv("LBP_DUMP") && nb[q] > ct * (1 + 1e-9) && !(lbs2[q] > ct * (1 + 1e-9)))
          printf("W q=%d bb=%d P=%d M=%lld worse %.3e gap %.3e\n", q, q >> 1, P, (long long)lf.M, (nb[q] - ct) / ct, (nb[q] - lbs2[q]) / nb[q]);
        if (lbs2[q] > nb[q] * (1 + 1e-12)) { printf("INADMISSIBLE rt lb %.17g > t %.17g\n", lbs2[q], nb[q]); return 2; }
        lb_gap_sum += nb[q] / lbs[q]; gap_n++;
        if (lbs[q] > nb[q] * (1 + 1e-12)) { printf("INADMISSIBLE lb %.17g > t %.17g\n", lbs[q], nb[q]); return 2; }
      }
      {
        // move prediction: rank of the steepest move among the neighbours by bound
        int bq = -1;
        for (int q = 0; q < 2 * (P - 1); ++q)
          if (nb[q] >= 0 && (bq < 0 || nb[q] < nb[bq])) bq = q;
        if (bq >= 0 && nb[bq] < ct) {
          // rank of this move among the previous step's neighbours by time
          if (!prev_t.empty()) {
            int pr = 0;
            const double tm = prev_t[bq];
            if (tm < 0) pr = 8;
            else for (int q = 0; q < 2 * (P - 1); ++q)
              if (q != prev_move && prev_t[q] >= 0 && q != bq && (prev_t[q] < tm || (prev_t[q] == tm && q < bq))) pr++;
            g_prank[pr < 8 ? pr : 8]++;
          }
          if (getenv("LBP_MOVES") && li == 0 + atoi(getenv("LBP_MOVES"))) printf("M %d %.3e %.3e\n", bq, (ct - nb[bq]) / ct, prev_t.empty() ? 0.0 : prev_t[bq]);
          prev_t.assign(nb.begin(), nb.begin() + 2 * (P - 1));
          prev_move = bq;
          int rank = 0;
          for (int q = 0; q < 2 * (P - 1); ++q)
            if (nb[q] >= 0 && q != bq && (lbs2[q] < lbs2[bq] || (lbs2[q] == lbs2[bq] && q < bq))) rank++;
          g_rank[rank < 7 ? rank : 7]++;
        } else {
          g_rank[8]++;
        }
      }
      std::fill(dl.begin(), dl.end(), 0);
      hill_step(c, lf, lg.data(), slots, cur.data(), uni.data(), prop.data(), bs.data(), hist.data(), hs,
                nb.data(), delta.data(), old.data(), tmp.data());
    }
  }
  printf("neighbours %.0f skip %.0f (%.1f%%), work skip %.1f%%, mean t/lb %.4f\n", n_all, n_skip,
         100 * n_skip / n_all, 100 * work_skip / work_all, lb_gap_sum / gap_n);
  printf("move rank among the previous step's neighbours by time (0..7, >=8):");
  for (int r = 0; r < 9; ++r) printf(" %ld", g_prank[r]);
  printf("\n");
  printf("move rank by bound (0..6, >=7, no move):");
  for (int r = 0; r < 9; ++r) printf(" %ld", g_rank[r]);
  printf("\n");
  printf("round-trip bound: skip %.0f (%.1f%%), work skip %.1f%%; strictly worse (ceiling) %.0f (%.1f%%), work %.1f%%\n",
         n_skip2, 100 * n_skip2 / n_all, 100 * work_skip2 / work_all, n_worse, 100 * n_worse / n_all,
         100 * work_worse / work_all);
  return 0;
}
