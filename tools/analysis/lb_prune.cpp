// Analysis (dev tool): how many hill-climb neighbours an admissible path
// lower bound would exclude from simulation. For each sampled C3 leaf the
// steepest descent runs on the CPU (hp_search_core.cuh); every non-memo,
// memory-feasible neighbour q with LB_q > cur_t * (1 + 1e-9) cannot be the
// step's improving move nor tie the leaf best, so its simulation could be
// skipped. Prints the fraction of simulated stage-ops (P*M weighted) saved.
#include <cstdio>
#include <cstring>
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

extern "C" int lb_analysis(const hp_problem* in, int sample_every, int max_pm) {
  hph::Problem p;
  if (!hph::load_problem(in, p).ok()) return 1;
  hph::enumerate(p);
  Consts c;
  hph::fill_consts(p, c);
  std::vector<double> hop = hph::hop_table(p);
  double work_all = 0, work_skip = 0, n_all = 0, n_skip = 0;
  double lb_gap_sum = 0; long gap_n = 0;
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
    auto eval = [&](const int* s, double* lbo) -> double {
      for (int i = 0; i < P; ++i) if (s[i] < 1) return T_INVALID;
      for (int i = 0; i < P; ++i) if (!stage_setup(c, lf, lg.data(), slots, hp, i, s[i], d[i])) return T_MEMORY;
      if (lbo) *lbo = lower_bound(c, lf, d.data());
      return simulate_serial(c.schedule == 0, P, lf.M, d.data(), st.data());
    };
    seed_splits(c, lf, lg.data(), slots, uni.data(), prop.data(), w.data(), frac.data(), order.data());
    HillState hs;
    double tu = eval(uni.data(), nullptr), tp = eval(prop.data(), nullptr);
    hill_init(c, lf, lg.data(), slots, uni.data(), prop.data(), tu, tp, cur.data(), bs.data(), hs, false);
    std::vector<double> lbs(2 * P);
    while (hs.active) {
      for (int q = 0; q < 2 * (P - 1); ++q) {
        int b = q >> 1, dd = (q & 1) ? -1 : 1;
        tmp = cur; tmp[b] += dd; tmp[b + 1] -= dd;
        lbs[q] = -1;
        nb[q] = eval(tmp.data(), &lbs[q]);
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
        lb_gap_sum += nb[q] / lbs[q]; gap_n++;
        if (lbs[q] > nb[q] * (1 + 1e-12)) { printf("INADMISSIBLE lb %.17g > t %.17g\n", lbs[q], nb[q]); return 2; }
      }
      std::fill(dl.begin(), dl.end(), 0);
      hill_step(c, lf, lg.data(), slots, cur.data(), uni.data(), prop.data(), bs.data(), hist.data(), hs,
                nb.data(), delta.data(), old.data(), tmp.data());
    }
  }
  printf("neighbours %.0f skip %.0f (%.1f%%), work skip %.1f%%, mean t/lb %.4f\n", n_all, n_skip,
         100 * n_skip / n_all, 100 * work_skip / work_all, lb_gap_sum / gap_n);
  return 0;
}
