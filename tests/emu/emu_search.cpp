#include <cstdlib>
#include <algorithm>
// TEST HARNESS ONLY — CPU emulation of the GPU search decomposition.
//
// Drives the exact per-candidate / per-leaf functions the sm_100a kernels run
// (paper_2405_16256_b200/csrc/hp_search_core.cuh) in plain loops on the host,
// so the algorithmic decomposition (level-synchronous simulator, on-device
// seed splits, memo-equivalent hill-climb counting, exact tie-break) can be
// checked against the reference oracle on CPU before it ever reaches a GPU.
// Never linked into the product library.
#include <cstring>
#include <vector>

#include "../../paper_2405_16256_b200/csrc/hp_host.hpp"
#include "../../paper_2405_16256_b200/csrc/hp_search_core.cuh"

using namespace hpc;

namespace {

long long g_screened = 0, g_neighbours = 0;  // nb_screen statistics (T_SKIP / all)
long long g_screen_mismatch = 0;              // nb_screen_pre != nb_screen (must stay 0)
long long g_bound_viol = 0;                   // nb_lb_pre above a simulated time (must stay 0)
int g_check_all = 0;                          // also simulate screened neighbours (emu_check_all)
long long g_checked = 0;                      // screened neighbours simulated for the check

struct LeafDev {
  Leaf lf;
  std::vector<LeafGroup> lg;
  const uint8_t* slots;
  const double* hop;
};

double eval(const Consts& c, const LeafDev& L, const int* split) {
  const int P = L.lf.P;
  std::vector<StageDur> d(P);
  std::vector<StageState> st(P);
  for (int i = 0; i < P; ++i) {
    if (split[i] < 1) return T_INVALID;
  }
  for (int i = 0; i < P; ++i)
    if (!stage_setup(c, L.lf, L.lg.data(), L.slots, L.hop, i, split[i], d[i])) return T_MEMORY;
  return simulate_serial(c.schedule == 0, P, L.lf.M, d.data(), st.data());
}

}  // namespace

extern "C" int emu_search_shard(const hp_problem* in, int shard, int count, hp_result* res) {
  hph::Problem p;
  hph::Status s = hph::load_problem(in, p);
  if (!s.ok()) return s.code;
  if (p.pruning) return HP_INTERNAL;  // emulation covers full mode
  hph::enumerate(p);
  Consts c;
  hph::fill_consts(p, c);
  const int G = c.n_groups;
  std::vector<double> hop(p.mbs.size() * p.links.size());
  for (size_t b = 0; b < p.mbs.size(); ++b)
    for (size_t l = 0; l < p.links.size(); ++l) hop[b * p.links.size() + l] = hph::hop_time(p, (int)l, p.mbs[b]);
  std::memset(res, 0, sizeof(*res));
  res->tasks = (long long)p.tasks.size();
  if (shard == 0)
  for (const hph::Task& t : p.tasks)
    if (t.no_link) { res->candidates_pruned++; res->reason_counts[HP_REASON_NO_LINK]++; }
    else if (t.leaf_begin == t.leaf_end) { res->candidates_pruned++; res->reason_counts[HP_REASON_NO_ASSIGNMENT]++; }

  bool have = false;
  double best_t = 0;
  LeafDev best_leaf;
  std::vector<int> best_split;
  int best_li = -1;
  for (int li : hph::shard_leaves(p, shard, count)) {
    const hph::LeafHost& h = p.leaves[li];
    const hph::Task& t = p.tasks[h.task];
    LeafDev L;
    L.lf = Leaf{h.task, t.pp, (int)h.M, h.dp, h.B, h.B_idx, t.layout_off, 0, 0,
                p.uniform_only ? 2 : (h.exhaustive ? 1 : 0), p.schedule};
    for (int g = 0; g < G; ++g)
      L.lg.push_back(hph::leaf_group(p, g, hph::leaf_tp(p, h, g), h.B, h.dp, hph::leaf_nodes(p, h, g)));
    L.slots = &p.layouts[t.layout_off];
    L.hop = &hop[h.B_idx * p.links.size()];
    const int P = t.pp;
    std::vector<int> uni(P), prop(P), cur(P), bs(P), order(P), delta(P, 0), tmp(P);
    std::vector<double> w(P), frac(P), nb(2 * P);
    std::vector<short> hist(4 * c.L + 1);
    std::vector<unsigned char> old(2 * P);
    HillState hs;
    seed_splits(c, L.lf, L.lg.data(), L.slots, uni.data(), prop.data(), w.data(), frac.data(), order.data());
    if (L.lf.mode == 1) {
      hs.simulated = hs.pruned = 0;
      hs.has_best = 0;
      std::vector<int> comp(P);
      unrank_composition(0, c.L, P, comp.data());
      do {
        double tt = eval(c, L, comp.data());
        if (tt >= 0) {
          hs.simulated++;
          if (!hs.has_best || tt < hs.best_time ||
              (tt == hs.best_time && split_enc_less(P, comp.data(), bs.data()))) {
            hs.has_best = 1; hs.best_time = tt; bs = comp;
          }
        } else hs.pruned++;
      } while (next_composition(comp.data(), P));
    } else {
      double tu = eval(c, L, uni.data());
      double tp = L.lf.mode == 2 ? -1 : eval(c, L, prop.data());
      hill_init(c, L.lf, L.lg.data(), L.slots, uni.data(), prop.data(), tu, tp, cur.data(), bs.data(),
                hs, L.lf.mode == 2);
      std::vector<StageLB> slb(P);
      std::vector<StageNb> snb(P);
      std::vector<double> lbv(2 * P);
      while (hs.active) {
        // the GPU's neighbour screen (nb_screen_pre over StageLB / StageNb
        // rows): only survivors are simulated
        for (int i = 0; i < P; ++i) {
          lb_stage(c, L.lf, L.lg.data(), L.slots, L.hop, i, cur[i], slb[i]);
          lb_stage_nb(c, L.lf, L.lg.data(), L.slots, L.hop, i, cur[i], snb[i]);
        }
        lb_scan(L.lf, slb.data());
        for (int q = 0; q < 2 * (P - 1); ++q) {
          const double lbq = nb_lb_pre(L.lf, slb.data(), snb.data(), q);
          if (getenv("EMU_DBG") && q < 4) {
            int b = q >> 1, d = (q & 1) ? -1 : 1;
            const int k0 = (q & 1) ? 0 : 1, k1 = 1 - k0;
            const double dA = (snb[b].f[k0] - slb[b].f) + (snb[b + 1].f[k1] - slb[b + 1].f);
            const double dB = (snb[b].b[k0] - slb[b].b) + (snb[b + 1].b[k1] - slb[b + 1].b);
            double pl = pair_lb_nb(L.lf, slb.data(), b, snb[b].f[k0], snb[b].b[k0], snb[b].dps[k0], snb[b + 1].f[k1],
                                   snb[b + 1].b[k1], snb[b + 1].dps[k1], b == 0 ? snb[0].dps[k0] : slb[0].dps, dA, dB);
            printf("q %d lb %.9g pair %.9g cur %.9g T0 %.9g PG %.3g SG %.3g sched %d\n", q, lbq, pl, hs.cur_time,
                   lb_total(L.lf, slb.data()), slb[b + 2 < P ? b + 2 : 0].SG, slb[0].SG, L.lf.sched);
            (void)d;
          }
          lbv[q] = lbq;
          double scr = screen_of(lbq, hs.cur_time);
          double ref = nb_screen(c, L.lf, L.lg.data(), L.slots, L.hop, cur.data(), slb.data(), q, hs.cur_time);
          if (!(scr == ref)) g_screen_mismatch++;
          g_neighbours++;
          if (scr == T_SKIP) g_screened++;
          if (scr == T_SKIP && g_check_all) {
            // admissibility of the screen itself: a screened neighbour's
            // simulated time must not be below its bound
            int b = q >> 1, d = (q & 1) ? -1 : 1;
            tmp = cur;
            tmp[b] += d; tmp[b + 1] -= d;
            const double t = eval(c, L, tmp.data());
            g_checked++;
            if (t >= 0 && lbq > t * (1.0 + 1e-9)) g_bound_viol++;
            if (t >= 0 && !(t > hs.cur_time)) g_bound_viol++;
          }
          if (scr != 0.0) {
            nb[q] = scr;
            continue;
          }
          int b = q >> 1, d = (q & 1) ? -1 : 1;
          tmp = cur;
          tmp[b] += d; tmp[b + 1] -= d;
          nb[q] = eval(c, L, tmp.data());
          // the bound must hold (up to the screen's rounding margin)
          if (nb[q] >= 0 && lbq > nb[q] * (1.0 + 1e-9)) g_bound_viol++;
        }
        hill_step(c, L.lf, L.lg.data(), L.slots, cur.data(), uni.data(), prop.data(), bs.data(),
                  hist.data(), hs, nb.data(), delta.data(), old.data(), tmp.data());
      }
    }
    res->candidates_simulated += hs.simulated;
    res->candidates_pruned += hs.pruned;
    res->reason_counts[HP_REASON_MEMORY] += hs.pruned;
    res->leaves++;
    if (hs.has_best && (!have || cand_less(c, hs.best_time, L.lf, L.lg.data(), L.slots, bs.data(), best_t,
                                           best_leaf.lf, best_leaf.lg.data(), best_leaf.slots, best_split.data()))) {
      have = true; best_t = hs.best_time; best_leaf = L; best_split = bs; best_li = li;
    }
  }
  if (!have) return count > 1 ? HP_OK : HP_INFEASIBLE;
  res->has_best = 1;
  res->best_time_s = best_t;
  res->best_pp = best_leaf.lf.P;
  hph::make_plan(p, p.leaves[best_li], best_split.data(), res->best_plan);
  return HP_OK;
}

extern "C" int emu_search(const hp_problem* in, hp_result* res) { return emu_search_shard(in, 0, 1, res); }

extern "C" void emu_screen_stats(long long* screened, long long* neighbours, int reset) {
  *screened = g_screened;
  *neighbours = g_neighbours;
  if (reset) g_screened = g_neighbours = 0;
}

extern "C" long long emu_screen_mismatches() { return g_screen_mismatch; }
extern "C" long long emu_bound_violations() { return g_bound_viol; }
extern "C" long long emu_check_all(int on) { g_check_all = on; return g_checked; }

// Explicit-plan evaluation through the same per-stage setup + serial
// level-synchronous simulation (mode 3 pseudo-leaf, like hp_evaluate_plans).
extern "C" int emu_evaluate(const hp_problem* in, const hp_plan* plan, double* out) {
  hph::Problem p;
  hph::Status s = hph::load_problem(in, p);
  if (!s.ok()) return s.code;
  Consts c;
  hph::fill_consts(p, c);
  const int P = plan->n_stages;
  int64_t B = plan->micro_batch_size > 0 ? plan->micro_batch_size : p.train.micro_batch_size;
  Leaf lf{-1, P, (int)plan->micro_batches_per_dp_replica, plan->stages[0].dp_degree, B, 0, 0, 0, 0, 3, 0};
  std::vector<LeafGroup> lg;
  std::vector<uint8_t> slots;
  std::vector<double> hop(p.links.size());
  for (size_t l = 0; l < p.links.size(); ++l) hop[l] = hph::hop_time(p, (int)l, B);
  for (int i = 0; i < P; ++i) {
    const hp_stage& st = plan->stages[i];
    lg.push_back(hph::leaf_group(p, st.group, st.tp_degree, B, st.dp_degree, st.nodes_used));
    slots.push_back((uint8_t)i);
  }
  std::vector<StageDur> d(P);
  std::vector<StageState> ss(P);
  for (int i = 0; i < P; ++i)
    stage_setup(c, lf, lg.data(), slots.data(), hop.data(), i,
                plan->stages[i].layer_end - plan->stages[i].layer_begin, d[i]);
  *out = simulate_serial(c.schedule == 0 || plan->schedule == HP_GPIPE, P, lf.M, d.data(), ss.data());
  return 0;
}

// Bounded-composition machinery of the exhaustive regime: enumerates every
// composition of L into P parts in lexicographic order (enumerate_splits,
// planner.cpp:149-162), keeps those with count_i <= caps[i], and checks that
// exh_table / unrank_bounded / next_bounded reproduce exactly that sequence.
// Returns the number of bounded compositions, or -1 on a mismatch.
extern "C" long long emu_check_bounded(int L, int P, const int* caps) {
  std::vector<long long> tbl((size_t)(P + 1) * (L + 1));
  long long F = exh_table(L, P, caps, tbl.data());
  std::vector<int> sufcap(P + 1, 0);
  for (int j = P - 1; j >= 0; --j) sufcap[j] = sufcap[j + 1] + caps[j];
  std::vector<int> comp(P), want(P), got(P);
  long long n = 0;
  bool have_iter = false;
  unrank_composition(0, L, P, comp.data());
  do {
    bool ok = true;
    for (int i = 0; i < P; ++i) ok = ok && comp[i] <= caps[i];
    if (!ok) continue;
    unrank_bounded(n, L, P, caps, tbl.data(), got.data());
    if (got != comp) return -1;
    if (!have_iter) {
      want = comp;
      have_iter = true;
    } else {
      if (!next_bounded(want.data(), P, caps, sufcap.data())) return -1;
      if (want != comp) return -1;
    }
    ++n;
  } while (next_composition(comp.data(), P));
  if (have_iter && next_bounded(want.data(), P, caps, sufcap.data())) return -1;
  return n == F ? n : -1;
}

// split_layers (hp_core.cuh) on positive weights with total >= parts.
extern "C" void emu_split_layers(int total, const double* w, int parts, int* out) {
  std::vector<double> frac(parts);
  std::vector<int> order(parts);
  split_layers(total, w, parts, out, frac.data(), order.data());
}
