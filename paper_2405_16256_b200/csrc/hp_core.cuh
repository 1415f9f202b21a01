// hp_core.cuh — per-candidate arithmetic shared by the sm_100a kernels.
//
// Everything here is __host__ __device__ so tests/emu can drive the exact
// device code paths on the CPU (test harness only; the product never runs
// these on the host). The arithmetic restates the reference cost model and
// simulator in the reference's association order; the library is compiled
// with --fmad=false so no a*b+c is contracted (SURVEY.md finding 3), making
// every double bit-identical to the x86 reference build.
#pragma once

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define HPD __host__ __device__ __forceinline__
#else
#define HPD inline
#endif

// Load of per-leaf search state another SM may have written during the
// same kernel (the hill climb's steps move between SMs): past L1 on the
// device, a plain load in the CPU emulation.
#if defined(__CUDA_ARCH__)
#define HP_LDX(p) __ldcg(p)
#else
#define HP_LDX(p) (*(p))
#endif

namespace hpc {

constexpr int MAXG = 16;     // device groups (HP_MAX_GROUPS)

// Problem-wide constants (one per search), __constant__ on the device.
struct Consts {
  int L;            // model.num_layers
  int n_groups;
  int schedule;     // HP_GPIPE = 0, HP_1F1B = 1
  int pruning;      // planner.time_bound_pruning
  double H;         // (double)hidden_size
  double seq;       // (double)seq_length
  double bytes;     // (double)bytes_per_element
  double act;       // activation_bytes_per_token_per_hidden
  double edge;      // edge_layer_cost_multiplier
  double osm;       // optimizer_state_multiplier
  double budget[MAXG];   // memory_bytes * memory_headroom   (planner.cpp:508)
  int link_inter[MAXG];  // index into hop table rows: inter-node link of group g
  int link_pair[MAXG][MAXG];  // inter-group link of (g, h), -1 if none
  int n_links;
  int n_B;               // micro-batch candidates
  // group names for encode_plan (tie-break): names + name_off[g], name_len[g]
  // bytes; `names` points at a device copy on the GPU (the caller sets it)
  const char* names;
  int name_off[MAXG];
  int name_len[MAXG];
};

// Split-independent per-(leaf, group) terms, computed on the host in the
// reference's exact order (layer_cost, cost_model.cpp:88-107; DP all-reduce
// constants of collective_time, cost_model.cpp:63-73).
struct LeafGroup {
  double fl;       // LayerCost.fwd_s
  double bl;       // LayerCost.bwd_s
  double pbytes;   // LayerCost.param_bytes
  double ar_lat;   // steps * latency_s of the DP link (dp > 1)
  double ar_mf;    // factor * (ranks - 1) / (double)ranks
  double ar_den;   // bandwidth_bits_per_s * efficiency of the DP link
  double weight;   // peak_tflops * compute_efficiency * tp  (stage_weights, planner.cpp:94)
  int tp;
  int nodes;
  int group;
  int dp;          // StageAssignment.dp_degree
};

// One leaf of the search tree: (task, dp, B, per-group tp), planner.cpp:353-391.
struct Leaf {
  int task;
  int P;
  int M;            // micro_batches_per_dp_replica (<= 5e6, sim.cpp:68)
  int dp;
  long long B;
  int B_idx;
  int layout_off;   // stage -> group bytes of the task
  int split_off;    // offset of this leaf's P-int rows in per-leaf split buffers
  int lg_off;       // offset of this leaf's LeafGroup rows (n_groups each)
  int mode;         // 0 hill climb, 1 exhaustive, 2 uniform only, 3 explicit plan
  int sched;        // hp_schedule of this leaf's candidates (explicit plans carry their own)
};

// ---------------------------------------------------------------- helpers

HPD double dmax(double a, double b) { return a < b ? b : a; }   // std::max

// stage_memory, cost_model.cpp:75-86 (layers = count > 0 always here).
HPD double stage_memory(const Consts& c, int count, int tp, double B, int in_flight) {
  const double layers = count;
  double weight_bytes = layers * 12.0 * c.H * c.H * c.bytes;
  double param_state = weight_bytes / tp * c.osm;
  double act_per_mb = layers * B * c.seq * c.H * c.act;
  return param_state + in_flight * act_per_mb / tp;
}

// one_f_one_b_in_flight, sim.hpp:81-84
HPD int in_flight(const Consts& c, int stage, int P, int M) {
  if (c.schedule == 0) return M;
  int bound = P - stage;
  return bound < M ? bound : M;
}

// Per-candidate, per-stage durations (plan_stage_times, evaluate.cpp:23-76).
struct StageDur {
  double f, b, sf, sb, dps;
};

// fwd/bwd of stage i with `count` layers, edge multipliers added first
// (evaluate.cpp:42-48).
HPD void stage_compute(const Consts& c, const LeafGroup& g, int i, int P, int count, StageDur& d) {
  double layers = count;
  if (i == 0) layers += c.edge;          // layer_range.begin == 0
  if (i == P - 1) layers += c.edge;      // layer_range.end == num_layers
  d.f = layers * g.fl;
  d.b = layers * g.bl;
}

// DP gradient sync of a stage, evaluate.cpp:65-73 + collective_time.
HPD double dp_sync(const LeafGroup& g, int count) {
  if (g.dp <= 1) return 0.0;
  double grad = (double)count * g.pbytes / g.tp;
  double moved = g.ar_mf * grad;
  return g.ar_lat + moved * 8.0 / g.ar_den;
}

// ---------------------------------------------------------------- simulator
//
// Level-synchronous evaluation of the 1F1B / GPipe max-plus DAG of
// simulate() (sim.cpp:63-195). At level t every stage runs its next op if
// the op it depends on ran at a level < t (the unit-time ASAP schedule).
// Each node value is max(predecessors) + duration and max is exact, so any
// topological order yields the reference's doubles bit for bit. Stage i
// only needs its neighbours' previous-level channel state: within this
// schedule the producer of sendF(i-1,m) has issued exactly m+1 forwards when
// F(i,m) runs (single-slot property, checked exhaustively in tests), so the
// channel's last end time IS the operand.
struct StageState {
  double free_t;  // stage_free[i]
  double chf;     // chan_fwd_free[i] == last sendF end
  double chb;     // chan_bwd_free[i] == last sendB end
  int nf, nb;     // forwards / backwards issued
};

HPD void stage_init(StageState& s) {
  s.free_t = 0.0;
  s.chf = 0.0;
  s.chb = 0.0;
  s.nf = 0;
  s.nb = 0;
}

HPD bool stage_done(const StageState& s, int M) { return s.nf >= M && s.nb >= M; }

// One level for stage i. lchf/lnf: stage i-1 snapshot; rchb/rnb: stage i+1
// snapshot (ignored at the pipeline ends). w = one_f_one_b_in_flight.
HPD void stage_level(bool gpipe, int i, int P, int M, int w, const StageDur& d, StageState& s,
                     double lchf, int lnf, double rchb, int rnb, double& max_end) {
  bool want_f;
  if (gpipe) {
    // stage_ops GPipe: all forwards, then all backwards (sim.cpp:46-50)
    if (s.nf < M) want_f = true;
    else if (s.nb < M) want_f = false;
    else return;
  } else {
    // stage_ops 1F1B: w warm-up F, then B/F alternation, trailing B (sim.cpp:51-58)
    if (s.nf < w || (s.nf < M && s.nb > s.nf - w)) want_f = true;
    else if (s.nb < M) want_f = false;
    else return;
  }
  if (want_f) {
    if (i > 0 && !(lnf > s.nf)) return;             // ready(), sim.cpp:102
    double ready = i > 0 ? lchf : 0.0;
    double start = dmax(s.free_t, ready);           // sim.cpp:116
    double end = start + d.f;
    s.free_t = end;
    max_end = dmax(max_end, end);
    if (i < P - 1) {                                // sim.cpp:125-134
      double st = dmax(end, s.chf);
      double e = st + d.sf;
      s.chf = e;
      max_end = dmax(max_end, e);
    }
    s.nf++;
  } else {
    if (i < P - 1 && !(rnb > s.nb)) return;         // ready(), sim.cpp:103
    double ready = i < P - 1 ? rchb : 0.0;
    double start = dmax(s.free_t, ready);
    double end = start + d.b;
    s.free_t = end;
    max_end = dmax(max_end, end);
    if (i > 0) {                                    // sim.cpp:135-145
      double st = dmax(end, s.chb);
      double e = st + d.sb;
      s.chb = e;
      max_end = dmax(max_end, e);
    }
    s.nb++;
  }
}

// ---------------------------------------------------------------- splits

// split_layers, planner.cpp:42-84 (weights already validated positive).
// frac/order are caller scratch of `parts` entries.
HPD void split_layers(int total, const double* w, int parts, int* counts, double* frac,
                      int* order) {
  double weight_sum = 0.0;
  for (int i = 0; i < parts; ++i) weight_sum += w[i];
  int assigned = 0;
  for (int i = 0; i < parts; ++i) {
    double quota = total * w[i] / weight_sum;
    double fl = floor(quota);
    counts[i] = (int)fl;
    frac[i] = quota - counts[i];
    assigned += counts[i];
  }
  int remainder = total - assigned;
  // std::stable_sort by fraction descending. Stages of one device group
  // (and tp) share a weight, so the fractions take few distinct values:
  // emit the indices of each distinct value, largest first, in index order
  // (O(parts x distinct)); many distinct values fall back to a stable
  // insertion sort. Both give exactly std::stable_sort's order.
  constexpr int kDistinct = 16;
  double dv[kDistinct];
  int nd = 0;
  for (int i = 0; i < parts && nd <= kDistinct; ++i) {
    int k = 0;
    while (k < nd && !(dv[k] == frac[i])) ++k;
    if (k == nd) {
      if (nd == kDistinct) {
        nd = kDistinct + 1;
        break;
      }
      dv[nd++] = frac[i];
    }
  }
  if (nd <= kDistinct) {
    for (int a = 1; a < nd; ++a) {  // distinct values, descending
      const double x = dv[a];
      int k = a;
      while (k > 0 && dv[k - 1] < x) {
        dv[k] = dv[k - 1];
        --k;
      }
      dv[k] = x;
    }
    int o = 0;
    for (int k = 0; k < nd; ++k)
      for (int i = 0; i < parts; ++i)
        if (frac[i] == dv[k]) order[o++] = i;
  } else {
    for (int i = 0; i < parts; ++i) {
      int j = i;
      while (j > 0 && frac[order[j - 1]] < frac[i]) {
        order[j] = order[j - 1];
        --j;
      }
      order[j] = i;
    }
  }
  for (int r = 0; r < remainder; ++r) ++counts[order[r % parts]];
  for (int i = 0; i < parts; ++i) {
    while (counts[i] == 0) {
      int donor = 0;
      for (int j = 1; j < parts; ++j)
        if (counts[j] > counts[donor]) donor = j;
      --counts[donor];
      ++counts[i];
    }
  }
}

// contiguous_split_count, planner.cpp:134-147
HPD long long contiguous_split_count(int layers, int parts) {
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

// Binomial without saturation for unranking (values here are <= limit).
HPD long long binom(int n, int k) {
  if (k < 0 || n < 0 || k > n) return 0;
  if (k > n - k) k = n - k;
  long long c = 1;
  for (int i = 1; i <= k; ++i) c = c * (n - k + i) / i;
  return c;
}

// Composition of `total` into `parts` positive parts with lexicographic rank
// `rank` (enumerate_splits order, planner.cpp:149-162: first part ascending).
HPD void unrank_composition(long long rank, int total, int parts, int* out) {
  int rem = total;
  for (int j = 0; j < parts - 1; ++j) {
    int left = parts - j;  // parts still to fill including this one
    for (int v = 1;; ++v) {
      long long cnt = binom(rem - v - 1, left - 2);
      if (rank < cnt) {
        out[j] = v;
        rem -= v;
        break;
      }
      rank -= cnt;
    }
  }
  out[parts - 1] = rem;
}

// Next composition in the same order; returns false after the last one.
HPD bool next_composition(int* c, int parts) {
  // The last part absorbs the remainder. Find the rightmost j < parts-1 that
  // can grow (c[parts-1] > 1): increment c[j], reset later parts to 1 and put
  // the rest in the last part.
  if (parts < 2) return false;
  int tail = c[parts - 1];
  int j = parts - 2;
  // accumulate the suffix sum as we move left
  int suffix = tail;
  while (j >= 0) {
    // parts j+1..parts-1 currently sum to `suffix`; they need at least parts-1-j
    if (suffix > parts - 1 - j) {
      c[j] += 1;
      int rest = suffix - 1;
      for (int k = j + 1; k < parts - 1; ++k) {
        c[k] = 1;
        rest -= 1;
      }
      c[parts - 1] = rest;
      return true;
    }
    suffix += c[j];
    --j;
  }
  return false;
}

// ---------------------------------------------------------------- ordering
//
// encode_plan (planner.cpp:192-200) as a lazy character stream, so the exact
// better_than tie-break (planner.cpp:178-183) can run without materialising
// strings: "1f1b|M|B" then per stage "|name:begin-end:nodes:tp:dp".
struct EncStream {
  const Consts* c;
  const uint8_t* slots;   // stage -> LeafGroup row
  const LeafGroup* lg;    // rows of this leaf
  const int* counts;      // layer counts, P entries
  int P;
  long long M, B;
  int dp;
  // cursor
  int field;           // 0 sched,1 '|',2 M,3 '|',4 B, then per stage 11 fields
  int stage;
  int pos;
  int begin;           // running layer begin
  char num[24];
  int numlen;
};

HPD int fmt_ll(long long v, char* buf) {
  char tmp[24];
  int n = 0;
  bool neg = v < 0;
  unsigned long long u = neg ? (unsigned long long)(-(v + 1)) + 1 : (unsigned long long)v;
  do {
    tmp[n++] = (char)('0' + (u % 10));
    u /= 10;
  } while (u);
  int k = 0;
  if (neg) buf[k++] = '-';
  while (n) buf[k++] = tmp[--n];
  return k;
}

HPD void enc_init(EncStream& e) {
  e.field = 0;
  e.stage = 0;
  e.pos = 0;
  e.begin = 0;
  e.numlen = -1;
}

// Returns the next byte (0..255) or -1 at the end.
HPD int enc_next(EncStream& e) {
  for (;;) {
    if (e.field == 0) {
      const char* s = e.c->schedule == 0 ? "gpipe" : "1f1b";
      int n = e.c->schedule == 0 ? 5 : 4;
      if (e.pos < n) return (unsigned char)s[e.pos++];
      e.field = 1; e.pos = 0; continue;
    }
    if (e.field == 1 || e.field == 3) {
      e.field++; e.pos = 0; e.numlen = -1;
      return '|';
    }
    if (e.field == 2 || e.field == 4) {
      if (e.numlen < 0) e.numlen = fmt_ll(e.field == 2 ? e.M : e.B, e.num);
      if (e.pos < e.numlen) return (unsigned char)e.num[e.pos++];
      e.field = e.field == 2 ? 3 : 5; e.pos = 0; e.numlen = -1; continue;
    }
    // stage fields: 5 '|', 6 name, 7 ':', 8 begin, 9 '-', 10 end, 11 ':', 12 nodes,
    // 13 ':', 14 tp, 15 ':', 16 dp
    if (e.stage >= e.P) return -1;
    const LeafGroup& row = e.lg[e.slots[e.stage]];
    int g = row.group;
    switch (e.field) {
      case 5: e.field = 6; e.pos = 0; return '|';
      case 6:
        if (e.pos < e.c->name_len[g]) return (unsigned char)e.c->names[e.c->name_off[g] + e.pos++];
        e.field = 7; e.pos = 0; continue;
      case 7: case 11: case 13: case 15:
        e.field++; e.pos = 0; e.numlen = -1;
        return ':';
      case 9:
        e.field = 10; e.pos = 0; e.numlen = -1;
        return '-';
      case 8: case 10: case 12: case 14: case 16: {
        if (e.numlen < 0) {
          long long v;
          if (e.field == 8) v = e.begin;
          else if (e.field == 10) v = e.begin + e.counts[e.stage];
          else if (e.field == 12) v = row.nodes;
          else if (e.field == 14) v = row.tp;
          else v = e.dp;
          e.numlen = fmt_ll(v, e.num);
        }
        if (e.pos < e.numlen) return (unsigned char)e.num[e.pos++];
        if (e.field == 16) {
          e.begin += e.counts[e.stage];
          e.stage++;
          e.field = 5;
        } else {
          e.field++;
        }
        e.pos = 0;
        e.numlen = -1;
        continue;
      }
    }
  }
}

// std::string operator< on the two encodings.
HPD bool enc_less(EncStream& a, EncStream& b) {
  enc_init(a);
  enc_init(b);
  for (;;) {
    int x = enc_next(a), y = enc_next(b);
    if (x != y) return x < y;  // -1 (end) sorts first
    if (x < 0) return false;
  }
}

}  // namespace hpc
