// hp_log.cpp — search-log replay and formatting (see hp_log.hpp).
#include "hp_log.hpp"

#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <unordered_map>

#include "hp_search_core.cuh"

namespace hpl {
namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

// nlohmann::json::dump() string escaping (ensure_ascii = false).
void json_str(std::string& o, const char* s) {
  o.push_back('"');
  for (const unsigned char* c = reinterpret_cast<const unsigned char*>(s); *c; ++c) {
    switch (*c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (*c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", *c);
          o += buf;
        } else {
          o.push_back(static_cast<char>(*c));
        }
    }
  }
  o.push_back('"');
}

std::string layout_json(const hph::Problem& p, const hph::Task& t) {
  std::string o = "[";
  for (size_t i = 0; i < t.layout.size(); ++i) {
    if (i) o.push_back(',');
    json_str(o, p.groups[t.layout[i]].name);
  }
  o.push_back(']');
  return o;
}

// task_descriptor + "level" (planner.cpp:306-310, 323-325, 396-398); keys in
// nlohmann's sorted order.
std::string task_level_desc(const hph::Problem& p, const hph::Task& t) {
  return "{\"layout\":" + layout_json(p, t) + ",\"level\":\"pipeline\",\"pp\":" + std::to_string(t.pp) +
         "}";
}

// Leaf descriptor (planner.cpp:409-416, 496) split around the "split" array.
struct LeafDesc {
  std::string prefix, suffix;
};

LeafDesc leaf_desc(const hph::Problem& p, const hph::LeafHost& h) {
  const hph::Task& t = p.tasks[h.task];
  LeafDesc d;
  d.prefix = "{\"dp\":" + std::to_string(h.dp) + ",\"layout\":" + layout_json(p, t) +
             ",\"micro_batch_size\":" + std::to_string(static_cast<long long>(h.B)) +
             ",\"pp\":" + std::to_string(t.pp) + ",\"split\":[";
  std::map<std::string, int> tp;  // std::map: nlohmann's object key order
  for (size_t g = 0; g < p.groups.size(); ++g)
    if (t.spg[g] > 0) tp.emplace(p.groups[g].name, hph::leaf_tp(p, h, static_cast<int>(g)));
  d.suffix = "],\"tp\":{";
  bool first = true;
  for (const auto& kv : tp) {
    if (!first) d.suffix.push_back(',');
    first = false;
    json_str(d.suffix, kv.first.c_str());
    d.suffix += ":" + std::to_string(kv.second);
  }
  d.suffix += "}}";
  return d;
}

struct Replay {
  const hph::Problem& p;
  Log& out;
  hpc::Consts c{};
  std::vector<double> hop;
  bool pruning;
  double gb;
  std::string err;
  // task state (default mode incumbent, planner.cpp:519)
  bool has_best = false;
  double best = 0.0;

  Replay(const hph::Problem& pr, Log& o, double bound) : p(pr), out(o), gb(bound) {
    hph::fill_consts(p, c);
    hop = hph::hop_table(p);
    pruning = p.pruning;
  }

  uint64_t put(const std::string& s) {
    uint64_t off = out.text.size();
    out.text += s;
    out.text.push_back('\0');
    return off;
  }

  void entry(int task, int leaf, const std::string& cand, double t, const std::string& reason) {
    hp_log_entry e;
    e.candidate = put(cand);
    e.reason = put(reason);
    e.time_s = t;
    e.task = task;
    e.leaf = leaf;
    out.entries.push_back(e);
  }
};

// Source of simulated times for one leaf.
struct Times {
  const std::vector<double>* stream = nullptr;  // hill (full) or everything (default)
  size_t* pos = nullptr;
  bool next(double& t) {
    if (!stream || *pos >= stream->size()) return false;
    t = (*stream)[(*pos)++];
    return true;
  }
};

struct LeafReplay {
  Replay& r;
  int task, leaf_in_task;
  hpc::Leaf lf{};
  std::vector<hpc::LeafGroup> rows;
  const uint8_t* slots;
  const double* hop;
  LeafDesc desc;
  std::unordered_map<std::string, double> memo;  // split bytes -> time, < 0 when pruned

  LeafReplay(Replay& rp, int t, int lit, int gleaf) : r(rp), task(t), leaf_in_task(lit) {
    const hph::Problem& p = r.p;
    lf = hph::device_leaf(p, gleaf);
    rows.resize(p.groups.size());
    hph::leaf_rows(p, gleaf, rows.data());
    slots = p.layouts.data() + lf.layout_off;
    hop = r.hop.data() + (size_t)lf.B_idx * p.links.size();
    desc = leaf_desc(p, p.leaves[gleaf]);
  }

  static std::string key(const int* s, int P) {
    return std::string(reinterpret_cast<const char*>(s), sizeof(int) * P);
  }

  std::string cand(const int* s) const {
    std::string o = desc.prefix;
    for (int i = 0; i < lf.P; ++i) {
      if (i) o.push_back(',');
      o += std::to_string(s[i]);
    }
    return o + desc.suffix;
  }

  // Memory gate (planner.cpp:503-517) and compute lower bound
  // (planner.cpp:524-528). Returns -1 when feasible, else the failing stage.
  int gate(const int* s, double* lower) const {
    double lo = 0.0;
    for (int i = 0; i < lf.P; ++i) {
      hpc::StageDur d;
      if (!hpc::stage_setup(r.c, lf, rows.data(), slots, hop, i, s[i], d)) return i;
      lo = hpc::dmax(lo, static_cast<double>(lf.M) * (d.f + d.b));
    }
    *lower = lo;
    return -1;
  }

  std::string memory_reason(const int* s, int i) const {
    const hpc::LeafGroup& row = rows[slots[i]];
    double need = hpc::stage_memory(r.c, s[i], row.tp, static_cast<double>(lf.B),
                                    hpc::in_flight(r.c, i, lf.P, lf.M));
    char buf[96];
    std::string o = "stage " + std::to_string(i) + " memory ";
    std::snprintf(buf, sizeof buf, "%g", need);  // std::ostream default format
    o += buf;
    o += " B exceeds ";
    std::snprintf(buf, sizeof buf, "%g", r.c.budget[row.group]);
    o += buf;
    o += " B (";
    o += r.p.groups[row.group].name;
    o += " x headroom)";
    return o;
  }

  // evaluate_split (planner.cpp:492-551) with the time taken from `src`
  // (have_t: the caller supplies it instead). Returns the time or -1.
  double evaluate(const int* s, Times* src, bool have_t, double t_given) {
    double lower = 0.0;
    int bad = gate(s, &lower);
    if (bad >= 0) {
      r.entry(task, leaf_in_task, cand(s), -1.0, memory_reason(s, bad));
      r.out.pruned++;
      return -1.0;
    }
    const double inc = r.has_best && r.best < r.gb ? r.best : r.gb;
    if (r.pruning && inc < kInf && lower > inc) {
      r.entry(task, leaf_in_task, cand(s), -1.0, "compute lower bound above incumbent");
      r.out.pruned++;
      return -1.0;
    }
    double t = t_given;
    if (!have_t && !src->next(t)) {
      r.err = "search log: GPU time stream ended early";
      return -1.0;
    }
    if (!(t >= 0)) {
      r.err = "search log: GPU reports a memory-feasible candidate as pruned";
      return -1.0;
    }
    r.entry(task, leaf_in_task, cand(s), t, "");
    r.out.simulated++;
    if (!r.has_best || t < r.best) {
      r.has_best = true;
      r.best = t;
    }
    return t;
  }

  // try_split (planner.cpp:425-432)
  double try_split(const int* s, Times* src, bool have_t = false, double t_given = 0.0) {
    std::string k = key(s, lf.P);
    auto it = memo.find(k);
    if (it != memo.end()) return it->second;
    double t = evaluate(s, src, have_t, t_given);
    memo.emplace(std::move(k), t);
    return t;
  }

  // leaf_splits (planner.cpp:404-490). full: times of seeds come from
  // tseed (hill leaves) or the exhaustive rank array; default: everything
  // from `src` in order.
  void run(bool full, const double* tseed, const double* exh, long long n_exh, Times* src) {
    const int P = lf.P;
    const int L = r.c.L;
    std::vector<int> uni(P), prop(P), order(P);
    std::vector<double> w(P), frac(P);
    hpc::seed_splits(r.c, lf, rows.data(), slots, uni.data(), prop.data(), w.data(), frac.data(),
                     order.data());
    const bool exhaustive = lf.mode == 1;
    double t_seed[2] = {0.0, 0.0};
    if (full && exhaustive) {
      // seed times: their positions among the memory-feasible compositions
      std::vector<int> comp(P);
      hpc::unrank_composition(0, L, P, comp.data());
      long long rank = 0;
      double lower;
      do {
        if (gate(comp.data(), &lower) < 0) {
          if (rank < n_exh) {
            if (comp == uni) t_seed[0] = exh[rank];
            if (comp == prop) t_seed[1] = exh[rank];
          }
          ++rank;
        }
      } while (hpc::next_composition(comp.data(), P));
    } else if (full) {
      t_seed[0] = tseed[0];
      t_seed[1] = tseed[1];
    }
    try_split(uni.data(), src, full, t_seed[0]);
    if (r.p.uniform_only || !r.err.empty()) return;
    try_split(prop.data(), src, full, t_seed[1]);
    if (!r.err.empty()) return;

    if (exhaustive) {
      std::vector<int> comp(P);
      hpc::unrank_composition(0, L, P, comp.data());
      long long rank = 0;
      do {
        double lower;
        if (full) {
          const bool feasible = gate(comp.data(), &lower) < 0;
          double t = 0.0;
          if (feasible) {
            if (rank >= n_exh) {
              r.err = "search log: exhaustive rank array too short";
              return;
            }
            t = exh[rank++];
          }
          try_split(comp.data(), src, true, t);
        } else {
          try_split(comp.data(), src);
        }
        if (!r.err.empty()) return;
      } while (hpc::next_composition(comp.data(), P));
      if (full && rank != n_exh) r.err = "search log: exhaustive rank count mismatch";
      return;
    }

    std::vector<int> cur = prop;
    double cur_t = try_split(cur.data(), src);
    if (cur_t < 0) {
      cur = uni;
      cur_t = try_split(cur.data(), src);
    }
    std::vector<int> nb(P), best_nb(P);
    for (int step = 0; step < 4 * L && cur_t >= 0; ++step) {
      double bt = -1.0;
      for (int i = 0; i + 1 < P; ++i) {
        for (int d : {+1, -1}) {
          nb = cur;
          nb[i] += d;
          nb[i + 1] -= d;
          if (nb[i] < 1 || nb[i + 1] < 1) continue;
          double t = try_split(nb.data(), src);
          if (!r.err.empty()) return;
          if (t >= 0 && (bt < 0 || t < bt)) {
            bt = t;
            best_nb = nb;
          }
        }
      }
      if (bt < 0 || !(bt < cur_t)) break;
      cur = best_nb;
      cur_t = bt;
    }
  }
};

std::string no_link_reason(const hph::Problem& p, const hph::Task& t) {
  for (size_t i = 0; i + 1 < t.layout.size(); ++i) {
    int a = t.layout[i], b = t.layout[i + 1];
    if (a != b && p.pair[a][b] < 0)
      return std::string("no heterogeneous link between '") + p.groups[a].name + "' and '" +
             p.groups[b].name + "'";
  }
  return "";
}

}  // namespace

hph::Status build(const hph::Problem& p, const hpd::LogRaw& raw, double global_bound,
                  bool task_entries, Log& out) {
  out.clear();
  Replay r(p, out, global_bound);
  const bool full = !p.pruning;
  const int T = static_cast<int>(p.tasks.size());
  std::vector<int> pos_of(full ? p.leaves.size() : p.tasks.size(), -1);
  for (size_t k = 0; k < raw.key_of.size(); ++k) pos_of[raw.key_of[k]] = static_cast<int>(k);
  std::vector<size_t> used(raw.streams.size(), 0);
  if (raw.streams.size() != raw.key_of.size())
    return hph::Status{HP_INTERNAL, "search log: stream count mismatch"};
  if (full && raw.tseed.size() != 2 * raw.key_of.size())
    return hph::Status{HP_INTERNAL, "search log: seed times missing"};

  // end of each exhaustive leaf's rank array (offsets ascend with k)
  std::vector<long long> exh_end(raw.exh_off.size(), 0);
  long long next_off = static_cast<long long>(raw.exh.size());
  for (size_t j = raw.exh_off.size(); j-- > 0;) {
    exh_end[j] = next_off;
    if (raw.exh_off[j] >= 0) next_off = raw.exh_off[j];
  }

  for (int ti = 0; ti < T; ++ti) {
    const hph::Task& t = p.tasks[ti];
    if (t.no_link || t.leaf_begin == t.leaf_end) {
      if (task_entries) {
        // planner.cpp:317-327 / 395-400
        std::string reason = t.no_link ? no_link_reason(p, t) : "no integral dp/tp/micro-batch assignment";
        r.entry(ti, -1, task_level_desc(p, t), -1.0, reason);
        out.pruned++;
      }
      continue;
    }
    if (full) {
      for (int li = t.leaf_begin; li < t.leaf_end; ++li) {
        const int k = pos_of[li];
        if (k < 0) continue;  // another shard's leaf
        r.has_best = false;   // no incumbent in full mode; kept per leaf
        Times src{&raw.streams[k], &used[k]};
        LeafReplay lr(r, ti, li - t.leaf_begin, li);
        const double* exh = nullptr;
        long long n_exh = 0;
        if (lr.lf.mode == 1) {
          if (raw.exh_off.size() != raw.key_of.size() || raw.exh_off[k] < 0)
            return hph::Status{HP_INTERNAL, "search log: exhaustive times missing"};
          exh = raw.exh.data() + raw.exh_off[k];
          n_exh = exh_end[k] - raw.exh_off[k];
        }
        lr.run(true, &raw.tseed[2 * k], exh, n_exh, &src);
        if (!r.err.empty()) return hph::Status{HP_INTERNAL, r.err};
      }
    } else {
      const int k = pos_of[ti];
      if (k < 0) continue;  // another shard's task
      r.has_best = false;
      Times src{&raw.streams[k], &used[k]};
      for (int li = t.leaf_begin; li < t.leaf_end; ++li) {
        LeafReplay lr(r, ti, li - t.leaf_begin, li);
        lr.run(false, nullptr, nullptr, 0, &src);
        if (!r.err.empty()) return hph::Status{HP_INTERNAL, r.err};
      }
    }
  }
  for (size_t k = 0; k < used.size(); ++k)
    if (used[k] != raw.streams[k].size())
      return hph::Status{HP_INTERNAL, "search log: GPU time stream not fully consumed"};
  out.valid = true;
  return hph::Status{};
}

}  // namespace hpl
