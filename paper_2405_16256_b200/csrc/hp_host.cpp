// hp_host.cpp — validation, enumeration and exact-order cost tables (host).
#include "hp_host.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <set>
#include <sstream>
#include <thread>

namespace hph {

namespace {

Status bad(const std::string& m) { return Status{HP_BAD_CONFIG, m}; }

std::string gname(const Problem& p, int g) { return p.names[g]; }

}  // namespace

Status load_problem(const hp_problem* in, Problem& p) {
  if (in == nullptr) return bad("null problem");
  p.model = in->model;
  const hp_cluster& c = in->cluster;
  if (c.n_groups < 0 || c.n_links < 0) return bad("cluster: negative counts");
  if (c.n_groups > HP_MAX_GROUPS)
    return bad("cluster: at most " + std::to_string(HP_MAX_GROUPS) + " device groups supported");
  p.groups.assign(c.groups, c.groups + c.n_groups);
  p.links.assign(c.links, c.links + c.n_links);
  p.names.assign(p.groups.size(), std::string());
  p.names_blob.clear();
  p.name_off.assign(p.groups.size(), 0);
  for (size_t g = 0; g < p.groups.size(); ++g) {
    if (p.groups[g].name) p.names[g] = p.groups[g].name;
    p.name_off[g] = static_cast<int>(p.names_blob.size());
    p.names_blob += p.names[g];
  }
  for (size_t g = 0; g < p.groups.size(); ++g) p.groups[g].name = p.names[g].c_str();
  p.train = in->train;

  // ---- validate_spec(ModelSpec), types.cpp:78-91
  const hp_model& m = p.model;
  if (m.num_layers < 1) return bad("model: num_layers must be >= 1");
  if (m.hidden_size < 1) return bad("model: hidden_size must be >= 1");
  if (m.seq_length < 1) return bad("model: seq_length must be >= 1");
  if (m.num_heads < 1) return bad("model: num_heads must be >= 1");
  if (m.hidden_size % m.num_heads != 0)
    return bad("model: hidden_size must be divisible by num_heads");
  if (m.bytes_per_element != 2 && m.bytes_per_element != 4)
    return bad("model: bytes_per_element must be 2 or 4");
  if (m.activation_bytes_per_token_per_hidden < 0)
    return bad("model: activation_bytes_per_token_per_hidden must be >= 0");
  if (m.edge_layer_cost_multiplier < 0)
    return bad("model: edge_layer_cost_multiplier must be >= 0");

  // ---- validate_spec(ClusterSpec), types.cpp:93-154
  if (p.groups.empty()) return bad("cluster: at least one device group required");
  std::set<std::string> names;
  for (hp_group& g : p.groups) {
    std::string n = g.name;
    if (n.empty()) return bad("cluster: group name must be non-empty");
    if (!names.insert(n).second) return bad("cluster: duplicate group name '" + n + "'");
    if (g.peak_tflops <= 0) return bad("cluster: group '" + n + "': peak_tflops must be > 0");
    if (g.memory_bytes <= 0) return bad("cluster: group '" + n + "': memory_bytes must be > 0");
    if (g.node_count < 1) return bad("cluster: group '" + n + "': node_count must be >= 1");
    if (g.devices_per_node < 1)
      return bad("cluster: group '" + n + "': devices_per_node must be >= 1");
    if (g.compute_efficiency <= 0 || g.compute_efficiency > 1.5)
      return bad("cluster: group '" + n + "': compute_efficiency must be in (0, 1.5]");
    if (g.bwd_fwd_ratio < 1.0)
      return bad("cluster: group '" + n + "': bwd_fwd_ratio must be >= 1");
  }
  const int G = static_cast<int>(p.groups.size());
  int intra_count[HP_MAX_GROUPS] = {0}, inter_count[HP_MAX_GROUPS] = {0};
  std::set<std::pair<int, int>> pairs;
  for (int g = 0; g < HP_MAX_GROUPS; ++g) {
    p.intra[g] = p.inter[g] = -1;
    for (int h = 0; h < HP_MAX_GROUPS; ++h) p.pair[g][h] = -1;
  }
  for (int i = 0; i < static_cast<int>(p.links.size()); ++i) {
    const hp_link& l = p.links[i];
    if (l.bandwidth_bits_per_s <= 0) return bad("cluster: link bandwidth_bits_per_s must be > 0");
    if (l.latency_s < 0) return bad("cluster: link latency_s must be >= 0");
    if (l.efficiency <= 0 || l.efficiency > 1) return bad("cluster: link efficiency must be in (0, 1]");
    if (l.path != HP_GPU_DIRECT && l.path != HP_CPU_STAGED) return bad("cluster: unknown path_kind");
    if (l.path == HP_CPU_STAGED && l.staging_copy_bytes_per_s <= 0)
      return bad("cluster: cpu-staged link must carry a positive staging_copy_bytes_per_s");
    if (l.scope == HP_INTRA_NODE || l.scope == HP_INTER_NODE) {
      if (l.group_a < 0 || l.group_a >= G)
        return bad(l.group_a_name ? "cluster: link references unknown group '" + std::string(l.group_a_name) + "'"
                                  : std::string("cluster: link references unknown group"));
      int& cnt = l.scope == HP_INTRA_NODE ? intra_count[l.group_a] : inter_count[l.group_a];
      if (++cnt > 1)
        return bad("cluster: group '" + gname(p, l.group_a) + "' has more than one " +
                   (l.scope == HP_INTRA_NODE ? "intra-node" : "inter-node-homogeneous") + " link");
      if (l.scope == HP_INTRA_NODE) p.intra[l.group_a] = i;
      else p.inter[l.group_a] = i;
    } else if (l.scope == HP_INTER_GROUP) {
      if (l.group_a < 0 || l.group_a >= G || l.group_b < 0 || l.group_b >= G)
        return bad("cluster: inter-group link references undeclared group");
      if (l.group_a == l.group_b) return bad("cluster: inter-group link must connect two distinct groups");
      auto key = std::minmax(gname(p, l.group_a), gname(p, l.group_b));
      int a = std::min(l.group_a, l.group_b), b = std::max(l.group_a, l.group_b);
      if (!pairs.insert({a, b}).second)
        return bad("cluster: duplicate inter-group link between '" + key.first + "' and '" +
                   key.second + "'");
      p.pair[l.group_a][l.group_b] = p.pair[l.group_b][l.group_a] = i;
    } else {
      return bad("cluster: unknown link scope kind");
    }
  }
  for (int g = 0; g < G; ++g) {
    if (intra_count[g] != 1)
      return bad("cluster: group '" + gname(p, g) + "' needs exactly one intra-node link");
    if (inter_count[g] != 1)
      return bad("cluster: group '" + gname(p, g) + "' needs exactly one inter-node-homogeneous link");
  }

  // ---- validate_spec(TrainConfig), types.cpp:156-163
  if (p.train.global_batch_size < 1) return bad("train: global_batch_size must be >= 1");
  if (p.train.micro_batch_size < 1) return bad("train: micro_batch_size must be >= 1");
  if (p.train.micro_batch_size > p.train.global_batch_size)
    return bad("train: micro_batch_size must not exceed global_batch_size");
  if (p.train.optimizer_state_multiplier <= 0)
    return bad("train: optimizer_state_multiplier must be > 0");

  // ---- planner normalisation, planner.cpp:585-607
  const hp_planner& pl = in->planner;
  p.total_nodes = 0;
  for (const hp_group& g : p.groups) p.total_nodes += g.node_count;
  p.pps.clear();
  if (pl.n_pipeline_degrees <= 0) {
    int cap = std::min(m.num_layers, p.total_nodes);
    for (int k = 1; k <= cap; ++k) p.pps.push_back(k);
  } else {
    p.pps.assign(pl.pipeline_degrees, pl.pipeline_degrees + pl.n_pipeline_degrees);
  }
  std::sort(p.pps.begin(), p.pps.end());
  p.pps.erase(std::unique(p.pps.begin(), p.pps.end()), p.pps.end());
  p.mbs.clear();
  if (pl.n_micro_batch_candidates <= 0) p.mbs.push_back(p.train.micro_batch_size);
  else p.mbs.assign(pl.micro_batch_candidates, pl.micro_batch_candidates + pl.n_micro_batch_candidates);
  std::sort(p.mbs.begin(), p.mbs.end());
  p.mbs.erase(std::unique(p.mbs.begin(), p.mbs.end()), p.mbs.end());
  for (int k : p.pps)
    if (k < 1) return bad("planner: pipeline degrees must be >= 1");
  for (int64_t b : p.mbs)
    if (b < 1) return bad("planner: micro-batch candidates must be >= 1");
  if (!(pl.memory_headroom > 0) || pl.memory_headroom > 1)
    return bad("planner: memory_headroom must be in (0, 1]");
  if (pl.stage_order_beam_width < 0) return bad("planner: stage_order_beam_width must be >= 0");
  if (pl.schedule != HP_GPIPE && pl.schedule != HP_1F1B) return bad("planner: unknown schedule");
  p.headroom = pl.memory_headroom;
  p.beam = pl.stage_order_beam_width;
  p.limit = pl.exhaustive_split_limit;
  p.uniform_only = pl.uniform_split_only != 0;
  p.interleave = pl.allow_group_interleaving != 0;
  p.pruning = pl.time_bound_pruning != 0;
  p.schedule = pl.schedule;
  for (int k : p.pps)
    if (k > HP_MAX_STAGES && k <= m.num_layers)
      return bad("planner: pipeline degree above HP_MAX_STAGES (" + std::to_string(HP_MAX_STAGES) + ")");
  return Status{};
}

// ------------------------------------------------------------ enumeration

namespace {

void layouts_for(Problem& p, int pp, const std::vector<int>& comp) {
  const int G = static_cast<int>(p.groups.size());
  std::vector<std::vector<int>> layouts;
  if (p.interleave) {
    std::vector<int> labels;
    for (int g = 0; g < G; ++g) labels.insert(labels.end(), comp[g], g);
    int seen = 0;
    do {
      layouts.push_back(labels);
      if (p.beam > 0 && ++seen >= p.beam) break;
    } while (std::next_permutation(labels.begin(), labels.end()));
  } else {
    std::vector<int> part;
    for (int g = 0; g < G; ++g)
      if (comp[g] > 0) part.push_back(g);
    std::vector<int> perm(part.size());
    std::iota(perm.begin(), perm.end(), 0);
    int seen = 0;
    do {
      std::vector<int> layout;
      for (int b : perm) layout.insert(layout.end(), comp[part[b]], part[b]);
      layouts.push_back(std::move(layout));
      if (p.beam > 0 && ++seen >= p.beam) break;
    } while (std::next_permutation(perm.begin(), perm.end()));
  }
  for (auto& l : layouts) {
    Task t;
    t.pp = pp;
    for (int g = 0; g < G; ++g) t.spg[g] = comp[g];
    t.layout = std::move(l);
    p.tasks.push_back(std::move(t));
  }
}

void compositions(Problem& p, int pp, int g, int remaining, std::vector<int>& cur) {
  const int G = static_cast<int>(p.groups.size());
  if (g == G) {
    if (remaining == 0) layouts_for(p, pp, cur);
    return;
  }
  int cap = std::min(remaining, p.groups[g].node_count);
  for (int s = 0; s <= cap; ++s) {
    cur.push_back(s);
    compositions(p, pp, g + 1, remaining - s, cur);
    cur.pop_back();
  }
}

}  // namespace

namespace {

// run_task's leaves of tasks [t0, t1) into out / tp (task-local tp_base and
// leaf_begin / leaf_end offsets, rebased by the caller).
void enumerate_leaves(Problem& p, int t0, int t1, const std::vector<long long>& dps, std::vector<LeafHost>& out,
                      std::vector<int32_t>& tp_out) {
  const int G = static_cast<int>(p.groups.size());
  const int L = p.model.num_layers;
  std::vector<std::vector<int>> tpo(G), okt(G);
  std::vector<size_t> idx(G);
  for (int ti = t0; ti < t1; ++ti) {
    Task& t = p.tasks[ti];
    t.leaf_begin = t.leaf_end = static_cast<int>(out.size());
    for (int i = 0; i + 1 < t.pp; ++i) {
      int a = t.layout[i], b = t.layout[i + 1];
      if (a != b && p.pair[a][b] < 0) {
        t.no_link = true;
        break;
      }
    }
    if (t.no_link) continue;
    long long dp_max = std::numeric_limits<long long>::max();
    for (int g = 0; g < G; ++g) {
      if (t.spg[g] == 0) continue;
      long long nps = p.groups[g].node_count / t.spg[g];
      dp_max = std::min(dp_max, nps * p.groups[g].devices_per_node);
    }
    for (int g = 0; g < G; ++g) {
      tpo[g].assign(1, 1);
      if (t.spg[g] > 0) {
        tpo[g].clear();
        for (int d = 1; d <= p.groups[g].devices_per_node; ++d)
          if (p.groups[g].devices_per_node % d == 0) tpo[g].push_back(d);
      }
    }
    const long long nsplit = hpc::contiguous_split_count(L, t.pp);
    // The allotment test (planner.cpp:366-379) is per group, so the leaves
    // of a (dp, B) are the product of each group's passing tp values, in the
    // odometer order (group 0 fastest) restricted to them.
    for (long long dp : dps) {
      if (dp > dp_max) continue;
      bool empty = false;
      for (int g = 0; g < G; ++g) {
        okt[g].clear();
        for (int tp : tpo[g]) {
          if (t.spg[g] == 0) {
            okt[g].push_back(tp);
            continue;
          }
          long long dev = dp * tp;
          if (dev % p.groups[g].devices_per_node != 0) continue;
          long long nu = dev / p.groups[g].devices_per_node;
          if (nu < 1 || nu * t.spg[g] > p.groups[g].node_count) continue;
          okt[g].push_back(tp);
        }
        empty = empty || okt[g].empty();
      }
      if (empty) continue;
      for (int bi = 0; bi < static_cast<int>(p.mbs.size()); ++bi) {
        int64_t B = p.mbs[bi];
        if (p.train.global_batch_size % (dp * B) != 0) continue;
        std::fill(idx.begin(), idx.end(), 0);
        for (;;) {
          LeafHost lf{};
          lf.task = ti;
          lf.dp = static_cast<int>(dp);
          lf.B = B;
          lf.B_idx = bi;
          lf.M = p.train.global_batch_size / (dp * B);
          lf.tp_base = static_cast<int>(tp_out.size());
          for (int g = 0; g < G; ++g) tp_out.push_back(okt[g][idx[g]]);
          lf.n_splits = nsplit;
          lf.exhaustive = !p.uniform_only && nsplit <= p.limit;
          double pm = static_cast<double>(t.pp) * static_cast<double>(lf.M);
          lf.cost = lf.exhaustive ? pm * static_cast<double>(nsplit) : pm * (2.0 + 12.0 * 2.0 * (t.pp - 1));
          out.push_back(lf);
          int g = 0;
          while (g < G && ++idx[g] == okt[g].size()) idx[g++] = 0;
          if (g == G) break;
        }
      }
    }
    t.leaf_end = static_cast<int>(out.size());
  }
}

}  // namespace

void enumerate(Problem& p) {
  p.tasks.clear();
  p.leaves.clear();
  p.leaf_tp.clear();
  p.layouts.clear();
  const int G = static_cast<int>(p.groups.size());
  const int L = p.model.num_layers;
  for (int pp : p.pps) {
    if (pp < 1 || pp > L) continue;
    std::vector<int> cur;
    compositions(p, pp, 0, pp, cur);
  }
  for (Task& t : p.tasks) {
    t.layout_off = static_cast<int>(p.layouts.size());
    for (int g : t.layout) p.layouts.push_back(static_cast<uint8_t>(g));
  }
  // dp values some micro-batch candidate divides the global batch with
  // (planner.cpp:355-357), descending; a task walks them from its dp_max
  long long dp_cap = 1;
  for (int g = 0; g < G; ++g)
    dp_cap = std::max(dp_cap, static_cast<long long>(p.groups[g].node_count) * p.groups[g].devices_per_node);
  std::vector<long long> dps;
  for (long long dp = dp_cap; dp >= 1; --dp)
    for (int64_t B : p.mbs)
      if (p.train.global_batch_size % (dp * B) == 0) {
        dps.push_back(dp);
        break;
      }
  // Tasks are independent here: contiguous task ranges on host threads,
  // concatenated in task order (the reference's leaf order).
  const int T = static_cast<int>(p.tasks.size());
  const int nth = std::max(1, std::min({T / 256, 8, static_cast<int>(std::thread::hardware_concurrency())}));
  std::vector<std::vector<LeafHost>> part(nth);
  std::vector<std::vector<int32_t>> part_tp(nth);
  std::vector<std::thread> th;
  for (int k = 0; k < nth; ++k) {
    const int t0 = static_cast<int>(static_cast<long long>(T) * k / nth);
    const int t1 = static_cast<int>(static_cast<long long>(T) * (k + 1) / nth);
    if (nth == 1) enumerate_leaves(p, t0, t1, dps, part[k], part_tp[k]);
    else th.emplace_back(enumerate_leaves, std::ref(p), t0, t1, std::cref(dps), std::ref(part[k]), std::ref(part_tp[k]));
  }
  for (auto& x : th) x.join();
  size_t nl = 0, ntp = 0;
  for (int k = 0; k < nth; ++k) {
    nl += part[k].size();
    ntp += part_tp[k].size();
  }
  p.leaves.reserve(nl);
  p.leaf_tp.reserve(ntp);
  for (int k = 0; k < nth; ++k) {
    const int t0 = static_cast<int>(static_cast<long long>(T) * k / nth);
    const int t1 = static_cast<int>(static_cast<long long>(T) * (k + 1) / nth);
    const int lo = static_cast<int>(p.leaves.size()), to = static_cast<int>(p.leaf_tp.size());
    for (int ti = t0; ti < t1; ++ti) {
      p.tasks[ti].leaf_begin += lo;
      p.tasks[ti].leaf_end += lo;
    }
    for (LeafHost& lf : part[k]) {
      lf.tp_base += to;
      p.leaves.push_back(lf);
    }
    p.leaf_tp.insert(p.leaf_tp.end(), part_tp[k].begin(), part_tp[k].end());
  }
}

// ------------------------------------------------------------ cost terms

double hop_time(const Problem& p, int link, int64_t B) {
  const hp_link& l = p.links[link];
  // p2p_activation_volume, cost_model.cpp:23-27
  double vol = static_cast<double>(B) * static_cast<double>(p.model.seq_length) *
               static_cast<double>(p.model.hidden_size) * p.model.bytes_per_element;
  // hop_time, cost_model.cpp:43-61: latency, then the hops in order
  double wire = vol * 8.0 / (l.bandwidth_bits_per_s * l.efficiency);
  double t = l.latency_s;
  if (l.path == HP_CPU_STAGED) {
    double copy = vol / l.staging_copy_bytes_per_s;
    t += copy;
    t += wire;
    t += copy;
  } else {
    t += wire;
  }
  return t;
}

namespace {

// collective_time AllReduce, cost_model.cpp:63-73
double allreduce(double vol, int ranks, const hp_link& l) {
  if (ranks == 1) return 0.0;
  double factor = 2.0;
  double steps = factor * (ranks - 1);
  double moved = factor * (ranks - 1) / static_cast<double>(ranks) * vol;
  return steps * l.latency_s + moved * 8.0 / (l.bandwidth_bits_per_s * l.efficiency);
}

}  // namespace

hpc::LeafGroup leaf_group(const Problem& p, int g, int tp, int64_t B, int dp, int nodes) {
  const hp_model& m = p.model;
  const hp_group& grp = p.groups[g];
  const hp_link& intra = p.links[p.intra[g]];
  hpc::LeafGroup r{};
  // layer_flops, cost_model.cpp:29-35
  const double Bd = static_cast<double>(B), Ld = static_cast<double>(m.seq_length),
               Hd = static_cast<double>(m.hidden_size);
  double fwd_flops = 24.0 * Bd * Ld * Hd * Hd + 4.0 * Bd * Ld * Ld * Hd;
  // compute_time, cost_model.cpp:37-41
  double fwd_compute = fwd_flops / (tp * grp.peak_tflops * 1e12 * grp.compute_efficiency);
  // layer_cost, cost_model.cpp:88-107
  double tp_volume = Bd * Ld * Hd * m.bytes_per_element;
  double tp_sync = 2.0 * allreduce(tp_volume, tp, intra);
  r.fl = fwd_compute + tp_sync;
  r.bl = fwd_compute * grp.bwd_fwd_ratio + tp_sync;
  r.pbytes = 12.0 * Hd * Hd * m.bytes_per_element;
  // DP sync link, evaluate.cpp:68; constants of collective_time
  const hp_link& dl = nodes > 1 ? p.links[p.inter[g]] : intra;
  double factor = 2.0;
  double steps = factor * (dp - 1);
  r.ar_lat = steps * dl.latency_s;
  r.ar_mf = factor * (dp - 1) / static_cast<double>(dp);
  r.ar_den = dl.bandwidth_bits_per_s * dl.efficiency;
  // stage_weights, planner.cpp:94
  r.weight = grp.peak_tflops * grp.compute_efficiency * tp;
  r.tp = tp;
  r.nodes = nodes;
  r.group = g;
  r.dp = dp;
  return r;
}

void fill_consts(const Problem& p, hpc::Consts& c) {
  std::memset(&c, 0, sizeof c);
  c.L = p.model.num_layers;
  c.n_groups = static_cast<int>(p.groups.size());
  c.schedule = p.schedule;
  c.pruning = p.pruning ? 1 : 0;
  c.H = static_cast<double>(p.model.hidden_size);
  c.seq = static_cast<double>(p.model.seq_length);
  c.bytes = p.model.bytes_per_element;
  c.act = p.model.activation_bytes_per_token_per_hidden;
  c.edge = p.model.edge_layer_cost_multiplier;
  c.osm = p.train.optimizer_state_multiplier;
  for (int g = 0; g < c.n_groups; ++g) {
    c.budget[g] = p.groups[g].memory_bytes * p.headroom;  // planner.cpp:508
    c.link_inter[g] = p.inter[g];
    for (int h = 0; h < c.n_groups; ++h) c.link_pair[g][h] = g == h ? p.inter[g] : p.pair[g][h];
    c.name_off[g] = p.name_off[g];
    c.name_len[g] = static_cast<int>(p.names[g].size());
  }
  c.names = p.names_blob.data();  // host copy; device users point it at a device copy
  c.n_links = static_cast<int>(p.links.size());
  c.n_B = static_cast<int>(p.mbs.size());
}

hpc::Leaf device_leaf(const Problem& p, int li) {
  const LeafHost& h = p.leaves[li];
  const Task& t = p.tasks[h.task];
  hpc::Leaf lf{};
  lf.task = h.task;
  lf.P = t.pp;
  lf.M = static_cast<int>(h.M);
  lf.dp = h.dp;
  lf.B = h.B;
  lf.B_idx = h.B_idx;
  lf.layout_off = t.layout_off;
  lf.mode = p.uniform_only ? 2 : (h.exhaustive ? 1 : 0);
  lf.sched = p.schedule;
  return lf;
}

void leaf_rows(const Problem& p, int li, hpc::LeafGroup* rows) {
  const LeafHost& h = p.leaves[li];
  for (int g = 0; g < static_cast<int>(p.groups.size()); ++g)
    rows[g] = leaf_group(p, g, leaf_tp(p, h, g), h.B, h.dp, leaf_nodes(p, h, g));
}

std::vector<double> hop_table(const Problem& p) {
  std::vector<double> hop(p.mbs.size() * p.links.size());
  for (size_t bi = 0; bi < p.mbs.size(); ++bi)
    for (size_t l = 0; l < p.links.size(); ++l)
      hop[bi * p.links.size() + l] = hop_time(p, static_cast<int>(l), p.mbs[bi]);
  return hop;
}

// ------------------------------------------------------------ sharding

std::vector<int> shard_leaves(const Problem& p, int shard, int count) {
  std::vector<int> out;
  if (count <= 1) {
    out.resize(p.leaves.size());
    std::iota(out.begin(), out.end(), 0);
    return out;
  }
  // Boustrophedon over leaves sorted by estimated cost: neighbours in that
  // order (similar P, M) land on different ranks, which averages out the
  // unpredictable hill-climb lengths far better than greedy LPT on the
  // estimate (C3: max/mean shard work 1.01-1.04 vs 1.35 for N = 2..8).
  std::vector<int> order(p.leaves.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return p.leaves[a].cost > p.leaves[b].cost; });
  std::vector<char> mine(p.leaves.size(), 0);
  for (size_t k = 0; k < order.size(); ++k) {
    const int c = static_cast<int>(k % (2 * count));
    const int owner = c < count ? c : 2 * count - 1 - c;
    if (owner == shard) mine[order[k]] = 1;
  }
  for (int li = 0; li < static_cast<int>(p.leaves.size()); ++li)
    if (mine[li]) out.push_back(li);
  return out;
}

std::vector<int> shard_tasks(const Problem& p, int shard, int count) {
  std::vector<int> out;
  if (count <= 1) {
    out.resize(p.tasks.size());
    std::iota(out.begin(), out.end(), 0);
    return out;
  }
  std::vector<double> tcost(p.tasks.size(), 1.0);
  for (const LeafHost& lf : p.leaves) tcost[lf.task] += lf.cost;
  std::vector<int> order(p.tasks.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tcost[a] > tcost[b]; });
  std::vector<char> mine(p.tasks.size(), 0);
  for (size_t k = 0; k < order.size(); ++k) {
    const int c = static_cast<int>(k % (2 * count));
    const int owner = c < count ? c : 2 * count - 1 - c;
    if (owner == shard) mine[order[k]] = 1;
  }
  for (int ti = 0; ti < static_cast<int>(p.tasks.size()); ++ti)
    if (mine[ti]) out.push_back(ti);
  return out;
}

// ------------------------------------------------------------ plans

void make_plan(const Problem& p, const LeafHost& lf, const int* split, hp_plan& out) {
  const Task& t = p.tasks[lf.task];
  std::memset(&out, 0, sizeof out);
  out.schedule = p.schedule;
  out.micro_batch_size = lf.B;
  out.micro_batches_per_dp_replica = lf.M;
  out.n_stages = t.pp;
  int begin = 0;
  for (int i = 0; i < t.pp; ++i) {
    int g = t.layout[i];
    hp_stage& s = out.stages[i];
    s.layer_begin = begin;
    s.layer_end = begin + split[i];
    begin += split[i];
    s.group = g;
    s.tp_degree = leaf_tp(p, lf, g);
    s.dp_degree = lf.dp;
    s.nodes_used = static_cast<int>(static_cast<long long>(lf.dp) * s.tp_degree /
                                    p.groups[g].devices_per_node);
  }
}

std::string encode_plan(const Problem& p, const hp_plan& plan) {
  std::ostringstream os;
  os << (plan.schedule == HP_GPIPE ? "gpipe" : "1f1b") << '|' << plan.micro_batches_per_dp_replica
     << '|' << plan.micro_batch_size;
  for (int i = 0; i < plan.n_stages; ++i) {
    const hp_stage& s = plan.stages[i];
    os << '|' << p.groups[s.group].name << ':' << s.layer_begin << '-' << s.layer_end << ':'
       << s.nodes_used << ':' << s.tp_degree << ':' << s.dp_degree;
  }
  return os.str();
}

int compare_plans(const Problem& p, double ta, const hp_plan& a, double tb, const hp_plan& b) {
  if (ta != tb) return ta < tb ? -1 : 1;
  if (a.n_stages != b.n_stages) return a.n_stages < b.n_stages ? -1 : 1;
  std::string ea = encode_plan(p, a), eb = encode_plan(p, b);
  if (ea == eb) return 0;
  return ea < eb ? -1 : 1;
}

}  // namespace hph
