// hp_kernels.cu — sm_100a kernels of the candidate-evaluation engine.
//
// The path is FP64 add/max and integer control work (no GEMM, no tensor
// cores): per candidate a max-plus recurrence over 2*P*M compute nodes and
// 2*(P-1)*M send nodes (simulate, sim.cpp:63-195). Layout in HBM: one Leaf
// record per leaf, LeafGroup rows per (leaf, group), P-int split rows per
// leaf (uniform / proportional / current / best), per-leaf move history;
// cost tables are a few KB and sit in __constant__ / L1. HBM traffic per
// candidate is O(P) bytes, so the kernels are bound by FP64/ALU issue and
// warp-shuffle exchange, not by DRAM.
//
// Kernels:
//   k_seeds        one thread per leaf: uniform + proportional splits
//                  (split_layers on device, planner.cpp:42-104).
//   k_eval<K>      warp-segment evaluator: a warp holds 32/W2 candidates of
//                  one leaf, lane = K consecutive pipeline stages; the 1F1B /
//                  GPipe DAG runs level-synchronously with __shfl exchange of
//                  the neighbours' channel state (hp_core.cuh).
//   k_hill_init / k_gen / k_hill_step
//                  steepest-descent layer-split search (planner.cpp:461-489)
//                  with memo-equivalent counting (hp_search_core.cuh).
//   k_exh_reduce   per-leaf reduction of exhaustively enumerated splits.
//   k_final        exact better_than argmin over leaf bests.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hp_device.hpp"
#include "hp_host.hpp"
#include "hp_search_core.cuh"

namespace hpk {

using namespace hpc;

__constant__ Consts c_consts;

// Work item of the evaluator: up to 32/W2 candidates of one leaf.
//   kind 0: seeds (cand s: first+s == 0 uniform, 1 prop)    -> tseed[2*leaf+first+s]
//   kind 1: hill neighbours, slots first..first+n-1 of cur   -> nb[nb_off+slot]
//   kind 2: exhaustive ranks first..first+n-1               -> xbuf[out+s]
struct Work {
  int leaf;
  int kind;
  long long first;
  int n;
  int out;
};

struct Bufs {
  const Leaf* leaves;
  const LeafGroup* lg;
  const uint8_t* layouts;
  const double* hop;      // [n_B][n_links]
  int* uni;
  int* prop;
  int* cur;
  int* best;
  short* hist;
  const int* hist_off;
  const int* nb_off;
  double* tseed;
  double* nb;
  double* xbuf;
  HillState* hs;
};

__device__ __forceinline__ int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// Lanes per candidate segment for a leaf with P stages at K stages per lane.
__host__ __device__ inline int seg_width(int P, int K) {
  int w = (P + K - 1) / K;
  int p = 1;
  while (p < w) p <<= 1;
  return p;
}

__host__ __device__ inline int k_class(int P) {
  int k = (P + 31) / 32;
  return k < 1 ? 1 : k;
}

// ------------------------------------------------------------------ seeds

__global__ void k_seeds(Bufs b, int n_leaves) {
  int li = blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= n_leaves) return;
  const Leaf lf = b.leaves[li];
  double w[HP_MAX_STAGES], frac[HP_MAX_STAGES];
  int order[HP_MAX_STAGES];
  seed_splits(c_consts, lf, b.lg + lf.lg_off, b.layouts + lf.layout_off, b.uni + lf.split_off,
              b.prop + lf.split_off, w, frac, order);
}

// ------------------------------------------------------------------ evaluator

// Counts of stage i for candidate s of work item w (composition unranking
// for exhaustive items is done per lane for its own stages).
__device__ __forceinline__ int cand_count(const Bufs& b, const Leaf& lf, const Work& w, int s,
                                          int i) {
  if (w.kind == 0) return (w.first + s == 0 ? b.uni : b.prop)[lf.split_off + i];
  if (w.kind == 1) {
    int q = (int)w.first + s;
    int mb = q >> 1, d = (q & 1) ? -1 : 1;
    int c = b.cur[lf.split_off + i];
    if (i == mb) c += d;
    if (i == mb + 1) c -= d;
    return c;
  }
  return 0;
}

template <int K>
__global__ void __launch_bounds__(256) k_eval(Bufs b, const Work* items, const int* n_items,
                                              int* next_item) {
  const int lane = threadIdx.x & 31;
  const bool gpipe = c_consts.schedule == 0;
  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(next_item, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= *n_items) return;
    const Work w = items[it];
    const Leaf lf = b.leaves[w.leaf];
    const int P = lf.P;
    const int M = lf.M;
    const int W2 = seg_width(P, K);
    const int seg = lane / W2;
    const int sl = lane % W2;
    const bool has_cand = seg < w.n;
    const LeafGroup* lg = b.lg + lf.lg_off;
    const uint8_t* slots = b.layouts + lf.layout_off;
    const double* hop = b.hop + lf.B_idx * c_consts.n_links;

    StageDur d[K];
    int wbound[K];
    bool valid = true, mem_ok = true;
    int cnt[K];
    if (w.kind == 2 && has_cand) {
      // unrank this candidate's composition up to my last stage
      long long rank = w.first + seg;
      int rem = c_consts.L;
      int last = min(P - 1, sl * K + K - 1);
      for (int j = 0; j <= last; ++j) {
        int v;
        if (j == P - 1) {
          v = rem;
        } else {
          int left = P - j;
          for (v = 1;; ++v) {
            long long cntv = binom(rem - v - 1, left - 2);
            if (rank < cntv) break;
            rank -= cntv;
          }
        }
        rem -= v;
        int r = j - sl * K;
        if (r >= 0 && r < K) cnt[r] = v;
      }
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int i = sl * K + r;
      wbound[r] = gpipe ? M : min(P - i, M);
      d[r].f = d[r].b = d[r].sf = d[r].sb = d[r].dps = 0.0;
      if (has_cand && i < P) {
        int c = w.kind == 2 ? cnt[r] : cand_count(b, lf, w, seg, i);
        if (c < 1) valid = false;
        else if (!stage_setup(c_consts, lf, lg, slots, hop, i, c, d[r])) mem_ok = false;
      }
    }
    const unsigned segmask = (W2 == 32 ? 0xffffffffu : ((1u << W2) - 1u)) << (seg * W2);
    const unsigned inv = __ballot_sync(0xffffffffu, !valid) & segmask;
    const unsigned mem = __ballot_sync(0xffffffffu, !mem_ok) & segmask;
    const bool run = has_cand && inv == 0 && mem == 0;

    StageState st[K];
#pragma unroll
    for (int r = 0; r < K; ++r) stage_init(st[r]);
    if (__any_sync(0xffffffffu, run)) {
      for (;;) {
        bool done = true;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int i = sl * K + r;
          if (run && i < P && !stage_done(st[r], M)) done = false;
        }
        if (__all_sync(0xffffffffu, done)) break;
        // previous-level neighbour state
        const double lchf = __shfl_up_sync(0xffffffffu, st[K - 1].chf, 1);
        const int lnf = __shfl_up_sync(0xffffffffu, st[K - 1].nf, 1);
        const double rchb = __shfl_down_sync(0xffffffffu, st[0].chb, 1);
        const int rnb = __shfl_down_sync(0xffffffffu, st[0].nb, 1);
        double pchf[K], pchb[K];
        int pnf[K], pnb[K];
#pragma unroll
        for (int r = 0; r < K; ++r) {
          pchf[r] = st[r].chf;
          pnf[r] = st[r].nf;
          pchb[r] = st[r].chb;
          pnb[r] = st[r].nb;
        }
        double dummy = 0.0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int i = sl * K + r;
          if (run && i < P) {
            const double l_chf = r == 0 ? lchf : pchf[r > 0 ? r - 1 : 0];
            const int l_nf = r == 0 ? lnf : pnf[r > 0 ? r - 1 : 0];
            const double r_chb = r == K - 1 ? rchb : pchb[r < K - 1 ? r + 1 : 0];
            const int r_nb = r == K - 1 ? rnb : pnb[r < K - 1 ? r + 1 : 0];
            stage_level(gpipe, i, P, M, wbound[r], d[r], st[r], l_chf, l_nf, r_chb, r_nb, dummy);
          }
        }
      }
    }
    // iteration = max(max over events, max_i(compute_end_i + dp_sync_i));
    // every per-stage/per-channel end sequence is non-decreasing, so the
    // maximum over events is the maximum of the final stage/channel times.
    double v = 0.0;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int i = sl * K + r;
      if (run && i < P) {
        v = dmax(v, st[r].free_t);
        v = dmax(v, st[r].chf);
        v = dmax(v, st[r].chb);
        v = dmax(v, st[r].free_t + d[r].dps);
      }
    }
    for (int off = W2 >> 1; off > 0; off >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (sl == 0 && has_cand) {
      double t = inv ? T_INVALID : (mem ? T_MEMORY : v);
      if (w.kind == 0) b.tseed[2 * w.leaf + (int)w.first + seg] = t;
      else if (w.kind == 1) b.nb[b.nb_off[w.leaf] + (int)w.first + seg] = t;
      else b.xbuf[w.out + seg] = t;
    }
  }
}

// ------------------------------------------------------------------ hill climb

__global__ void k_hill_init(Bufs b, const int* leaf_ids, int n, int uniform_only, int* active,
                            int* n_active) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int li = leaf_ids[k];
  const Leaf lf = b.leaves[li];
  HillState hs;
  hill_init(c_consts, lf, b.lg + lf.lg_off, b.layouts + lf.layout_off, b.uni + lf.split_off,
            b.prop + lf.split_off, b.tseed[2 * li], uniform_only ? -1.0 : b.tseed[2 * li + 1],
            b.cur + lf.split_off, b.best + lf.split_off, hs, uniform_only != 0);
  b.hs[li] = hs;
  if (hs.active) active[atomicAdd(n_active, 1)] = li;
}

// Work items for the neighbours of every active leaf, bucketed by K class.
__global__ void k_gen(Bufs b, const int* active, const int* n_active, Work* items, int cap,
                      int* n_items /*[4]*/) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *n_active) return;
  int li = active[k];
  const Leaf lf = b.leaves[li];
  int K = k_class(lf.P);
  int cls = K >= 4 ? 3 : K - 1;
  int cpw = 32 / seg_width(lf.P, K);
  int nslots = 2 * (lf.P - 1);
  int nit = (nslots + cpw - 1) / cpw;
  int base = atomicAdd(&n_items[cls], nit);
  Work* q = items + (size_t)cls * cap;
  for (int j = 0; j < nit; ++j) {
    Work w;
    w.leaf = li;
    w.kind = 1;
    w.first = j * cpw;
    w.n = min(cpw, nslots - j * cpw);
    w.out = 0;
    q[base + j] = w;
  }
}

__global__ void k_hill_step(Bufs b, const int* active, const int* n_active, int* next_active,
                            int* n_next) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *n_active) return;
  int li = active[k];
  const Leaf lf = b.leaves[li];
  HillState hs = b.hs[li];
  int delta[HP_MAX_STAGES];
  unsigned char old[2 * HP_MAX_STAGES];
  int tmp[HP_MAX_STAGES];
  for (int i = 0; i < lf.P; ++i) delta[i] = 0;
  hill_step(c_consts, lf, b.lg + lf.lg_off, b.layouts + lf.layout_off, b.cur + lf.split_off,
            b.uni + lf.split_off, b.prop + lf.split_off, b.best + lf.split_off,
            b.hist + b.hist_off[li], hs, b.nb + b.nb_off[li], delta, old, tmp);
  b.hs[li] = hs;
  if (hs.active) next_active[atomicAdd(n_next, 1)] = li;
}

// ------------------------------------------------------------------ exhaustive

// One thread per exhaustive leaf of the chunk: ranks [first, first+n) of the
// leaf have times at xbuf[out..]. Sequential in rank order with the exact
// comparator; state persists in hs/best across chunks.
struct ExhSpan {
  int leaf;
  int out;
  long long first;
  long long n;
};

__global__ void k_exh_reduce(Bufs b, const ExhSpan* spans, int n_spans) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_spans) return;
  const ExhSpan sp = spans[k];
  const Leaf lf = b.leaves[sp.leaf];
  const LeafGroup* lg = b.lg + lf.lg_off;
  const uint8_t* slots = b.layouts + lf.layout_off;
  HillState hs = b.hs[sp.leaf];
  int* best = b.best + lf.split_off;
  int comp[HP_MAX_STAGES];
  for (long long j = 0; j < sp.n; ++j) {
    double t = b.xbuf[sp.out + j];
    if (t < 0) {
      hs.pruned++;
      continue;
    }
    hs.simulated++;
    bool better = !hs.has_best || t < hs.best_time;
    if (!better && t == hs.best_time) {
      unrank_composition(sp.first + j, c_consts.L, lf.P, comp);
      better = cand_less(c_consts, t, lf, lg, slots, comp, hs.best_time, lf, lg, slots, best);
    }
    if (better) {
      hs.has_best = 1;
      hs.best_time = t;
      unrank_composition(sp.first + j, c_consts.L, lf.P, best);
    }
  }
  b.hs[sp.leaf] = hs;
}

// ------------------------------------------------------------------ final

// Block-wide exact argmin over leaf bests (time, pp, encoding). One block.
__global__ void k_final(Bufs b, int n_leaves, int* out_leaf, long long* counts) {
  __shared__ int s_best[1024];
  __shared__ long long s_sim[1024], s_pr[1024];
  int tid = threadIdx.x;
  int mine = -1;
  long long sim = 0, pr = 0;
  for (int li = tid; li < n_leaves; li += blockDim.x) {
    const HillState hs = b.hs[li];
    sim += hs.simulated;
    pr += hs.pruned;
    if (!hs.has_best) continue;
    if (mine < 0) {
      mine = li;
      continue;
    }
    const Leaf la = b.leaves[li], lb = b.leaves[mine];
    if (cand_less(c_consts, hs.best_time, la, b.lg + la.lg_off, b.layouts + la.layout_off,
                  b.best + la.split_off, b.hs[mine].best_time, lb, b.lg + lb.lg_off,
                  b.layouts + lb.layout_off, b.best + lb.split_off))
      mine = li;
  }
  s_best[tid] = mine;
  s_sim[tid] = sim;
  s_pr[tid] = pr;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (tid < s) {
      int a = s_best[tid], o = s_best[tid + s];
      if (o >= 0) {
        bool take = a < 0;
        if (!take) {
          const Leaf la = b.leaves[o], lb = b.leaves[a];
          take = cand_less(c_consts, b.hs[o].best_time, la, b.lg + la.lg_off,
                           b.layouts + la.layout_off, b.best + la.split_off, b.hs[a].best_time, lb,
                           b.lg + lb.lg_off, b.layouts + lb.layout_off, b.best + lb.split_off);
        }
        if (take) s_best[tid] = o;
      }
      s_sim[tid] += s_sim[tid + s];
      s_pr[tid] += s_pr[tid + s];
    }
    __syncthreads();
  }
  if (tid == 0) {
    *out_leaf = s_best[0];
    counts[0] = s_sim[0];
    counts[1] = s_pr[0];
  }
}

}  // namespace hpk

// ====================================================================== host

namespace hpd {

using namespace hpc;
using hpk::Work;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      return hph::Status{HP_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
    }                                                                             \
  } while (0)

template <typename T>
static hph::Status upload(Arena& a, const char* name, const std::vector<T>& v, T** out) {
  void* p = nullptr;
  hph::Status s = a.get(name, std::max<size_t>(1, v.size()) * sizeof(T), &p);
  if (!s.ok()) return s;
  if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, a.stream));
  *out = static_cast<T*>(p);
  return s;
}

template <typename T>
static hph::Status scratch(Arena& a, const char* name, size_t n, T** out) {
  void* p = nullptr;
  hph::Status s = a.get(name, std::max<size_t>(1, n) * sizeof(T), &p);
  *out = static_cast<T*>(p);
  return s;
}

static void launch_eval(int K, const hpk::Bufs& b, const Work* items, const int* n_items,
                        int* next, int grid, cudaStream_t st) {
  switch (K) {
    case 1: hpk::k_eval<1><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 2: hpk::k_eval<2><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 3: hpk::k_eval<3><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    default: hpk::k_eval<8><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
  }
}

hph::Status search_full(Arena& a, const hph::Problem& p, const std::vector<int>& my_leaves,
                        SearchOut& out) {
  cudaStream_t st = a.stream;
  const int G = static_cast<int>(p.groups.size());
  const int nL = static_cast<int>(my_leaves.size());
  Consts c;
  hph::fill_consts(p, c);
  CK(cudaMemcpyToSymbolAsync(hpk::c_consts, &c, sizeof c, 0, cudaMemcpyHostToDevice, st));

  // ---- host tables (split-independent, exact reference order)
  std::vector<Leaf> leaves(nL);
  std::vector<LeafGroup> lgs((size_t)nL * G);
  std::vector<int> hist_off(nL), nb_off(nL);
  std::vector<double> hop(p.mbs.size() * p.links.size());
  for (size_t bi = 0; bi < p.mbs.size(); ++bi)
    for (size_t l = 0; l < p.links.size(); ++l)
      hop[bi * p.links.size() + l] = hph::hop_time(p, (int)l, p.mbs[bi]);
  int split_total = 0, hist_total = 0, nb_total = 0;
  std::vector<int> hill_ids, exh_ids;
  for (int k = 0; k < nL; ++k) {
    const hph::LeafHost& h = p.leaves[my_leaves[k]];
    const hph::Task& t = p.tasks[h.task];
    Leaf& lf = leaves[k];
    lf.task = h.task;
    lf.P = t.pp;
    lf.M = static_cast<int>(h.M);
    lf.dp = h.dp;
    lf.B = h.B;
    lf.B_idx = h.B_idx;
    lf.layout_off = t.layout_off;
    lf.split_off = split_total;
    lf.lg_off = k * G;
    lf.mode = p.uniform_only ? 2 : (h.exhaustive ? 1 : 0);
    split_total += t.pp;
    for (int g = 0; g < G; ++g)
      lgs[(size_t)k * G + g] = hph::leaf_group(p, g, h.tp[g], h.B, h.dp, h.nodes[g]);
    hist_off[k] = hist_total;
    nb_off[k] = nb_total;
    if (lf.mode == 0) {
      hist_total += 4 * p.model.num_layers;
      nb_total += 2 * (t.pp - 1);
    }
    if (lf.mode == 1) exh_ids.push_back(k);
    else hill_ids.push_back(k);
  }

  hpk::Bufs b{};
  hph::Status s;
  Leaf* d_leaves;
  LeafGroup* d_lg;
  uint8_t* d_layouts;
  double* d_hop;
  int *d_hist_off, *d_nb_off;
  if (!(s = upload(a, "leaves", leaves, &d_leaves)).ok()) return s;
  if (!(s = upload(a, "lg", lgs, &d_lg)).ok()) return s;
  if (!(s = upload(a, "layouts", p.layouts, &d_layouts)).ok()) return s;
  if (!(s = upload(a, "hop", hop, &d_hop)).ok()) return s;
  if (!(s = upload(a, "hist_off", hist_off, &d_hist_off)).ok()) return s;
  if (!(s = upload(a, "nb_off", nb_off, &d_nb_off)).ok()) return s;
  b.leaves = d_leaves;
  b.lg = d_lg;
  b.layouts = d_layouts;
  b.hop = d_hop;
  b.hist_off = d_hist_off;
  b.nb_off = d_nb_off;
  if (!(s = scratch(a, "uni", split_total, &b.uni)).ok()) return s;
  if (!(s = scratch(a, "prop", split_total, &b.prop)).ok()) return s;
  if (!(s = scratch(a, "cur", split_total, &b.cur)).ok()) return s;
  if (!(s = scratch(a, "best", split_total, &b.best)).ok()) return s;
  if (!(s = scratch(a, "hist", hist_total, &b.hist)).ok()) return s;
  if (!(s = scratch(a, "tseed", 2 * (size_t)nL, &b.tseed)).ok()) return s;
  if (!(s = scratch(a, "nb", nb_total, &b.nb)).ok()) return s;
  if (!(s = scratch(a, "hs", nL, &b.hs)).ok()) return s;
  CK(cudaMemsetAsync(b.hs, 0, sizeof(HillState) * std::max(1, nL), st));

  int* d_ctr;  // [0..3] item counts per class, [4..7] next counters, [8] n_active, [9] n_next
  if (!(s = scratch(a, "ctr", 16, &d_ctr)).ok()) return s;
  const int grid = a.sm_count * 8;
  const int T = 128;

  // ---- seeds
  if (nL > 0) {
    hpk::k_seeds<<<(nL + T - 1) / T, T, 0, st>>>(b, nL);
    out.launches++;
  }

  // ---- seed evaluation (uniform + proportional of hill / uniform-only leaves)
  std::vector<std::vector<Work>> seedq(4);
  for (int k : hill_ids) {
    int K = hpk::k_class(leaves[k].P);
    int cls = K >= 4 ? 3 : K - 1;
    int cpw = 32 / hpk::seg_width(leaves[k].P, K);
    int n = p.uniform_only ? 1 : 2;
    if (cpw >= n) {
      seedq[cls].push_back(Work{k, 0, 0, n, 0});
    } else {
      // one candidate per work item
      seedq[cls].push_back(Work{k, 0, 0, 1, 0});
      if (n == 2) seedq[cls].push_back(Work{k, 0, 1, 1, 0});
    }
  }
  auto run_queues = [&](std::vector<std::vector<Work>>& qs, const char* tag) -> hph::Status {
    for (int cls = 0; cls < 4; ++cls) {
      if (qs[cls].empty()) continue;
      Work* d_items;
      std::string nm = std::string(tag) + std::to_string(cls);
      hph::Status s2 = upload(a, nm.c_str(), qs[cls], &d_items);
      if (!s2.ok()) return s2;
      int cnt[2] = {static_cast<int>(qs[cls].size()), 0};
      CK(cudaMemcpyAsync(d_ctr + 12, cnt, sizeof cnt, cudaMemcpyHostToDevice, st));
      launch_eval(cls == 3 ? 8 : cls + 1, b, d_items, d_ctr + 12, d_ctr + 13, grid, st);
      out.launches++;
      CK(cudaStreamSynchronize(st));  // host count buffer reused per queue
    }
    return hph::Status{};
  };
  if (!(s = run_queues(seedq, "seedq")).ok()) return s;

  // ---- hill climb
  int *d_ids, *d_act0, *d_act1;
  std::vector<int> ids(hill_ids.begin(), hill_ids.end());
  if (!(s = upload(a, "hill_ids", ids, &d_ids)).ok()) return s;
  if (!(s = scratch(a, "act0", ids.size(), &d_act0)).ok()) return s;
  if (!(s = scratch(a, "act1", ids.size(), &d_act1)).ok()) return s;
  size_t cap = 0;
  for (int k : hill_ids) cap = std::max<size_t>(cap, 2 * leaves[k].P);
  cap = std::max<size_t>(1, cap * hill_ids.size());
  Work* d_items;
  if (!(s = scratch(a, "items", 4 * cap, &d_items)).ok()) return s;
  CK(cudaMemsetAsync(d_ctr, 0, 16 * sizeof(int), st));
  if (!hill_ids.empty()) {
    hpk::k_hill_init<<<((int)ids.size() + T - 1) / T, T, 0, st>>>(b, d_ids, (int)ids.size(),
                                                                   p.uniform_only ? 1 : 0, d_act0,
                                                                   d_ctr + 8);
    out.launches++;
  }
  int n_active = 0;
  CK(cudaMemcpyAsync(&n_active, d_ctr + 8, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int iter = 0;
  while (n_active > 0) {
    CK(cudaMemsetAsync(d_ctr, 0, 8 * sizeof(int), st));
    CK(cudaMemsetAsync(d_ctr + 9, 0, sizeof(int), st));
    hpk::k_gen<<<(n_active + T - 1) / T, T, 0, st>>>(b, d_act0, d_ctr + 8, d_items, (int)cap, d_ctr);
    out.launches++;
    for (int cls = 0; cls < 4; ++cls) {
      launch_eval(cls == 3 ? 8 : cls + 1, b, d_items + (size_t)cls * cap, d_ctr + cls, d_ctr + 4 + cls,
                  grid, st);
      out.launches++;
    }
    hpk::k_hill_step<<<(n_active + T - 1) / T, T, 0, st>>>(b, d_act0, d_ctr + 8, d_act1, d_ctr + 9);
    out.launches++;
    CK(cudaMemcpyAsync(d_ctr + 8, d_ctr + 9, sizeof(int), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(&n_active, d_ctr + 9, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::swap(d_act0, d_act1);
    ++iter;
  }
  out.hill_iterations = iter;

  // ---- exhaustive leaves, in chunks of candidates
  if (!exh_ids.empty()) {
    const long long kChunk = 1 << 24;
    double* d_x;
    if (!(s = scratch(a, "xbuf", kChunk, &d_x)).ok()) return s;
    b.xbuf = d_x;
    size_t e = 0;
    long long pos = 0;  // rank position within exh_ids[e]
    while (e < exh_ids.size()) {
      std::vector<std::vector<Work>> q(4);
      std::vector<hpk::ExhSpan> spans;
      long long used = 0;
      while (e < exh_ids.size() && used < kChunk) {
        int k = exh_ids[e];
        const Leaf& lf = leaves[k];
        long long total = p.leaves[my_leaves[k]].n_splits;
        long long take = std::min(total - pos, kChunk - used);
        int K = hpk::k_class(lf.P);
        int cls = K >= 4 ? 3 : K - 1;
        int cpw = 32 / hpk::seg_width(lf.P, K);
        for (long long j = 0; j < take; j += cpw)
          q[cls].push_back(Work{k, 2, pos + j, (int)std::min<long long>(cpw, take - j), (int)(used + j)});
        spans.push_back(hpk::ExhSpan{k, (int)used, pos, take});
        used += take;
        pos += take;
        if (pos == total) {
          ++e;
          pos = 0;
        }
      }
      if (!(s = run_queues(q, "exhq")).ok()) return s;
      hpk::ExhSpan* d_spans;
      if (!(s = upload(a, "spans", spans, &d_spans)).ok()) return s;
      hpk::k_exh_reduce<<<((int)spans.size() + T - 1) / T, T, 0, st>>>(b, d_spans, (int)spans.size());
      out.launches++;
      CK(cudaStreamSynchronize(st));
    }
  }

  // ---- final argmin
  int* d_best_leaf;
  long long* d_counts;
  if (!(s = scratch(a, "best_leaf", 1, &d_best_leaf)).ok()) return s;
  if (!(s = scratch(a, "counts", 2, &d_counts)).ok()) return s;
  hpk::k_final<<<1, 1024, 0, st>>>(b, nL, d_best_leaf, d_counts);
  out.launches++;
  CK(cudaGetLastError());
  int best_leaf = -1;
  long long counts[2];
  CK(cudaMemcpyAsync(&best_leaf, d_best_leaf, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(counts, d_counts, sizeof counts, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out.simulated = counts[0];
  out.pruned = counts[1];
  out.has_best = best_leaf >= 0;
  if (out.has_best) {
    HillState hs;
    const Leaf& lf = leaves[best_leaf];
    out.best_split.resize(lf.P);
    CK(cudaMemcpy(&hs, b.hs + best_leaf, sizeof hs, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out.best_split.data(), b.best + lf.split_off, sizeof(int) * lf.P,
                  cudaMemcpyDeviceToHost));
    out.best_time = hs.best_time;
    out.best_leaf = my_leaves[best_leaf];
  }
  return hph::Status{};
}

}  // namespace hpd

namespace hpd {

// hp_evaluate_plans: each plan becomes a one-candidate pseudo-leaf whose
// LeafGroup rows are per stage (stage tp / dp / nodes may differ), evaluated
// by the same warp-segment kernel. evaluate_plan_unchecked has no memory
// gate (mode 3).
hph::Status evaluate_plans(Arena& a, const hph::Problem& p, const hp_plan* plans, int n,
                           double* out_times) {
  if (n == 0) return hph::Status{};
  cudaStream_t st = a.stream;
  Consts c;
  hph::fill_consts(p, c);
  c.n_B = n;
  CK(cudaMemcpyToSymbolAsync(hpk::c_consts, &c, sizeof c, 0, cudaMemcpyHostToDevice, st));
  std::vector<Leaf> leaves(n);
  std::vector<LeafGroup> lgs;
  std::vector<uint8_t> layouts;
  std::vector<int> splits;
  std::vector<double> hop((size_t)n * p.links.size());
  std::vector<std::vector<Work>> q(4);
  for (int k = 0; k < n; ++k) {
    const hp_plan& pl = plans[k];
    const int P = pl.n_stages;
    int64_t B = pl.micro_batch_size > 0 ? pl.micro_batch_size : p.train.micro_batch_size;
    Leaf& lf = leaves[k];
    lf.task = -1;
    lf.P = P;
    lf.M = static_cast<int>(pl.micro_batches_per_dp_replica);
    lf.dp = pl.stages[0].dp_degree;
    lf.B = B;
    lf.B_idx = k;
    lf.layout_off = static_cast<int>(layouts.size());
    lf.split_off = static_cast<int>(splits.size());
    lf.lg_off = static_cast<int>(lgs.size());
    lf.mode = 3;
    for (size_t l = 0; l < p.links.size(); ++l) hop[(size_t)k * p.links.size() + l] = hph::hop_time(p, (int)l, B);
    for (int i = 0; i < P; ++i) {
      const hp_stage& s = pl.stages[i];
      layouts.push_back(static_cast<uint8_t>(i));
      splits.push_back(s.layer_end - s.layer_begin);
      lgs.push_back(hph::leaf_group(p, s.group, s.tp_degree, B, s.dp_degree, s.nodes_used));
    }
    int K = hpk::k_class(P);
    q[K >= 4 ? 3 : K - 1].push_back(Work{k, 0, 0, 1, 0});
  }
  hpk::Bufs b{};
  hph::Status s;
  Leaf* d_leaves;
  LeafGroup* d_lg;
  uint8_t* d_layouts;
  double* d_hop;
  int* d_split;
  if (!(s = upload(a, "e_leaves", leaves, &d_leaves)).ok()) return s;
  if (!(s = upload(a, "e_lg", lgs, &d_lg)).ok()) return s;
  if (!(s = upload(a, "e_layouts", layouts, &d_layouts)).ok()) return s;
  if (!(s = upload(a, "e_hop", hop, &d_hop)).ok()) return s;
  if (!(s = upload(a, "e_split", splits, &d_split)).ok()) return s;
  b.leaves = d_leaves;
  b.lg = d_lg;
  b.layouts = d_layouts;
  b.hop = d_hop;
  b.uni = d_split;
  if (!(s = scratch(a, "e_tseed", 2 * (size_t)n, &b.tseed)).ok()) return s;
  int* d_ctr;
  if (!(s = scratch(a, "e_ctr", 2, &d_ctr)).ok()) return s;
  for (int cls = 0; cls < 4; ++cls) {
    if (q[cls].empty()) continue;
    Work* d_items;
    std::string nm = "e_q" + std::to_string(cls);
    if (!(s = upload(a, nm.c_str(), q[cls], &d_items)).ok()) return s;
    int cnt[2] = {static_cast<int>(q[cls].size()), 0};
    CK(cudaMemcpyAsync(d_ctr, cnt, sizeof cnt, cudaMemcpyHostToDevice, st));
    launch_eval(cls == 3 ? 8 : cls + 1, b, d_items, d_ctr, d_ctr + 1, a.sm_count * 8, st);
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaGetLastError());
  std::vector<double> t(2 * (size_t)n);
  CK(cudaMemcpyAsync(t.data(), b.tseed, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int k = 0; k < n; ++k) out_times[k] = t[2 * (size_t)k];
  return hph::Status{};
}

}  // namespace hpd
