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
//   k_hill_init / k_async_seed / k_hill_async
//                  steepest-descent layer-split search (planner.cpp:461-489)
//                  with memo-equivalent counting (hp_search_core.cuh); every
//                  leaf advances independently through a device work queue.
//   k_default      time-bound-pruned (default) mode: one warp per task,
//                  speculative batch evaluation + in-order replay of the
//                  incumbent (planner.cpp:519-534).
//   k_exh_reduce   per-leaf reduction of exhaustively enumerated splits.
//   k_final        exact better_than argmin over leaf bests.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <type_traits>
#include <unordered_map>
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
  const long long* ids;  // optional: candidate s is ids[first + s]
};

__device__ __forceinline__ long long cand_id(const Work& w, int s) {
  // ids may have been written by another SM (a leaf's step): read past L1
  return w.ids ? __ldcg(w.ids + w.first + s) : w.first + s;
}

// Search-log sink (HP_FLAG_LOG). Kernels append, per decided batch, the
// iteration times of the candidates the reference simulates, in the
// reference's visit order, as segments keyed (stream, seq); the host replays
// the reference's control flow over them (hp_log.cpp). Capacity overflow is
// detected from the counters, which keep counting past the capacity.
struct LogSeg {
  int key;             // shard leaf position (full mode) or shard task position (default)
  int seq;             // hill step (full mode) or per-task batch counter (default)
  long long off;       // first value in vals
  long long n;
};

struct LogSink {
  double* vals = nullptr;
  LogSeg* segs = nullptr;
  unsigned long long* ctr = nullptr;  // [0] values, [1] segments
  unsigned long long val_cap = 0, seg_cap = 0;
  double* exh = nullptr;              // full mode: time per bounded rank of exhaustive leaves
  const long long* exh_off = nullptr;
};

// Reserves n values for segment (key, seq); returns their offset, or -1 when
// n == 0 or the sink is full (the caller then writes nothing).
__device__ inline long long log_reserve(const LogSink& s, int key, int seq, int n) {
  if (n <= 0) return -1;
  const unsigned long long off = atomicAdd(s.ctr, (unsigned long long)n);
  const unsigned long long k = atomicAdd(s.ctr + 1, 1ULL);
  if (off + n > s.val_cap || k >= s.seg_cap) return -1;
  s.segs[k] = LogSeg{key, seq, (long long)off, (long long)n};
  return (long long)off;
}

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
  unsigned long long* ops;  // algorithmic FP64 add/max ops of simulated candidates
  // exhaustive regime: per-leaf bounded-composition tables (exh_table) and
  // memory caps; ranks of kind-2 work items index the bounded compositions
  unsigned long long* trace;  // optional (HP_DEBUG_TRACE): [0] = count, then (ns, event) records
  int trace_items;            // HP_DEBUG_TRACE_ITEMS: also item / screen / push events
  const long long* etbl;
  const int* etbl_off;
  const int* ecap;
  LogSink log;
  // neighbour screen (nb_screen): per-stage bound terms of each leaf's
  // current split, and the surviving neighbour slots of its current step
  StageLB* lbs;
  StageNb* lbn;
  long long* nb_ids;
  // memo distances of the climb: memo_d[hist_off + t] = ||S_k - S_t||_1
  // between the current point k and path point t (prefix-sum space)
  int* memo_d;
  int nb_rows;  // kind-1 items are screened neighbours with StageLB/StageNb rows (full-mode climb)
  int n_lg;     // LeafGroup rows / hop entries uploaded (host-side sizes for table staging)
  int n_hop;
};

// count of bounded compositions continuing with part value v at position j
__device__ __forceinline__ long long exh_count(const Bufs& b, const Leaf& lf, int leaf, int j, int rem,
                                               int v) {
  if (b.etbl == nullptr) return binom(rem - v - 1, lf.P - j - 2);  // unbounded (default mode)
  const int W = c_consts.L + 1;
  const int cap = b.ecap[lf.split_off + j];
  if (v > cap || rem - v < 0) return 0;
  return b.etbl[b.etbl_off[leaf] + (j + 1) * W + rem - v];
}

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

// Evaluator classes. 0..3: fast 1F1B kernel (closed-form level schedule,
// needs M >= P) with K = 2,4,6,8 stages per lane; 4..7: generic
// counter-driven kernel (GPipe, M < P) with K = 1,2,3,8.
constexpr int NCLS = 8;

__host__ __device__ inline int class_K(int cls) {
  return cls < 4 ? 2 * (cls + 1) : (cls == 7 ? 8 : cls - 3);
}

// Lanes per candidate.
__host__ __device__ inline int class_width(int cls, int P) {
  int K = class_K(cls);
  return cls < 4 ? (P + K - 1) / K : seg_width(P, K);
}

// Fast-kernel K maximising throughput: lane utilisation P*floor(32/W)/(32K),
// W = ceil(P/K), times the core loop's rate at K stages per lane with the
// climb kernel's 8 warps per SM (tools/micro/corebench: 6.4, 10.0, 11.5,
// 11.2 T ops/s for K = 2..8 — more stages per lane is more independent FP64
// work per warp, which at this occupancy hides the level's latency).
#ifndef HP_FAST_KMAX
#define HP_FAST_KMAX 8  // tuning: largest K chosen when a smaller one fits (K = 8 needs the most registers)
#endif
__host__ __device__ inline int fast_K(int P) {
  const double rate[4] = {6.4, 10.0, 11.5, 11.2};
  int bestK = 8;
  double bestU = -1.0;
  for (int K = 2; K <= HP_FAST_KMAX; K += 2) {
    int W = (P + K - 1) / K;
    if (W > 32) continue;
    double u = (double)P * (32 / W) / (32.0 * K) * rate[K / 2 - 1];
    if (u > bestU + 1e-12) {
      bestU = u;
      bestK = K;
    }
  }
  return bestK;
}

__host__ __device__ inline int eval_class(int P, int M, bool gpipe) {
  if (!gpipe && M >= P && P <= 256) return fast_K(P) / 2 - 1;
  int K = k_class(P);
  return 4 + (K >= 4 ? 3 : K - 1);
}

__host__ __device__ inline int class_cpw(int cls, int P) { return 32 / class_width(cls, P); }

// ------------------------------------------------------------------ table staging
//
// The split-independent cost tables of a search — LeafGroup rows (one per
// distinct (dp, B, tp, nodes) tuple, ~600 for C3) and the hop table — are
// staged once per block into shared memory with TMA bulk copies
// (cp.async.bulk global -> shared, completion counted on an mbarrier), so
// every stage_setup of the climb and default-mode kernels (screen rows,
// seeds, gates, neighbour durations) reads them a few cycles away instead
// of through L1/L2. `stage_bytes` is 0 when they do not fit (the kernels
// then read global memory).
struct StagedTables {
  unsigned lg_bytes;   // LeafGroup rows, padded to 16 bytes
  unsigned hop_bytes;  // hop table, padded to 16 bytes
};

__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :
               : "r"(dst), "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// Whole block. Returns b with lg / hop pointing at the shared copies.
__device__ inline Bufs stage_tables(const Bufs& b, const StagedTables& t, unsigned char* smem,
                                    unsigned long long* bar) {
  if (t.lg_bytes == 0) return b;
  const unsigned sbar = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  const unsigned sdst = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" : : "r"(sbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" : : : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :
                 : "r"(sbar), "r"(t.lg_bytes + t.hop_bytes)
                 : "memory");
    constexpr unsigned kChunk = 32768;
    for (unsigned off = 0; off < t.lg_bytes; off += kChunk)
      bulk_g2s(sdst + off, reinterpret_cast<const unsigned char*>(b.lg) + off, min(kChunk, t.lg_bytes - off),
               sbar);
    bulk_g2s(sdst + t.lg_bytes, b.hop, t.hop_bytes, sbar);
  }
  __syncthreads();
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra WAIT_%=;\n\t}"
      :
      : "r"(sbar)
      : "memory");
  Bufs s = b;
  s.lg = reinterpret_cast<const LeafGroup*>(smem);
  s.hop = reinterpret_cast<const double*>(smem + t.lg_bytes);
  return s;
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
  if (w.kind == 0) return (cand_id(w, s) == 0 ? b.uni : b.prop)[lf.split_off + i];
  if (w.kind == 1) {
    int q = (int)cand_id(w, s);
    int mb = q >> 1, d = (q & 1) ? -1 : 1;
    int c = __ldcg(b.cur + lf.split_off + i);  // written by another SM's hill step
    if (i == mb) c += d;
    if (i == mb + 1) c -= d;
    return c;
  }
  return 0;
}

// Generic evaluator (GPipe, M < P): counter-driven readiness per level.
template <int K>
__device__ __forceinline__ void eval_item_generic(const Bufs& b, const Work& w, const int lane) {
  {
    const Leaf lf = b.leaves[w.leaf];
    const bool gpipe = lf.sched == 0;
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
      long long rank = cand_id(w, seg);
      int rem = c_consts.L;
      int last = min(P - 1, sl * K + K - 1);
      for (int j = 0; j <= last; ++j) {
        int v;
        if (j == P - 1) {
          v = rem;
        } else {
          for (v = 1;; ++v) {
            long long cntv = exh_count(b, lf, w.leaf, j, rem, v);
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
    if (gpipe && __any_sync(0xffffffffu, run)) {
      // GPipe in closed form: the unit-time ASAP level of F(i,m) is i+m and
      // that of B(i,j) is 2P-2-i+M+j (F(i,m) needs F(i-1,m)'s send, one
      // level earlier; B(P-1,0) follows the last forward of the last stage;
      // B(i,j) needs B(i+1,j)'s send). So all forwards run in levels
      // [0, M+P-2] and all backwards in [M+P-1, 2M+2P-3]: a forward
      // wavefront (stage i active in [i, i+M-1]) and a backward one (stage i
      // active in [P-1-i, P-2-i+M] of the second phase), each stage reading
      // its neighbour's channel from the previous level (single slot, as in
      // the counter-driven path below) — no counters, no readiness tests.
      const int LV = M + P - 1;
      for (int t = 0; t < LV; ++t) {
        const double lchf = __shfl_up_sync(0xffffffffu, st[K - 1].chf, 1);
#pragma unroll
        for (int r = K - 1; r >= 0; --r) {  // descending: chf[r-1] is still the previous level's
          const int i = sl * K + r;
          const double recv = i == 0 ? 0.0 : (r == 0 ? lchf : st[r > 0 ? r - 1 : 0].chf);
          const double nfr = dmax(st[r].free_t, recv) + d[r].f;   // sim.cpp:106-121
          const double nch = dmax(nfr, st[r].chf) + d[r].sf;      // sim.cpp:125-134
          if (run && i < P && t >= i && t <= i + M - 1) {
            st[r].free_t = nfr;
            if (i < P - 1) st[r].chf = nch;
          }
        }
      }
      for (int t = 0; t < LV; ++t) {
        const double rchb = __shfl_down_sync(0xffffffffu, st[0].chb, 1);
#pragma unroll
        for (int r = 0; r < K; ++r) {  // ascending: chb[r+1] is still the previous level's
          const int i = sl * K + r;
          const double recv = i == P - 1 ? 0.0 : (r == K - 1 ? rchb : st[r < K - 1 ? r + 1 : 0].chb);
          const double nfr = dmax(st[r].free_t, recv) + d[r].b;
          const double nch = dmax(nfr, st[r].chb) + d[r].sb;      // sim.cpp:135-145
          if (run && i < P && t >= P - 1 - i && t <= P - 2 - i + M) {
            st[r].free_t = nfr;
            if (i > 0) st[r].chb = nch;
          }
        }
      }
    } else if (__any_sync(0xffffffffu, run)) {
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
      if (w.kind == 0) b.tseed[2 * w.leaf + (int)cand_id(w, seg)] = t;
      else if (w.kind == 1) b.nb[b.nb_off[w.leaf] + (int)cand_id(w, seg)] = t;
      else b.xbuf[w.out + seg] = t;
      if (run && b.ops) {
        atomicAdd(b.ops, (unsigned long long)(8LL * P * M - 4LL * M));
        atomicAdd(b.ops + 1, 1ULL);
      }
    }
  }
}

// Fast 1F1B evaluator (M >= P). The unit-time ASAP level of every op has a
// closed form (checked against the counter-driven schedule in tests):
//   F(i,m) at level i+m (m < P-i, warm-up) or 2m+i (m >= P-i),
//   B(i,j) at level 2P-1-i+2j,   T = 2(M+P-1) levels.
// With an even number K of consecutive stages per lane, the F/B type of
// local stage r in the steady state depends only on the parity of t - r, so
// the whole warp follows one instruction stream (no divergence) and only the
// warm-up/cool-down windows are predicated. Segments are packed at exact
// width W = ceil(P/K) (floor(32/W) candidates per warp).
// HP_DEBUG_TRACE_ITEMS cycle records from inside the evaluator (ev 5: core
// loop cycles, ev 6: whole item cycles; the timestamp slot holds the count,
// aux = 1 when the core ran without channel maxima).
__device__ void trace_cycles(const Bufs& b, int ev, int li, int P, int M, unsigned aux, long long cyc) {
  unsigned long long k = atomicAdd(b.trace, 1ULL);
  if (k < (1ULL << 22)) {
    b.trace[1 + 2 * k] = (unsigned long long)cyc;
    b.trace[2 + 2 * k] = ((unsigned long long)ev << 59) | ((unsigned long long)(P & 0xff) << 48) |
                         ((unsigned long long)(M & 0xffff) << 32) | ((unsigned long long)(aux & 0xfff) << 20) |
                         (unsigned)(li & 0xfffff);
  }
}

// Core-loop level pairs between early-abort checks of a screened neighbour.
// The check (per stage frontier + remaining work + the backward drain, with
// two segment scans) costs more than the levels it saves on C3: it runs only
// on items longer than 2 x 4096 levels (M > ~4000).
#ifndef HP_ABORT_CODE
#define HP_ABORT_CODE 0  // 1 compiles the early-abort check in (C3, 1 GPU: 219-222 ms with it, 212-218 without)
#endif
#ifndef HP_UNROLL_CORE
#define HP_UNROLL_CORE 2  // tuning: level-pair unroll of the K != 4 core loops
#endif
constexpr int kUnrollCore = HP_UNROLL_CORE;
#ifndef HP_UNROLL_K4
#define HP_UNROLL_K4 4  // tuning: level-pair unroll of the K = 4 (latency) core loop
// (lone P = 96 climbs, C3:96: 1 -> 89.2 ms, 2 -> 81.0, 4 -> 77.3, 8 -> 75.6,
// 12/16 -> 74.8; the C3 sweep is ~1 % slower from 8 up: kept at 4)
#endif
constexpr int kUnrollK4 = HP_UNROLL_K4;
#ifndef HP_ABORT_PAIRS
#define HP_ABORT_PAIRS 4096  // tuning (C3, 1 GPU: 64 -> 236-249 ms, 128 -> 226-234, 512 -> 218-226, 4096 -> 215-219)
#endif
constexpr int kAbortPairs = HP_ABORT_PAIRS;

template <int K>
__device__ __forceinline__ void eval_item_fast(const Bufs& b, const Work& w, const int lane) {
  const Leaf lf = b.leaves[w.leaf];
  const int P = lf.P;
  const int M = lf.M;
  const int W = (P + K - 1) / K;
  const int cpw = 32 / W;
  const int seg = lane / W;
  const int sl = lane - seg * W;
  const bool has_cand = seg < cpw && seg < w.n;
  const LeafGroup* lg = b.lg + lf.lg_off;
  const uint8_t* slots = b.layouts + lf.layout_off;
  const double* hop = b.hop + lf.B_idx * c_consts.n_links;
  const double NEG = -__longlong_as_double(0x7ff0000000000000LL) * 1.0;  // -inf

  // per stage: durations and forward hop; the backward hop of stage i is
  // the forward hop of stage i-1 (same link and volume, evaluate.cpp:59-62)
  double f[K], bw[K], sf[K];
  bool valid = true, mem_ok = true;
  int cnt[K];
  if (w.kind == 2 && has_cand) {
    long long rank = cand_id(w, seg);
    int rem = c_consts.L;
    int last = min(P - 1, sl * K + K - 1);
    for (int j = 0; j <= last; ++j) {
      int v;
      if (j == P - 1) {
        v = rem;
      } else {
        for (v = 1;; ++v) {
          long long cntv = exh_count(b, lf, w.leaf, j, rem, v);
          if (rank < cntv) break;
          rank -= cntv;
        }
      }
      rem -= v;
      int r = j - sl * K;
      if (r >= 0 && r < K) cnt[r] = v;
    }
  }
  double dps[K];
  if (w.kind == 1 && b.nb_rows) {
    // screened neighbour (screen_neighbours): feasible, and its stage rows
    // are the current split's (StageLB) except the two the move changes
    // (StageNb at count -1 / +1)
    const int q = has_cand ? (int)cand_id(w, seg) : 0;
    const int mb = q >> 1, k0 = (q & 1) ? 0 : 1;
    const StageLB* rl = b.lbs + lf.split_off;
    const StageNb* rn = b.lbn + lf.split_off;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int i = sl * K + r;
      f[r] = bw[r] = NEG;
      sf[r] = 0.0;
      dps[r] = 0.0;
      if (has_cand && i < P) {
        if (i == mb || i == mb + 1) {
          const int k = i == mb ? k0 : 1 - k0;
          f[r] = __ldcg(&rn[i].f[k]);
          bw[r] = __ldcg(&rn[i].b[k]);
          dps[r] = __ldcg(&rn[i].dps[k]);
        } else {
          f[r] = __ldcg(&rl[i].f);
          bw[r] = __ldcg(&rl[i].b);
          dps[r] = __ldcg(&rl[i].dps);
        }
        sf[r] = i == P - 1 ? NEG : __ldcg(&rl[i].sf);
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int i = sl * K + r;
      f[r] = bw[r] = NEG;
      sf[r] = 0.0;
      dps[r] = 0.0;
      if (has_cand && i < P) {
        int c = w.kind == 2 ? cnt[r] : cand_count(b, lf, w, seg, i);
        StageDur d;
        if (c < 1) {
          valid = false;
        } else {
          if (!stage_setup(c_consts, lf, lg, slots, hop, i, c, d)) mem_ok = false;
          f[r] = d.f;
          bw[r] = d.b;
          dps[r] = d.dps;
          // The last stage sends no activations forward and stage 0 no
          // gradients backward (sim.cpp:127,137): a -inf hop keeps those
          // channels at -inf, which doubles as the "no dependency" operand for
          // the neighbouring segment / padding lanes (max(x, -inf) = x).
          sf[r] = i == P - 1 ? NEG : d.sf;
        }
      }
    }
  }
  const unsigned segmask = (W == 32 ? 0xffffffffu : ((1u << W) - 1u)) << (seg * W);
  const unsigned inv = __ballot_sync(0xffffffffu, !valid) & segmask;
  const unsigned mem = __ballot_sync(0xffffffffu, !mem_ok) & segmask;
  const bool run = has_cand && inv == 0 && mem == 0;

  // Lanes that do not simulate (padding, idle or pruned segments) hold -inf
  // everywhere, so every exchange across a segment boundary reads -inf.
  double fr[K], chf[K], chb[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = sl * K + r;
    const bool real = run && i < P;
    if (!real) {
      f[r] = bw[r] = NEG;
      sf[r] = 0.0;
    }
    fr[r] = real ? 0.0 : NEG;
    chf[r] = (real && i != P - 1) ? 0.0 : NEG;
    chb[r] = (real && i != 0) ? 0.0 : NEG;
  }
  const int src_l = (lane + 31) & 31;   // rotate: lane 0 reads lane 31 (-inf)
  const int src_r = (lane + 1) & 31;
  // backward hop of the lane's first stage; stage 0 sends no gradient (-inf)
  const double sb_in = __shfl_sync(0xffffffffu, sf[K - 1], src_l);
  const double sb0 = sl == 0 ? NEG : sb_in;
  // early-abort limit of a screened neighbour: the current point's time
  const double lim = (w.kind == 1 && b.nb_rows) ? __ldcg(&b.hs[w.leaf].cur_time) * (1.0 + kScreenMargin)
                                                : __builtin_huge_val();
  bool dead = false;
  int dead_t = 0;
  const bool tr = b.trace && b.trace_items && lane == 0 &&
                  ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) % b.trace_items == 0;
  const long long c_start = tr ? clock64() : 0;
  long long c_core0 = 0, c_core1 = 0;
  bool tr_noch = false;
  if (__any_sync(0xffffffffu, run)) {
    // ---- warm-up, levels 0..P-1: stage i runs F(i, t-i) once t >= i
    for (int t = 0; t < P; ++t) {
      const double lchf = __shfl_sync(0xffffffffu, chf[K - 1], src_l);
#pragma unroll
      for (int r = K - 1; r >= 0; --r) {  // descending: read chf[r-1] before it moves
        const int i = sl * K + r;
        const double recv = r == 0 ? lchf : chf[r > 0 ? r - 1 : 0];
        const double nfr = dmax(fr[r], recv) + f[r];
        const double nch = dmax(nfr, chf[r]) + sf[r];
        if (i <= t) {
          fr[r] = nfr;
          chf[r] = nch;
        }
      }
    }
    const int T = 2 * (M + P - 1);
    const int core_lo = 2 * P, core_hi = 2 * M - 2;  // every stage busy
    // One level of parity PAR after the warm-up: stage r runs F iff
    // (PAR - r) is even (i = sl*K + r with K even), B otherwise; adjacent
    // stages always run opposite ops, so nothing needs a snapshot. PRED
    // levels (transition and cool-down windows) gate each op on its closed
    // form window with selects; core levels run every op unconditionally.
    // MODE 0: every op as simulate() does it; 1: the same and checks that no
    // send waits for its channel (base_ok); 2: channel maxima dropped (see
    // the core loop below).
    bool base_ok = true;
    // Cross-lane operands of the next even level (see `level`): the left
    // neighbour's last forward channel and the right neighbour's first
    // backward channel.
    double xl = __shfl_sync(0xffffffffu, chf[K - 1], src_l);
    double xr = __shfl_sync(0xffffffffu, chb[0], src_r);
    auto level = [&](auto par_tag, auto pred_tag, auto mode_tag, int t) {
      constexpr int PAR = decltype(par_tag)::value;
      constexpr bool PRED = decltype(pred_tag)::value;
      constexpr int MODE = decltype(mode_tag)::value;
      const int u0 = t + sl * K;  // t + i - r
      const int v0 = t - sl * K;  // t - i + r
      auto op = [&](int r) {
        if (((PAR - r) & 1) == 0) {
          const double recv = r == 0 ? xl : chf[r > 0 ? r - 1 : 0];
          const double nfr = dmax(fr[r], recv) + f[r];
          if (MODE == 1) base_ok = base_ok && !(chf[r] > nfr);
          const double nch = (MODE == 2 ? nfr : dmax(nfr, chf[r])) + sf[r];
          if (PRED) {
            // F(i,m) at level 2m+i: 2P-i <= t <= 2M-2+i
            const bool act = (u0 + r >= 2 * P) && (v0 - r <= 2 * M - 2);
            fr[r] = act ? nfr : fr[r];
            chf[r] = act ? nch : chf[r];
          } else {
            fr[r] = nfr;
            chf[r] = nch;
          }
        } else {
          const double recv = r == K - 1 ? xr : chb[r < K - 1 ? r + 1 : 0];
          const double nfr = dmax(fr[r], recv) + bw[r];
          if (MODE == 1) base_ok = base_ok && !(chb[r] > nfr);
          const double nch = (MODE == 2 ? nfr : dmax(nfr, chb[r])) + (r == 0 ? sb0 : sf[r > 0 ? r - 1 : 0]);
          if (PRED) {
            // B(i,j) at level 2P-1-i+2j: 2P-1-i <= t <= 2M+2P-3-i
            const bool act = (u0 + r >= 2 * P - 1) && (u0 + r <= 2 * M + 2 * P - 3);
            fr[r] = act ? nfr : fr[r];
            chb[r] = act ? nch : chb[r];
          } else {
            fr[r] = nfr;
            chb[r] = nch;
          }
        }
      };
      // K is even: at odd levels a lane's first stage runs a backward and
      // its last a forward, both fed by the lane's own stages, and they
      // produce exactly what the neighbours need at the next (even) level.
      // So odd levels compute those two stages first and send their channel
      // ends right away — the exchange overlaps the interior stages — and
      // even levels read them (xl, xr) without exchanging.
      if (PAR == 1) {
        op(0);
        op(K - 1);
        xl = __shfl_sync(0xffffffffu, chf[K - 1], src_l);
        xr = __shfl_sync(0xffffffffu, chb[0], src_r);
#pragma unroll
        for (int r = 1; r < K - 1; ++r) op(r);
      } else {
#pragma unroll
        for (int r = 0; r < K; ++r) op(r);
      }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using PT = std::true_type;
    using PF = std::false_type;
    using M0 = std::integral_constant<int, 0>;
    using M1 = std::integral_constant<int, 1>;
    using M2 = std::integral_constant<int, 2>;
    int t = P;
    // predicated levels [t, t1) in (even, odd) pairs, so the two parities
    // are compile-time and the scheduler sees two levels at a time
    auto pred_range = [&](auto mode_tag, int t1) {
      if (t < t1 && (t & 1)) level(I1{}, PT{}, mode_tag, t++);
#pragma unroll 1
      for (; t + 1 < t1; t += 2) {
        level(I0{}, PT{}, mode_tag, t);
        level(I1{}, PT{}, mode_tag, t + 1);
      }
      if (t < t1) level(I0{}, PT{}, mode_tag, t++);
    };
    pred_range(M0{}, min(T, core_lo));
    bool cool_noch = false;  // cool-down without channel maxima (below)
    if (core_lo <= core_hi) {
      // core_lo is even: pairs (even, odd), then the final even level.
      // Channel maxima: in the core every stage alternates F and B, so
      // between two forwards of stage i there is a backward and
      // F_end(m+1) >= fl(fl(F_end(m) + b) + f). If send(m) did not wait
      // (its channel end is F_end(m) + sf) and sf < f + b by more than the
      // rounding of those adds, send(m+1) cannot wait either: the channel
      // max is max(F_end, ...) = F_end, exactly. Same for backward sends
      // (sb < f + b). So after a first pair that checks every send of the
      // core starts without waiting (MODE 1), the channel maxima are no-ops
      // and are dropped (MODE 2). The rounding slack is 4 ulps of an upper
      // bound on every node value: M * sum over stages of (f + b + sf + sb).
      bool chok = true, chok2 = true;
      {
        double vs = 0.0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int i = sl * K + r;
          if (run && i < P) {
            const double sbk = r == 0 ? sb0 : sf[r > 0 ? r - 1 : 0];
            vs = vs + (f[r] + bw[r]) + (dmax(sf[r], 0.0) + dmax(sbk, 0.0));
          }
        }
        for (int off = 1; off < W; off <<= 1) {
          const double o = __shfl_down_sync(0xffffffffu, vs, off);
          if (sl + off < W) vs = vs + o;
        }
        vs = __shfl_sync(0xffffffffu, vs, min(31, seg * W));
        const double slack = vs * (double)M * 0x1p-50;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int i = sl * K + r;
          if (run && i < P) {
            const double sbk = r == 0 ? sb0 : sf[r > 0 ? r - 1 : 0];
            const double fb = (f[r] + bw[r]) - slack;
            chok = chok && sf[r] < fb && sbk < fb;
            chok2 = chok2 && sbk < bw[r] - slack;
          }
        }
      }
      bool noch = false;
      if (tr) c_core0 = clock64();
      if (t + 1 <= core_hi) {
        level(I0{}, PF{}, M1{}, t);
        level(I1{}, PF{}, M1{}, t + 1);
        t += 2;
        noch = __all_sync(0xffffffffu, !run || (chok && base_ok));
        // Cool-down: a stage keeps alternating until its last forward, then
        // runs its trailing backwards two levels apart with nothing between,
        // so B_end(j+1) >= B_end(j) + b: with sb < b (same rounding margin)
        // the backward sends cannot wait either.
        cool_noch = noch && __all_sync(0xffffffffu, !run || chok2);
      }
      // Every kAbortPairs pairs a screened neighbour checks the bound below.
      for (; t + 1 <= core_hi;) {
        const int stop = min(core_hi - 1, t + 2 * kAbortPairs - 2);
        if (noch) {
          // unrolled so the scheduler can overlap the tail of one level pair
          // with the next (deeper for K = 4, the latency evaluator)
          if constexpr (K == 4) {
#pragma unroll kUnrollK4
            for (; t <= stop; t += 2) {
              level(I0{}, PF{}, M2{}, t);
              level(I1{}, PF{}, M2{}, t + 1);
            }
          } else {
#pragma unroll kUnrollCore
            for (; t <= stop; t += 2) {
              level(I0{}, PF{}, M2{}, t);
              level(I1{}, PF{}, M2{}, t + 1);
            }
          }
        } else {
          for (; t <= stop; t += 2) {
            level(I0{}, PF{}, M0{}, t);
            level(I1{}, PF{}, M0{}, t + 1);
          }
        }
        if (HP_ABORT_CODE && lim < __builtin_huge_val()) {
          // Early abort: levels < t are done; stage i has issued
          // nF = (t-1-i)/2 + 1 forwards and nB = (t-2P+i)/2 + 1 backwards
          // (closed form above, every stage past its warm-up). Its remaining
          // ops run in order after fr, so compute_end_i + dp_sync_i >=
          // fr + (M-nF) f + (M-nB) b + dps (rounding is monotone; the
          // margin absorbs the summation order), a lower bound on the
          // iteration time (evaluate.cpp:90-97). A neighbour above the
          // current point's time can neither be the move nor tie the leaf
          // best (nb_screen), so it stops here as T_SKIP.
          // Drain: stage i's last op is B(i, M-1), whose gradient still
          // travels down to stage 0 (send j -> j-1, then B(j-1, M-1)), so
          // compute_end_0 >= compute_end_i + sum_{k<i} (sf_k + b_k) and the
          // iteration is >= that + dps_0 (sim.cpp:127-141, evaluate.cpp:90-97).
          // Summed in another order than the simulation; the margin absorbs it.
          double dr[K];
          double acc = 0.0;
#pragma unroll
          for (int r = 0; r < K; ++r) {
            const int i = sl * K + r;
            dr[r] = acc;
            if (run && i < P - 1) acc = acc + (sf[r] + bw[r]);
          }
          double ex = acc;
          for (int off = 1; off < W; off <<= 1) {
            const double o = __shfl_up_sync(0xffffffffu, ex, off);
            if (sl >= off) ex = ex + o;
          }
          ex = __shfl_up_sync(0xffffffffu, ex, 1);
          if (sl == 0) ex = 0.0;
          const double dps0 = dmax(__shfl_sync(0xffffffffu, dps[0], min(31, seg * W)), 0.0);
          double lb = NEG;
#pragma unroll
          for (int r = 0; r < K; ++r) {
            const int i = sl * K + r;
            if (run && i < P) {
              const int nf = min(M, (t - 1 - i) / 2 + 1), nbk = min(M, (t - 2 * P + i) / 2 + 1);
              const double tail = dmax(dps[r], (ex + dr[r]) + dps0);
              lb = dmax(lb, fr[r] + ((double)(M - nf) * f[r] + (double)(M - nbk) * bw[r]) + tail);
            }
          }
          for (int off = 1; off < W; off <<= 1) {
            const double o = __shfl_down_sync(0xffffffffu, lb, off);
            if (sl + off < W) lb = dmax(lb, o);
          }
          lb = __shfl_sync(0xffffffffu, lb, min(31, seg * W));
          if (run && !dead && lb > lim) {
            dead = true;
            dead_t = t;
          }
          if (__all_sync(0xffffffffu, dead || !run)) {
            t = T;  // every candidate of the warp is out
            break;
          }
        }
      }
      if (t <= core_hi) {
        level(I0{}, PF{}, M0{}, t);
        ++t;
      }
      if (tr) {
        c_core1 = clock64();
        tr_noch = noch;
      }
    }
    if (cool_noch) pred_range(M2{}, T);
    else pred_range(M0{}, T);
  }
  if (tr) {
    trace_cycles(b, 5, w.leaf, P, M, tr_noch ? 1 : 0, c_core1 - c_core0);
    trace_cycles(b, 6, w.leaf, P, M, K, clock64() - c_start);
  }
  double v = 0.0;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = sl * K + r;
    if (run && i < P) {
      v = dmax(v, fr[r]);
      v = dmax(v, chf[r]);
      v = dmax(v, chb[r]);
      v = dmax(v, fr[r] + dps[r]);
    }
  }
  for (int off = 1; off < W; off <<= 1) {
    double o = __shfl_down_sync(0xffffffffu, v, off);
    if (sl + off < W) v = dmax(v, o);
  }
  if (sl == 0 && has_cand) {
    double tt = inv ? T_INVALID : (mem ? T_MEMORY : (dead ? T_SKIP : v));
    if (w.kind == 0) b.tseed[2 * w.leaf + (int)cand_id(w, seg)] = tt;
    else if (w.kind == 1) b.nb[b.nb_off[w.leaf] + (int)cand_id(w, seg)] = tt;
    else b.xbuf[w.out + seg] = tt;
    // algorithmic ops of the levels this candidate needed
    const long long full = 8LL * P * M - 4LL * M;
    if (run && b.ops) {
      atomicAdd(b.ops, (unsigned long long)(dead ? full * dead_t / (2LL * (M + P - 1)) : full));
      atomicAdd(b.ops + (dead ? 2 : 1), 1ULL);
    }
  }
}

template <int K, bool FAST>
__device__ __forceinline__ void eval_item(const Bufs& b, const Work& w, const int lane) {
  if constexpr (FAST) eval_item_fast<K>(b, w, lane);
  else eval_item_generic<K>(b, w, lane);
}

// Batch evaluator: warps pull work items from a list.
template <int K, bool FAST>
__global__ void __launch_bounds__(256) k_eval(Bufs b, const Work* items, const int* n_items,
                                              int* next_item) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(next_item, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= *n_items) return;
    const Work w = items[it];
    eval_item<K, FAST>(b, w, lane);
  }
}

// ------------------------------------------------------------------ hill climb

// Device-side work queue of the asynchronous steepest-descent search. Every
// leaf advances on its own: the warp that finishes the last neighbour item of
// a leaf runs that leaf's step (hill_step) and enqueues its next neighbours,
// so there is no global per-step barrier and no host round trip; the kernel
// ends when no leaf is still climbing. One persistent kernel serves every
// evaluator class (the item's leaf selects the evaluator), so the long climbs
// of one class overlap the bulk of the others instead of forming a serial
// tail per class.
// Three FIFO rings with ticket claims, in priority order: ring 0 receives
// the steps of the critical leaves — the host's pick of the longest expected
// climbs (P^2 M), as many as one warp per SM sub-partition can run — ring 1
// those of any leaf whose climb so far is long (steps x levels per
// simulation >= hi_levels), ring 2 everything else. The long climbs are the
// critical path: a step waits for all of its items, so a climb queued behind
// a full ring advances one ring's worth of items per step. Ring-0 items run
// the lowest-latency evaluator for their P (K = 4 up to P = 128: fewer
// stages per lane, a shorter level) and only warps 0-3 of each block serve
// ring 0 (one per SM sub-partition). Each warp holds at most one ticket per
// ring and serves a held ticket as soon as it is filled (pop_item), so a
// filled slot stays unread for at most one item's run; the ring capacity
// (one step per climbing leaf plus the resident warps, + slack) bounds the
// unread slots otherwise. A consumer that finds its slot's sequence number
// past its ticket (lapped) aborts the search with an error instead of
// hanging.
constexpr int kRings = 3;

struct AsyncQ {
  Work* slots[kRings];
  unsigned long long* seq[kRings];   // slot k holds ticket t when seq[k] == t + 1
  unsigned long long* head[kRings];  // next ticket to hand out
  unsigned long long* tail[kRings];  // next ticket to produce
  int* pending;                 // per leaf: items of the current step not yet done
  int* active;                  // leaves still climbing
  int* abort;                   // 1: watchdog (no global progress), 2: ring overwrite
  unsigned long long* progress; // items completed (global progress for the watchdog)
  unsigned long long cap;
  long long hi_levels;          // priority threshold (see above)
  const unsigned char* crit;    // per leaf: critical (level 0 from the first step)
  int lat;                      // level-0 items use lat_class
  int lead;                     // level 0 is served by warps 0-3 of each block only
  int crit_sms;                 // > 0: level 0 only on the first crit_sms blocks (one per SM),
                                // whose warps 4-7 exit: critical items run alone on their
                                // sub-partitions (see k_hill_async)
  int r1_thr;                   // see pop_item (0: every warp serves ring 1)
  int r0_thr;                   // < 0: ring 0 only on lead warps; else also on the others while
                                // its backlog exceeds r0_thr
  int crit_mode;                // with crit_sms: 0 warps 0-3 of those blocks serve ring 0 first,
                                // then the others, warps 4-7 exit; 1 warps 0-3 serve ring 0
                                // only, warps 4-7 the other rings; 2 warps 0-3 ring 0 only,
                                // warps 4-7 exit
};

__device__ __forceinline__ int leaf_class(const Leaf& lf) { return eval_class(lf.P, lf.M, lf.sched == 0); }

// Lowest-latency fast class for a leaf (see AsyncQ); generic leaves keep theirs.
__host__ __device__ inline int lat_class(int P, int cls) {
  if (cls >= 4) return cls;
  return P <= 128 ? 1 : (P <= 192 ? 2 : 3);
}

// HP_DEBUG_TRACE record: (globaltimer ns, ev << 59 | cls << 56 | P << 48 |
// M << 32 | aux << 20 | leaf). ev 0: step done (aux = move), 1: item
// start, 2: item end, 3: neighbourhood screened (aux = survivors), 4: items
// pushed.
__device__ void trace_event(const Bufs& b, int ev, int li, const Leaf& lf, unsigned aux) {
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  unsigned long long k = atomicAdd(b.trace, 1ULL);
  if (k < (1ULL << 22)) {
    b.trace[1 + 2 * k] = now;
    b.trace[2 + 2 * k] = ((unsigned long long)ev << 59) | ((unsigned long long)leaf_class(lf) << 56) |
                         ((unsigned long long)(lf.P & 0xff) << 48) | ((unsigned long long)(lf.M & 0xffff) << 32) |
                         ((unsigned long long)(aux & 0xfff) << 20) | (unsigned)(li & 0xfffff);
  }
}

// Whole warp: enqueues the n surviving neighbours (nb_ids of the leaf) of a
// leaf's current step, cpw per item, one item per lane.
__device__ void push_items(const Bufs& b, const AsyncQ& q, int li, const Leaf& lf, int level, int nslots,
                           int lane) {
  const int cls = level == 0 && q.lat ? lat_class(lf.P, leaf_class(lf)) : leaf_class(lf);
  const int cpw = class_cpw(cls, lf.P);
  const int nit = (nslots + cpw - 1) / cpw;
  unsigned long long t = 0;
  if (lane == 0) {
    q.pending[li] = nit;
    __threadfence();  // pending is set before any item of the step is visible
    t = atomicAdd(q.tail[level], (unsigned long long)nit);
  }
  t = __shfl_sync(0xffffffffu, t, 0);
  for (int j0 = 0; j0 < nit; j0 += 32) {
    const int j = j0 + lane;
    unsigned long long k = 0;
    if (j < nit) {
      Work w;
      w.leaf = li;
      w.kind = 1;
      w.first = j * cpw;
      w.n = min(cpw, nslots - j * cpw);
      w.out = cls + 1;  // evaluator class + 1 (kind-1 items have no output slot)
      w.ids = nullptr;
      k = (t + j) % q.cap;
      q.slots[level][k] = w;
    }
    __threadfence();
    if (j < nit) atomicExch(q.seq[level] + k, t + j + 1);
  }
}

// Warp scans over per-stage values held in contiguous chunks of C stages
// per lane (lane l: stages [l*C, l*C+C)). Exclusive prefix sum / prefix max
// and inclusive-from-the-right suffix max of the lanes' chunk totals.
__device__ __forceinline__ double warp_excl_sum(double v, int lane) {
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = x + y;
  }
  const double e = __shfl_up_sync(0xffffffffu, x, 1);
  return lane == 0 ? 0.0 : e;
}
__device__ __forceinline__ double warp_excl_max(double v, int lane) {
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = dmax(x, y);
  }
  const double e = __shfl_up_sync(0xffffffffu, x, 1);
  return lane == 0 ? neg_inf() : e;
}
__device__ __forceinline__ double warp_excl_suffix_max(double v, int lane) {
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_down_sync(0xffffffffu, x, o);
    if (lane + o < 32) x = dmax(x, y);
  }
  const double e = __shfl_down_sync(0xffffffffu, x, 1);
  return lane == 31 ? neg_inf() : e;
}

// lb_scan (hp_search_core.cuh) across the warp: the prefix sums are added in
// a different order than the path, which kScreenMargin absorbs.
__device__ void lb_scan_warp(const Leaf& lf, StageLB* s, int lane) {
  const int P = lf.P;
  const int C = (P + 31) >> 5;
  const int i0 = min(P, lane * C), i1 = min(P, i0 + C);
  const double M = (double)lf.M;
  double sa = 0.0, sb = 0.0;
  double f[8], bk[8], sf[8], dps[8];  // the lane's chunk (C <= 8)
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + r;
    if (i < i1) {
      f[r] = __ldcg(&s[i].f);
      bk[r] = __ldcg(&s[i].b);
      sf[r] = __ldcg(&s[i].sf);
      dps[r] = __ldcg(&s[i].dps);
      sa = sa + f[r] + sf[r];
      sb = sb + sf[r] + bk[r];
    } else {
      f[r] = bk[r] = sf[r] = dps[r] = 0.0;
    }
  }
  double A = warp_excl_sum(sa, lane), Bt = warp_excl_sum(sb, lane);
  const double Bt0 = Bt;
  double mx = neg_inf(), my = neg_inf();
  double X[8], Y[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + r;
    if (i < i1) {
      __stcg(reinterpret_cast<double2*>(&s[i].A), make_double2(A, Bt));
      const double core = A + M * (f[r] + bk[r]);
      X[r] = core + Bt;
      Y[r] = core + dps[r];
      mx = dmax(mx, X[r]);
      my = dmax(my, Y[r]);
      A = A + f[r] + sf[r];
      Bt = Bt + sf[r] + bk[r];
    }
  }
  double px = warp_excl_max(mx, lane), py = warp_excl_max(my, lane);
  const double qx = warp_excl_suffix_max(mx, lane), qy = warp_excl_suffix_max(my, lane);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + r;
    if (i < i1) {
      __stcg(reinterpret_cast<double2*>(&s[i].PX), make_double2(px, py));
      px = dmax(px, X[r]);
      py = dmax(py, Y[r]);
    }
  }
  double sx = qx, sy = qy;
#pragma unroll
  for (int r = 7; r >= 0; --r) {
    const int i = i0 + r;
    if (i < i1) {
      sx = dmax(sx, X[r]);
      sy = dmax(sy, Y[r]);
      __stcg(reinterpret_cast<double2*>(&s[i].SX), make_double2(sx, sy));
    }
  }
  // pair circuits (pair_gain, lb_scan): pair i needs stage i+1's f, b, dps
  // and Bt_{i+1}; the chunk's last pair takes them from the next lane (whose
  // chunk starts at Bt_{i1}, this lane's running Bt)
  const double nf = __shfl_down_sync(0xffffffffu, f[0], 1);
  const double nbk = __shfl_down_sync(0xffffffffu, bk[0], 1);
  const double ndps = __shfl_down_sync(0xffffffffu, dps[0], 1);
  const bool pairs = lf.sched == 1;
  double gx[8], gy[8];
  double mg = neg_inf(), mgy = neg_inf();
  double bt = Bt0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + r;
    gx[r] = gy[r] = neg_inf();
    if (i < i1) {
      const double bt1 = bt + sf[r] + bk[r];  // Bt_{i+1}
      if (pairs && i + 1 < P) {
        const bool in = r + 1 < 8 && i + 1 < i1;
        const double fe = in ? f[r < 7 ? r + 1 : 7] : nf;
        const double be = in ? bk[r < 7 ? r + 1 : 7] : nbk;
        const double de = in ? dps[r < 7 ? r + 1 : 7] : ndps;
        gx[r] = pair_gain(lf.M, P, i, pair_cyc(f[r], bk[r], fe, be, sf[r]), be);
        gy[r] = gx[r] - bt1 + de;
      }
      mg = dmax(mg, gx[r]);
      mgy = dmax(mgy, gy[r]);
      bt = bt1;
    }
  }
  double pg = warp_excl_max(mg, lane), pgy = warp_excl_max(mgy, lane);
  double sg = warp_excl_suffix_max(mg, lane), sgy = warp_excl_suffix_max(mgy, lane);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + r;
    if (i < i1) {
      __stcg(reinterpret_cast<double2*>(&s[i].PG), make_double2(pg, pgy));
      pg = dmax(pg, gx[r]);
      pgy = dmax(pgy, gy[r]);
    }
  }
#pragma unroll
  for (int r = 7; r >= 0; --r) {
    const int i = i0 + r;
    if (i < i1) {
      sg = dmax(sg, gx[r]);
      sgy = dmax(sgy, gy[r]);
      __stcg(reinterpret_cast<double2*>(&s[i].SG), make_double2(sg, sgy));
    }
  }
}

// HP_DEBUG_PHASES: cycles per phase of the step logic, summed over every
// step of the search (lane 0's clock; printed by search_full)
// Compiled in only with -DHP_PHASES=1 (tools/tune/build_variants.py): even
// untaken, the checks in the item loop cost the C3 sweep ~7 %.
#ifndef HP_PHASES
#define HP_PHASES 0
#endif
__device__ unsigned long long g_phase[16];
__constant__ int c_dbg_phases;
#if HP_PHASES
#define PHASE_T0 long long ph_t = c_dbg_phases ? clock64() : 0
#define PHASE_MARK(k)                                                        \
  if (c_dbg_phases && lane == 0) {                                           \
    const long long now_ = clock64();                                        \
    atomicAdd(&g_phase[k], (unsigned long long)(now_ - ph_t));               \
    ph_t = now_;                                                             \
  }
#define PHASE_COUNT(k) \
  if (c_dbg_phases && lane == 0) atomicAdd(&g_phase[k], 1ULL)
#else
#define PHASE_T0 (void)0
#define PHASE_MARK(k) (void)0
#define PHASE_COUNT(k) (void)0
#endif

// Whole warp: screens the neighbours of leaf li's current split (nb_screen;
// off while the search log is recorded) and lists the survivors in nb_ids.
// Screened slots get their T_SKIP / T_MEMORY / T_INVALID value in nb right
// away. Returns the survivor count (warp-uniform).
__device__ int screen_neighbours(const Bufs& b, int li, const Leaf& lf, int lane, int moved) {
  const int P = lf.P;
  const int nslots = 2 * (P - 1);
  const LeafGroup* lg = b.lg + lf.lg_off;
  const uint8_t* slots = b.layouts + lf.layout_off;
  const double* hop = b.hop + lf.B_idx * c_consts.n_links;
  const int* cur = b.cur + lf.split_off;
  double* nbt = b.nb + b.nb_off[li];
  long long* ids = b.nb_ids + b.nb_off[li];
  StageLB* sl = b.lbs + lf.split_off;
  StageNb* sn = b.lbn + lf.split_off;
  const bool screen = b.log.vals == nullptr;
  PHASE_T0;
  const double cur_t = __ldcg(&b.hs[li].cur_time);
  if (screen) {
    // (cur was last written by whichever SM ran the previous step)
    // per-stage rows: all stages on the first step, afterwards only the two
    // stages the last move changed (moved, moved + 1)
    if (moved < 0) {
      const int C = (P + 31) >> 5;
      const int i1 = min(P, lane * C + C);
      for (int i = lane * C; i < i1; ++i) {
        const int ci = __ldcg(cur + i);
        lb_stage(c_consts, lf, lg, slots, hop, i, ci, sl[i]);
        lb_stage_nb(c_consts, lf, lg, slots, hop, i, ci, sn[i]);
      }
    } else if (lane < 2) {
      const int i = moved + lane;
      const int ci = __ldcg(cur + i);
      StageLB t;
      lb_stage(c_consts, lf, lg, slots, hop, i, ci, t);
      __stcg(&sl[i].f, t.f);
      __stcg(&sl[i].b, t.b);
      __stcg(&sl[i].sf, t.sf);
      __stcg(&sl[i].dps, t.dps);
      StageNb u;
      lb_stage_nb(c_consts, lf, lg, slots, hop, i, ci, u);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        __stcg(&sn[i].f[k], u.f[k]);
        __stcg(&sn[i].b[k], u.b[k]);
        __stcg(&sn[i].dps[k], u.dps[k]);
        __stcg(&sn[i].st[k], u.st[k]);
      }
    }
    __syncwarp();
    PHASE_MARK(0);
    lb_scan_warp(lf, sl, lane);
    __syncwarp();
    PHASE_MARK(1);
  }
  // One boundary per lane and round (bb = lane + 32 j): both of its slots
  // read the same rows, loaded as one batch (nb_rows_load) before the two
  // bounds are computed; the survivors are listed in slot order.
  int n = 0;
  int nskip = 0;
  if (screen) {
#pragma unroll 1
    for (int j = 0; 32 * j < P - 1; ++j) {
      const int bb = lane + 32 * j;
      bool s0 = false, s1 = false;
      if (bb < P - 1) {
        NbRows r;
        nb_rows_load(lf, sl, sn, bb, r);
        const double c0 = screen_of(nb_lb_rows(lf, r, bb, 0), cur_t);
        const double c1 = screen_of(nb_lb_rows(lf, r, bb, 1), cur_t);
        s0 = c0 == 0.0;
        s1 = c1 == 0.0;
        if (!s0) nbt[2 * bb] = c0;
        if (!s1) nbt[2 * bb + 1] = c1;
        nskip += (c0 == T_SKIP ? 1 : 0) + (c1 == T_SKIP ? 1 : 0);
      }
      const unsigned m0 = __ballot_sync(0xffffffffu, s0), m1 = __ballot_sync(0xffffffffu, s1);
      const unsigned lower = (1u << lane) - 1u;
      int pos = n + __popc(m0 & lower) + __popc(m1 & lower);
      if (s0) ids[pos++] = 2 * bb;
      if (s1) ids[pos] = 2 * bb + 1;
      n += __popc(m0) + __popc(m1);
    }
  } else {
    for (int qq = lane; qq < nslots; qq += 32) ids[qq] = qq;
    n = nslots;
  }
  nskip = __reduce_add_sync(0xffffffffu, (unsigned)nskip);
  PHASE_MARK(2);
  if (lane == 0 && nskip && b.ops) atomicAdd(b.ops + 3, (unsigned long long)nskip);
  __threadfence();
  __syncwarp();
  PHASE_MARK(3);
  return n;
}

// Whole warp: hill_step (hp_search_core.cuh, planner.cpp:470-489) with the
// memo scan and the neighbour loop spread over the lanes; same decisions,
// counts and leaf best. Boundary bb (slots 2bb, 2bb+1) belongs to lane
// bb & 31, register k = bb >> 5. Returns hs.active.
__device__ int hill_step_warp(const Bufs& b, int li, const Leaf& lf, int lane, int& moved) {
  const unsigned FULL = 0xffffffffu;
  const int P = lf.P;
  const int nslots = 2 * (P - 1);
  int* cur = b.cur + lf.split_off;
  int* best = b.best + lf.split_off;
  short* hist = b.hist + b.hist_off[li];
  const double* nb = b.nb + b.nb_off[li];
  PHASE_T0;
  HillState hs;
  hs.cur_time = __ldcg(&b.hs[li].cur_time);
  hs.best_time = __ldcg(&b.hs[li].best_time);
  hs.steps = __ldcg(&b.hs[li].steps);
  hs.has_best = __ldcg(&b.hs[li].has_best);
  constexpr int NK = (HP_MAX_STAGES + 31) / 32;
  // Everything the step reads is loaded up front in one round of independent
  // L2 loads (the leaf's state was written by whichever SM ran the previous
  // step): the neighbour times, this lane's chunk of the current split, and
  // the newest 32 * BV path points' move codes and memo distances. Only a
  // climb longer than the window reads its older points chunk by chunk.
  const int C = (P + 31) >> 5;
  const int i0 = min(P, lane * C), i1 = min(P, i0 + C);
  double nv[NK][2];
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int bb = lane + 32 * k;
    nv[k][0] = nv[k][1] = T_INVALID;
    if (bb + 1 < P) {
      nv[k][0] = __ldcg(nb + 2 * bb);
      nv[k][1] = __ldcg(nb + 2 * bb + 1);
    }
  }
  int cv[8], rv2[2][8];  // cur[i0 + r] (C <= 8); the seeds' (uniform, proportional)
  {
    const int* ru = b.uni + lf.split_off;
    const int* rp = b.prop + lf.split_off;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const bool in = i0 + r < i1;
      cv[r] = in ? __ldcg(cur + i0 + r) : 0;
      rv2[0][r] = in ? ru[i0 + r] : 0;
      rv2[1][r] = in ? rp[i0 + r] : 0;
    }
  }
  long long g_sim = 0, g_pru = 0;
  if (lane == 0) {
    g_sim = __ldcg(&b.hs[li].simulated);
    g_pru = __ldcg(&b.hs[li].pruned);
  }
  int* memo = b.memo_d + b.hist_off[li];
  constexpr int BV = 16;
  const int top = hs.steps - 1;
  int hv[BV], dv[BV];  // point top - 32 v - lane: move code, D
#pragma unroll
  for (int v = 0; v < BV; ++v) {
    const int idx = top - 32 * v - lane;
    hv[v] = idx >= 0 ? __ldcg(hist + idx) : 0;
    dv[v] = idx >= 0 ? __ldcg(memo + idx) : 3;
  }

  // ---- mark_old (hp_search_core.cuh): path points t with D_t = ||S_k - S_t||_1
  // <= 2 (memo_d, maintained incrementally below). For those the nonzero
  // boundaries of S_k - S_t come from undoing moves k-1..t (rare beyond t =
  // k-2 on a strictly improving path).
  unsigned oldm = 0;  // bit 2k + (dir < 0) for my boundary lane + 32k
  bool all_old = false;
#pragma unroll
  for (int v = 0; v < BV; ++v) {
    if (top - 32 * v < 0) break;
    unsigned fl = __ballot_sync(FULL, dv[v] <= 2);
    while (fl) {
      const int j = __ffs(fl) - 1;
      fl &= fl - 1;
      const int t = top - 32 * v - j;
      if (__shfl_sync(FULL, dv[v], j) == 0) {
        all_old = true;
        continue;
      }
      int dl[NK];
#pragma unroll
      for (int k = 0; k < NK; ++k) dl[k] = 0;
      for (int u = top; u >= t; --u) {
        const int off = top - u, vv = off >> 5;
        int x = 0;
#pragma unroll
        for (int w = 0; w < BV; ++w)
          if (w == vv) x = hv[w];
        const int code = __shfl_sync(FULL, x, off & 31);
        const int bb = code >> 1;
        if ((bb & 31) == lane) {
          const int r = bb >> 5;
#pragma unroll
          for (int k = 0; k < NK; ++k)
            if (k == r) dl[k] += (code & 1) ? -1 : 1;
        }
      }
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (dl[k] != 0) oldm |= 1u << (2 * k + (dl[k] > 0 ? 1 : 0));  // toward c_t
    }
  }
  for (int t1 = top - 32 * BV; t1 >= 0; t1 -= 128) {  // beyond the window
   int dvs[4];
#pragma unroll
   for (int u = 0; u < 4; ++u) {
    const int idx = t1 - 32 * u - lane;
    dvs[u] = idx >= 0 ? __ldcg(memo + idx) : 3;
   }
#pragma unroll
   for (int u = 0; u < 4; ++u) {
    const int t0 = t1 - 32 * u;
    const int dvu = dvs[u];
    unsigned fl = __ballot_sync(FULL, dvu <= 2);
    while (fl) {
      const int j = __ffs(fl) - 1;
      fl &= fl - 1;
      const int t = t0 - j;
      if (__shfl_sync(FULL, dvu, j) == 0) {
        all_old = true;
        continue;
      }
      int dl[NK];
#pragma unroll
      for (int k = 0; k < NK; ++k) dl[k] = 0;
      for (int u2 = top; u2 >= t; --u2) {
        const int code = __ldcg(hist + u2);
        const int bb = code >> 1;
        if ((bb & 31) == lane) {
          const int r = bb >> 5;
#pragma unroll
          for (int k = 0; k < NK; ++k)
            if (k == r) dl[k] += (code & 1) ? -1 : 1;
        }
      }
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (dl[k] != 0) oldm |= 1u << (2 * k + (dl[k] > 0 ? 1 : 0));  // toward c_t
    }
   }
  }
  // seeds at distance 1: prefix sums of cur - ref over each lane's chunk
  {
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
      const int (&rv)[8] = rv2[sd];
      int loc = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) loc += cv[r] - rv[r];
      int x = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
      }
      int e = __shfl_up_sync(FULL, x, 1);
      if (lane == 0) e = 0;
      int dist = 0, cb = -1, cd = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + r;
        if (i < i1 && i + 1 < P) {
          e += cv[r] - rv[r];
          if (e != 0) {
            dist += abs(e);
            cb = i;
            cd = e;
          }
        }
      }
      dist = __reduce_add_sync(FULL, dist);
      if (dist == 1) {  // one boundary at distance 1: move its bit to the owner lane
        const int src = __ffs(__ballot_sync(FULL, cb >= 0)) - 1;
        const int gb = __shfl_sync(FULL, cb, src);
        const int gd = __shfl_sync(FULL, cd, src);
        if ((gb & 31) == lane) oldm |= 1u << (2 * (gb >> 5) + (gd > 0 ? 1 : 0));
      }
    }
  }

  PHASE_MARK(4);
  // ---- neighbour loop: counts, move argmin (time, slot), best candidate
  long long sim = 0, pru = 0;
  double mt = __builtin_huge_val();
  int mq = 0x7fffffff;                 // feasible argmin (first slot on ties)
  double nt = __builtin_huge_val();
  int nq = 0x7fffffff, ntie = 0;       // non-old feasible minimum
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int bb = lane + 32 * k;
    if (bb + 1 < P) {
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        const int q = 2 * bb + sd;
        const double t = nv[k][sd];
        if (t == T_INVALID) continue;
        const bool old = all_old || ((oldm >> (2 * k + sd)) & 1u);
        if (!old) {
          if (t >= 0) ++sim;
          else ++pru;
        }
        if (t < 0) continue;
        if (t < mt || (t == mt && q < mq)) {
          mt = t;
          mq = q;
        }
        if (!old) {
          if (t < nt || (t == nt && q < nq)) {
            if (t < nt) ntie = 0;
            nt = t;
            nq = q;
          }
          if (t == nt) ++ntie;
        }
      }
    }
  }
  sim = __reduce_add_sync(FULL, (unsigned)sim);
  pru = __reduce_add_sync(FULL, (unsigned)pru);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t2 = __shfl_xor_sync(FULL, mt, o);
    const int q2 = __shfl_xor_sync(FULL, mq, o);
    if (t2 < mt || (t2 == mt && q2 < mq)) {
      mt = t2;
      mq = q2;
    }
    const double u2 = __shfl_xor_sync(FULL, nt, o);
    const int r2 = __shfl_xor_sync(FULL, nq, o);
    const int c2 = __shfl_xor_sync(FULL, ntie, o);
    if (u2 < nt) {
      nt = u2;
      nq = r2;
      ntie = c2;
    } else if (u2 == nt) {
      ntie += c2;
      nq = min(nq, r2);
    }
  }
  // leaf best: the minimum of (best, non-old feasible neighbours) in the
  // (time, encoding) order; ties in time need the encodings (rare: serial)
  const bool have_n = nq != 0x7fffffff;
  bool serial_best = false;
  bool take_n = false;
  if (have_n) {
    if (!hs.has_best || nt < hs.best_time) {
      if (ntie == 1) take_n = true;
      else serial_best = true;
    } else if (nt == hs.best_time) {
      serial_best = true;
    }
  }
  if (serial_best) {
    // slot old flags to scratch (nb_ids is rewritten by the next screen)
    unsigned char* oldb = reinterpret_cast<unsigned char*>(b.nb_ids + b.nb_off[li]);
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const int bb = lane + 32 * k;
      if (bb + 1 < P) {
        oldb[2 * bb] = all_old || ((oldm >> (2 * k)) & 1u);
        oldb[2 * bb + 1] = all_old || ((oldm >> (2 * k + 1)) & 1u);
      }
    }
    __syncwarp();
    if (lane == 0) {
      int cl[HP_MAX_STAGES], bl[HP_MAX_STAGES], tmp[HP_MAX_STAGES];
      for (int i = 0; i < P; ++i) {
        cl[i] = __ldcg(cur + i);
        bl[i] = __ldcg(best + i);
      }
      for (int q = 0; q < nslots; ++q) {
        const double t = __ldcg(nb + q);
        if (t < 0 || oldb[q]) continue;
        bool better = !hs.has_best || t < hs.best_time;
        const int bq = q >> 1, d = (q & 1) ? -1 : 1;
        if (!better && t == hs.best_time) {
          for (int i = 0; i < P; ++i) tmp[i] = cl[i];
          tmp[bq] += d;
          tmp[bq + 1] -= d;
          better = split_enc_less(P, tmp, bl);
        }
        if (better) {
          hs.has_best = 1;
          hs.best_time = t;
          for (int i = 0; i < P; ++i) bl[i] = cl[i];
          bl[bq] += d;
          bl[bq + 1] -= d;
        }
      }
      for (int i = 0; i < P; ++i) __stcg(best + i, bl[i]);
    }
    __syncwarp();
  } else if (take_n) {
    const int bq = nq >> 1, d = (nq & 1) ? -1 : 1;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = i0 + r;
      if (i < i1) __stcg(best + i, cv[r] + (i == bq ? d : (i == bq + 1 ? -d : 0)));
    }
    hs.has_best = 1;
    hs.best_time = nt;
  }
  __syncwarp();
  // (warp-uniform after the reductions)
  int active = (mq == 0x7fffffff || !(mt < hs.cur_time)) ? 0 : 1;  // no feasible neighbour, or no improvement
  if (active) {
    // the move: the owner lanes of stages bq, bq + 1 update cur
    const int bq = mq >> 1, d = (mq & 1) ? -1 : 1;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = i0 + r;
      if (i < i1 && (i == bq || i == bq + 1)) __stcg(cur + i, cv[r] + (i == bq ? d : -d));
    }
    if (hs.steps + 1 >= 4 * c_consts.L) active = 0;
  }
  if (lane == 0) {
    HillState& g = b.hs[li];
    __stcg(&g.simulated, g_sim + sim);
    __stcg(&g.pruned, g_pru + pru);
    __stcg(&g.has_best, hs.has_best);
    __stcg(&g.best_time, hs.best_time);
    if (!(mq == 0x7fffffff || !(mt < hs.cur_time))) {
      __stcg(hist + hs.steps, (short)mq);
      __stcg(&g.steps, hs.steps + 1);
      __stcg(&g.cur_time, mt);
    }
    __stcg(&g.active, active);
  }
  moved = mq >> 1;
  if (active) {
    // D_t(k+1) = D_t(k) + |c(t) + d| - |c(t)|, c(t) = sum of the moves of
    // boundary mb over t..k-1 (a suffix scan, 32 path points per round);
    // D_k(k+1) = 1
    const int mb = mq >> 1, md = (mq & 1) ? -1 : 1;
    int carry = 0;
#pragma unroll
    for (int v = 0; v < BV; ++v) {
      if (top - 32 * v < 0) break;
      const int idx = top - 32 * v - lane;
      int x = (idx >= 0 && (hv[v] >> 1) == mb) ? ((hv[v] & 1) ? -1 : 1) : 0;
      if (__ballot_sync(FULL, x != 0)) {  // (most blocks hold no move of boundary mb)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, x, o);
          if (lane >= o) x += y;
        }
      }
      const int c = carry + x;
      if (idx >= 0) __stcg(memo + idx, dv[v] + abs(c + md) - abs(c));
      carry = __shfl_sync(FULL, c, 31);
    }
    for (int t1 = top - 32 * BV; t1 >= 0; t1 -= 128) {  // beyond the window
      int xs[4], ms[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = t1 - 32 * u - lane;
        xs[u] = 0;
        ms[u] = 0;
        if (idx >= 0) {
          const int code = __ldcg(hist + idx);
          if ((code >> 1) == mb) xs[u] = (code & 1) ? -1 : 1;
          ms[u] = __ldcg(memo + idx);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = t1 - 32 * u - lane;
        int x = xs[u];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, x, o);
          if (lane >= o) x += y;
        }
        const int c = carry + x;
        if (idx >= 0) __stcg(memo + idx, ms[u] + abs(c + md) - abs(c));
        carry = __shfl_sync(FULL, c, 31);
      }
    }
    if (lane == 0) __stcg(memo + hs.steps, 1);
  }
  PHASE_MARK(5);
  __threadfence();
  __syncwarp();
  PHASE_MARK(6);
  PHASE_COUNT(7);
  return active;
}

// Whole warp, after the last item of leaf li's step (do_step) or for its
// first step: lane 0 runs the step (hill_step), then the warp screens the
// next neighbourhood and enqueues the survivors. A neighbourhood with no
// survivor cannot improve, so the next step runs at once (and stops).
__device__ void advance_leaf(const Bufs& b, const AsyncQ& q, int li, int lane, bool do_step) {
  const Leaf lf = b.leaves[li];
  int moved = -1;  // boundary of the last move (screen rows to refresh), -1: all
  for (;;) {
    if (do_step) {
      int active = 0;
      if (b.log.vals == nullptr) {
        active = hill_step_warp(b, li, lf, lane, moved);
        if (lane == 0) {
          if (b.trace) {
            const int st = b.hs[li].steps;
            trace_event(b, 0, li, lf, st > 0 ? (unsigned)b.hist[b.hist_off[li] + st - 1] : 0xfff);
          }
          if (!active) {
            __threadfence();
            atomicSub(q.active, 1);
          }
        }
        if (!active) return;
      } else {
        if (lane == 0) {
          HillState hs = b.hs[li];
          int delta[HP_MAX_STAGES];
          unsigned char old[2 * HP_MAX_STAGES];
          int tmp[HP_MAX_STAGES];
          for (int i = 0; i < lf.P; ++i) delta[i] = 0;
          const int seq = hs.steps;
          hill_step(c_consts, lf, b.lg + lf.lg_off, b.layouts + lf.layout_off, b.cur + lf.split_off,
                    b.uni + lf.split_off, b.prop + lf.split_off, b.best + lf.split_off,
                    b.hist + b.hist_off[li], hs, b.nb + b.nb_off[li], delta, old, tmp);
          b.hs[li] = hs;
          // simulated, non-memo neighbours in visit order (planner.cpp:472-476)
          const double* nbt = b.nb + b.nb_off[li];
          const int nslots = 2 * (lf.P - 1);
          int n = 0;
          for (int k = 0; k < nslots; ++k) n += (!old[k] && nbt[k] >= 0) ? 1 : 0;
          long long off = log_reserve(b.log, li, seq, n);
          if (off >= 0)
            for (int k = 0; k < nslots; ++k)
              if (!old[k] && nbt[k] >= 0) b.log.vals[off++] = nbt[k];
          if (b.trace) trace_event(b, 0, li, lf, hs.steps > 0 ? (unsigned)b.hist[b.hist_off[li] + hs.steps - 1] : 0xfff);
          active = hs.active;
          if (!active) {
            __threadfence();
            atomicSub(q.active, 1);
          }
        }
        active = __shfl_sync(0xffffffffu, active, 0);
        if (!active) return;
        __syncwarp();
      }
    }
    do_step = true;
    const int n = screen_neighbours(b, li, lf, lane, moved);
    if (b.trace && b.trace_items && lane == 0) trace_event(b, 3, li, lf, n);
    if (n > 0) {
      const long long lv = (long long)__ldcg(&b.hs[li].steps) * (2 * (lf.M + lf.P - 1));
      const int ring = (q.crit && q.crit[li]) ? 0 : (lv >= q.hi_levels ? 1 : 2);
      push_items(b, q, li, lf, ring, n, lane);
      if (b.trace && b.trace_items && lane == 0) trace_event(b, 4, li, lf, 0);
      return;
    }
  }
}

// Enqueue the first step of every climbing leaf (a warp per leaf).
__global__ void k_async_seed(Bufs b, AsyncQ q, const int* ids, int n) {
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= n) return;
  const int li = ids[k];
  if (!b.hs[li].active) return;
  if (lane == 0) atomicAdd(q.active, 1);
  advance_leaf(b, q, li, lane, false);
}

// Slot state of a claimed ticket h: 1 filled (item read into w), 0 not yet
// filled, -1 lapped (the slot's sequence number is past the ticket: the
// producer of ticket h + cap overwrote the unread item).
__device__ __forceinline__ int try_slot(const AsyncQ& q, int lv, unsigned long long h, Work& w) {
  const unsigned long long k = h % q.cap;
  const unsigned long long sq = *(volatile unsigned long long*)(q.seq[lv] + k);
  if (sq != h + 1) return sq > h + 1 ? -1 : 0;
  __threadfence();
  const Work* sl = q.slots[lv] + k;
  w.leaf = __ldcg(&sl->leaf);
  w.kind = __ldcg(&sl->kind);
  w.first = __ldcg(&sl->first);
  w.n = __ldcg(&sl->n);
  w.out = __ldcg(&sl->out);
  return 1;
}

// Lane 0: next item for this warp (see AsyncQ). Tickets are claimed with
// atomicAdd only when the ring shows unclaimed items (a CAS claim caps the
// claim rate at one per L2 round trip, 4x slower on C3); racing claims can
// pass the tail, and such a ticket is held until a later push fills it while
// the warp serves other rings. A held ticket that is filled is served before
// anything else, so it stays unread for at most the one item in progress
// when it was filled. Returns false when the warp should exit (no leaf
// climbing, or abort).
__device__ bool pop_item(const AsyncQ& q, Work& w, long long (&tk)[kRings], int lv0, bool lead,
                         int lv_end = kRings) {
  unsigned ns = 32;
  long long t0 = clock64();
  unsigned long long seen = *(volatile unsigned long long*)q.progress;
  for (;;) {
    // 1) a held ticket that has been filled meanwhile
    for (int lv = 0; lv < kRings; ++lv) {
      if (tk[lv] < 0) continue;
      const int r = try_slot(q, lv, (unsigned long long)tk[lv], w);
      if (r < 0) {
        atomicExch(q.abort, 2);
        return false;
      }
      if (r > 0) {
        tk[lv] = -1;
        return true;
      }
    }
    // 2) new claims, highest-priority ring first; a claimed higher-priority
    // ticket that is being filled (the producer bumps the tail before it
    // writes the slot) is waited for rather than a lower ring started
    bool held = false;
    int lv_start = lv0;
    if (lv0 == 1 && q.r0_thr >= 0 &&
        *(volatile unsigned long long*)q.tail[0] - *(volatile unsigned long long*)q.head[0] >
            (unsigned long long)q.r0_thr)
      lv_start = 0;  // a deep critical backlog: help it
    for (int lv = lv_start; lv < lv_end && !held; ++lv) {
      const unsigned long long tl = *(volatile unsigned long long*)q.tail[lv];
      const unsigned long long hd = *(volatile unsigned long long*)q.head[lv];
      // (r1_thr > 0: a non-lead warp takes a long-climber item only from a
      // backlog above r1_thr, so a thin ring 1 runs one item per sub-partition)
      if (tk[lv] < 0 && tl > hd && (lv != 1 || lead || tl - hd > (unsigned long long)q.r1_thr)) {
        tk[lv] = (long long)atomicAdd(q.head[lv], 1ULL);
        const int r = try_slot(q, lv, (unsigned long long)tk[lv], w);
        if (r < 0) {
          atomicExch(q.abort, 2);
          return false;
        }
        if (r > 0) {
          tk[lv] = -1;
          return true;
        }
      }
      // (a ticket past the tail — claimed in a race — waits for a future
      // push and must not hold back the lower rings)
      held = tk[lv] >= 0 && (unsigned long long)tk[lv] < *(volatile unsigned long long*)q.tail[lv];
    }
    const int act = *(volatile int*)q.active;
    if (act == 0 || *(volatile int*)q.abort) return false;
    // watchdog: no item completed anywhere for ~35 s while leaves are
    // active means a lost item (a single item takes at most ~1e9 cycles:
    // 2(M+P-1) levels with M <= 5e6)
    const unsigned long long pg = *(volatile unsigned long long*)q.progress;
    if (pg != seen) {
      seen = pg;
      t0 = clock64();
    } else if (clock64() - t0 > (1LL << 36)) {
      atomicExch(q.abort, 1);
      return false;
    }
    __nanosleep(held ? 32 : ns);
    if (ns < 256) ns <<= 1;
  }
}

// Resident 256-thread blocks per SM the hill-climb kernel is compiled for
// (register cap 65536 / (256 * n)). Fewer resident warps shorten each
// warp's level latency (the long climbs are a chain of simulations whose
// latency, not throughput, bounds the search); HP_ALL_MINB overrides at
// build time (tuning).
#ifndef HP_ALL_MINB
#define HP_ALL_MINB 1
#endif
// threads per block of the climb kernel (tuning: 384 = 12 warps per SM at
// <= 168 registers)
#ifndef HP_CLIMB_K8
#define HP_CLIMB_K8 1  // tuning: 0 leaves the K = 8 evaluators out of the climb kernel
#endif
#ifndef HP_ASYNC_MAXT
#define HP_ASYNC_MAXT 256
#endif

#ifndef HP_EVAL_INLINE
#define HP_EVAL_INLINE 0  // tuning: 1 inlines the evaluators into the climb kernel
#endif
#if HP_EVAL_INLINE
template <int K, bool FAST>
__device__ __forceinline__ void eval_item_call(const Bufs& b, const Work& w, int lane) {
  eval_item<K, FAST>(b, w, lane);
}
#else
template <int K, bool FAST>
__device__ __noinline__ void eval_item_call(const Bufs& b, const Work& w, int lane) {
  eval_item<K, FAST>(b, w, lane);
}
#endif

__global__ void __launch_bounds__(HP_ASYNC_MAXT, HP_ALL_MINB) k_hill_async(Bufs bg, AsyncQ q, StagedTables tt) {
  extern __shared__ __align__(128) unsigned char smem_tables[];
  __shared__ __align__(8) unsigned long long tables_bar;
  const Bufs b = stage_tables(bg, tt, smem_tables, &tables_bar);
  const int lane = threadIdx.x & 31;
  long long tk[kRings] = {-1, -1, -1};
  const bool crit_blk = q.crit_sms > 0 && (int)blockIdx.x < q.crit_sms;
  if (crit_blk && (threadIdx.x >> 5) >= 4 && q.crit_mode != 1) return;
  for (;;) {
    int quit = 0, cls = 0;
    Work w{};
    PHASE_T0;
    if (lane == 0) {
      // priority items go to one warp per SM sub-partition (warps 0-3 of
      // the SM's one block), so two of them never share one: a climb step
      // waits for its slowest item
      const int wib = threadIdx.x >> 5;
      int lv0 = wib < 4 || !q.lead ? 0 : 1;
      if (q.crit_sms > 0) lv0 = crit_blk && wib < 4 ? 0 : 1;
      const int lv_end = crit_blk && wib < 4 && q.crit_mode != 0 ? 1 : kRings;
      // (with every SM reserved in mode 1, warps 4-7 are the only ring-1
      // servers; otherwise the unreserved SMs' lead warps are, and warps 4-7
      // of the reserved ones taking ring 1 eagerly costs 4 GPUs 86 -> 97 ms)
      const bool lead = wib < 4 || (crit_blk && q.crit_mode == 1 && q.crit_sms >= (int)gridDim.x);
      quit = pop_item(q, w, tk, lv0, lead, lv_end) ? 0 : 1;
      if (!quit) cls = w.out > 0 ? w.out - 1 : leaf_class(b.leaves[w.leaf]);
    }
    quit = __shfl_sync(0xffffffffu, quit, 0);
    if (quit) return;
    PHASE_MARK(8);
    cls = __shfl_sync(0xffffffffu, cls, 0);
    w.leaf = __shfl_sync(0xffffffffu, w.leaf, 0);
    w.kind = __shfl_sync(0xffffffffu, w.kind, 0);
    w.first = __shfl_sync(0xffffffffu, w.first, 0);
    w.n = __shfl_sync(0xffffffffu, w.n, 0);
    w.out = 0;
    w.ids = w.kind == 1 ? b.nb_ids + b.nb_off[w.leaf] : nullptr;
    const bool tr_item = b.trace && b.trace_items &&
                         ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) % b.trace_items == 0;
    if (tr_item && lane == 0) trace_event(b, 1, w.leaf, b.leaves[w.leaf], w.first);
    switch (cls) {
      case 0: eval_item_call<2, true>(b, w, lane); break;
      case 1: eval_item_call<4, true>(b, w, lane); break;
      case 2: eval_item_call<6, true>(b, w, lane); break;
#if HP_CLIMB_K8
      case 3: eval_item_call<8, true>(b, w, lane); break;
#endif
      case 4: eval_item_call<1, false>(b, w, lane); break;
      case 5: eval_item_call<2, false>(b, w, lane); break;
      case 6: eval_item_call<3, false>(b, w, lane); break;
#if HP_CLIMB_K8
      default: eval_item_call<8, false>(b, w, lane); break;
#else
      default: break;  // (tuning builds without the K = 8 evaluators)
#endif
    }
    __syncwarp();
    PHASE_MARK(9);
    if (tr_item && lane == 0) trace_event(b, 2, w.leaf, b.leaves[w.leaf], w.first);
    int last = 0;
    if (lane == 0) {
      __threadfence();
      last = atomicSub(q.pending + w.leaf, 1) == 1;
      if (last) __threadfence();
      atomicAdd(q.progress, 1ULL);
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    PHASE_MARK(10);
    PHASE_COUNT(11);
    if (last) advance_leaf(b, q, w.leaf, lane, true);
    __syncwarp();
  }
}

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
  HillState hs = b.hs[sp.leaf];
  int* best = b.best + lf.split_off;
  int comp[HP_MAX_STAGES];
  for (long long j = 0; j < sp.n; ++j) {
    double t = b.xbuf[sp.out + j];
    if (b.log.exh) b.log.exh[b.log.exh_off[sp.leaf] + sp.first + j] = t;
    if (t < 0) {
      hs.pruned++;
      continue;
    }
    hs.simulated++;
    bool better = !hs.has_best || t < hs.best_time;
    const int* caps = b.ecap + lf.split_off;
    const long long* tbl = b.etbl + b.etbl_off[sp.leaf];
    if (!better && t == hs.best_time) {
      unrank_bounded(sp.first + j, c_consts.L, lf.P, caps, tbl, comp);
      better = split_enc_less(lf.P, comp, best);
    }
    if (better) {
      hs.has_best = 1;
      hs.best_time = t;
      unrank_bounded(sp.first + j, c_consts.L, lf.P, caps, tbl, best);
    }
  }
  b.hs[sp.leaf] = hs;
}

// ------------------------------------------------------------------ exhaustive (bounded)

// Per exhaustive leaf: memory caps, bounded-composition table, feasible count.
__global__ void k_exh_prep(Bufs b, const int* ids, int n, long long* feas, long long* etbl, int* ecap) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int li = ids[k];
  const Leaf lf = b.leaves[li];
  int* caps = ecap + lf.split_off;
  exh_caps(c_consts, lf, b.lg + lf.lg_off, b.layouts + lf.layout_off, caps);
  feas[li] = exh_table(c_consts.L, lf.P, caps, etbl + b.etbl_off[li]);
}

struct ExhItem {
  int leaf;
  int pad;
  long long first;  // first bounded rank
  long long n;      // ranks in this item (<= 32 * kExhChunk)
};

struct ExhRec {
  double t;
  long long rank;
  long long sim;
  int leaf;
  int has;
};

constexpr int kExhChunk = 64;  // consecutive ranks per thread

// decimal-string order of two ints followed by ':' (encode_plan fields)
__device__ __forceinline__ bool dec_less(long long x, long long y) {
  char da[24], db[24];
  const int na = fmt_ll(x, da), nb = fmt_ll(y, db);
  for (int k = 0;; ++k) {
    const int u = k < na ? (unsigned char)da[k] : ':';
    const int v = k < nb ? (unsigned char)db[k] : ':';
    if (u != v) return u < v;
    if (k >= na && k >= nb) return false;
  }
}

template <int P>
__device__ __forceinline__ bool enc_less_t(const int (&a)[P], const int (&b)[P]) {
  int s = 0;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (a[i] != b[i]) return dec_less(s + a[i], s + b[i]);
    s += a[i];
  }
  return false;
}

template <int P>
__device__ __forceinline__ void unrank_bounded_t(long long rank, int L, const int (&caps)[P],
                                                 const long long* tbl, int (&out)[P]) {
  const int W = L + 1;
  int rem = L;
#pragma unroll
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

template <int P>
__device__ __forceinline__ bool next_bounded_t(int (&c)[P], const int (&caps)[P], const int (&sufcap)[P + 1]) {
  int suffix = c[P - 1];
#pragma unroll
  for (int j = P - 2; j >= 0; --j) {
    const int rest = suffix - 1;
    if (c[j] + 1 <= caps[j] && rest >= P - 1 - j && rest <= sufcap[j + 1]) {
      c[j] += 1;
      int r = rest;
#pragma unroll
      for (int k = j + 1; k < P - 1; ++k) {
        int v = r - sufcap[k + 1];
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

// Serial closed-form 1F1B (M >= P) for a compile-time P, state in registers.
// All threads of a warp share (P, M), so every phase test is warp-uniform.
template <int P>
__device__ __forceinline__ double sim_thread(int M, const double (&f)[P], const double (&bw)[P],
                                             const double (&sf)[P], const double (&sb)[P],
                                             const double (&dps)[P]) {
  double fr[P], chf[P], chb[P];
#pragma unroll
  for (int i = 0; i < P; ++i) fr[i] = chf[i] = chb[i] = 0.0;
  for (int t = 0; t < P; ++t) {  // warm-up: F(i, t-i) for i <= t
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
      if (i <= t) {
        fr[i] = (i == 0 ? fr[i] : dmax(fr[i], chf[i > 0 ? i - 1 : 0])) + f[i];
        if (i < P - 1) chf[i] = dmax(fr[i], chf[i]) + sf[i];
      }
    }
  }
  const int T = 2 * (M + P - 1);
  auto lvl = [&](auto par_tag, auto pred_tag, int t) {
    constexpr int PAR = decltype(par_tag)::value;
    constexpr bool PRED = decltype(pred_tag)::value;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      if (((PAR - i) & 1) == 0) {
        if (!PRED || (t >= 2 * P - i && t <= 2 * M - 2 + i)) {
          fr[i] = (i == 0 ? fr[i] : dmax(fr[i], chf[i > 0 ? i - 1 : 0])) + f[i];
          if (i < P - 1) chf[i] = dmax(fr[i], chf[i]) + sf[i];
        }
      } else {
        if (!PRED || (t >= 2 * P - 1 - i && t <= 2 * M + 2 * P - 3 - i)) {
          fr[i] = (i == P - 1 ? fr[i] : dmax(fr[i], chb[i < P - 1 ? i + 1 : 0])) + bw[i];
          if (i > 0) chb[i] = dmax(fr[i], chb[i]) + sb[i];
        }
      }
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  int t = P;
  for (; t < T && t < 2 * P; ++t) {
    if (t & 1) lvl(I1{}, std::true_type{}, t);
    else lvl(I0{}, std::true_type{}, t);
  }
  const int core_hi = 2 * M - 2;
  for (; t + 1 <= core_hi; t += 2) {
    lvl(I0{}, std::false_type{}, t);
    lvl(I1{}, std::false_type{}, t + 1);
  }
  for (; t < T; ++t) {
    if (t & 1) lvl(I1{}, std::true_type{}, t);
    else lvl(I0{}, std::true_type{}, t);
  }
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    v = dmax(v, fr[i]);
    v = dmax(v, fr[i] + dps[i]);
    if (i < P - 1) v = dmax(v, chf[i]);
    if (i > 0) v = dmax(v, chb[i]);
  }
  return v;
}

// Thread-per-candidate exhaustive evaluation (1F1B, M >= P, P <= 8): a warp
// owns one item of consecutive bounded ranks, each thread kExhChunk of them
// walked with next_bounded; per-thread exact argmin, then warp argmin.
template <int P>
__global__ void __launch_bounds__(128) k_exh_thread(Bufs b, const ExhItem* items, int n_items,
                                                    ExhRec* recs) {
  const int lane = threadIdx.x & 31;
  const int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (it >= n_items) return;
  const ExhItem w = items[it];
  const Leaf lf = b.leaves[w.leaf];
  const LeafGroup* lg = b.lg + lf.lg_off;
  const uint8_t* slots = b.layouts + lf.layout_off;
  const double* hop = b.hop + lf.B_idx * c_consts.n_links;
  const int L = c_consts.L;
  const long long* tbl = b.etbl + b.etbl_off[w.leaf];
  int caps[P], sufcap[P + 1];
  sufcap[P] = 0;
#pragma unroll
  for (int i = P - 1; i >= 0; --i) {
    caps[i] = b.ecap[lf.split_off + i];
    sufcap[i] = sufcap[i + 1] + caps[i];
  }
  double fl[P], bl[P], sf[P], sb[P];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const LeafGroup& row = lg[slots[i]];
    fl[i] = row.fl;
    bl[i] = row.bl;
    sf[i] = i + 1 < P ? hop[c_consts.link_pair[row.group][lg[slots[i + 1]].group]] : 0.0;
    sb[i] = i > 0 ? hop[c_consts.link_pair[lg[slots[i - 1]].group][row.group]] : 0.0;
  }
  const long long r0 = w.first + (long long)lane * kExhChunk;
  long long cnt = w.first + w.n - r0;
  if (cnt > kExhChunk) cnt = kExhChunk;
  double bt = 0.0;
  long long brank = -1;
  int bcomp[P], comp[P];
  long long sim = 0, ran = 0;
  const bool screen = b.log.exh == nullptr;  // the log needs every time
  const double Md = (double)lf.M;
  if (cnt > 0) unrank_bounded_t<P>(r0, L, caps, tbl, comp);
  for (long long k = 0; k < cnt; ++k) {
    if (k) next_bounded_t<P>(comp, caps, sufcap);
    double f[P], bw[P], dps[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const LeafGroup& row = lg[slots[i]];
      double layers = comp[i];
      if (i == 0) layers += c_consts.edge;
      if (i == P - 1) layers += c_consts.edge;
      f[i] = layers * fl[i];
      bw[i] = layers * bl[i];
      dps[i] = dp_sync(row, comp[i]);
    }
    ++sim;
    if (screen && brank >= 0) {
      // path lower bound (hp_search_core.cuh, nb_screen): a candidate above
      // this thread's best can neither win nor tie, so it is not simulated
      double A = 0.0, Bt = 0.0, lb = 0.0;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        lb = dmax(lb, A + Md * (f[i] + bw[i]) + dmax(Bt + dps[0], dps[i]));
        A = A + f[i] + sf[i];
        Bt = Bt + sf[i] + bw[i];
      }
      if (lb > bt * (1.0 + kScreenMargin)) continue;
    }
    const double t = sim_thread<P>(lf.M, f, bw, sf, sb, dps);
    if (b.log.exh) b.log.exh[b.log.exh_off[w.leaf] + r0 + k] = t;
    ++ran;
    if (brank < 0 || t < bt || (t == bt && enc_less_t<P>(comp, bcomp))) {
      bt = t;
      brank = r0 + k;
#pragma unroll
      for (int i = 0; i < P; ++i) bcomp[i] = comp[i];
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
    const long long orank = __shfl_xor_sync(0xffffffffu, brank, off);
    int ocomp[P];
#pragma unroll
    for (int i = 0; i < P; ++i) ocomp[i] = __shfl_xor_sync(0xffffffffu, bcomp[i], off);
    sim += __shfl_xor_sync(0xffffffffu, sim, off);
    ran += __shfl_xor_sync(0xffffffffu, ran, off);
    const bool take = orank >= 0 && (brank < 0 || ot < bt || (ot == bt && enc_less_t<P>(ocomp, bcomp)));
    if (take) {
      bt = ot;
      brank = orank;
#pragma unroll
      for (int i = 0; i < P; ++i) bcomp[i] = ocomp[i];
    }
  }
  if (lane == 0) {
    recs[it] = ExhRec{bt, brank, sim, w.leaf, brank >= 0 ? 1 : 0};
    if (b.ops) {
      atomicAdd(b.ops, (unsigned long long)ran * (unsigned long long)(8LL * P * lf.M - 4LL * lf.M));
      atomicAdd(b.ops + 1, (unsigned long long)ran);
      atomicAdd(b.ops + 3, (unsigned long long)(sim - ran));
    }
  }
}

// Per leaf: merge its item records (exact comparator, ties re-unranked).
__global__ void k_exh_merge(Bufs b, const ExhRec* recs, const int* rec_begin, const int* rec_end,
                            const int* ids, int n) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int li = ids[k];
  const Leaf lf = b.leaves[li];
  const int* caps = b.ecap + lf.split_off;
  const long long* tbl = b.etbl + b.etbl_off[li];
  HillState hs = b.hs[li];
  int* best = b.best + lf.split_off;
  int tmp[HP_MAX_STAGES];
  for (int r = rec_begin[k]; r < rec_end[k]; ++r) {
    const ExhRec e = recs[r];
    hs.simulated += e.sim;
    if (!e.has) continue;
    bool better = !hs.has_best || e.t < hs.best_time;
    if (!better && e.t == hs.best_time) {
      unrank_bounded(e.rank, c_consts.L, lf.P, caps, tbl, tmp);
      better = split_enc_less(lf.P, tmp, best);
    }
    if (better) {
      hs.has_best = 1;
      hs.best_time = e.t;
      unrank_bounded(e.rank, c_consts.L, lf.P, caps, tbl, best);
    }
  }
  b.hs[li] = hs;
}

// Memory-pruned compositions of every exhaustive leaf, counted analytically.
__global__ void k_exh_fix(Bufs b, const int* ids, int n, const long long* feas) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int li = ids[k];
  const Leaf lf = b.leaves[li];
  b.hs[li].pruned += contiguous_split_count(c_consts.L, lf.P) - feas[li];
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

#include "hp_default.cuh"

// Exact argmin over per-task bests of the default mode (one block).
__global__ void k_final_tasks(Bufs b, const TaskRes* res, const TaskDev* tasks, const int* tbest_rows,
                              int n, int* out_task, long long* counts) {
  __shared__ int s_best[1024];
  __shared__ long long s_c[3][1024];
  const int tid = threadIdx.x;
  int mine = -1;
  long long c0 = 0, c1 = 0, c2 = 0;
  auto less = [&](int x, int y) {
    const TaskRes& rx = res[x];
    const TaskRes& ry = res[y];
    const Leaf lx = b.leaves[rx.best_leaf], ly = b.leaves[ry.best_leaf];
    return cand_less(c_consts, rx.best_time, lx, b.lg + lx.lg_off, b.layouts + lx.layout_off,
                     tbest_rows + tasks[x].best_off, ry.best_time, ly, b.lg + ly.lg_off,
                     b.layouts + ly.layout_off, tbest_rows + tasks[y].best_off);
  };
  for (int k = tid; k < n; k += blockDim.x) {
    c0 += res[k].simulated;
    c1 += res[k].pruned_mem;
    c2 += res[k].pruned_bound;
    if (!res[k].has_best) continue;
    if (mine < 0 || less(k, mine)) mine = k;
  }
  s_best[tid] = mine;
  s_c[0][tid] = c0;
  s_c[1][tid] = c1;
  s_c[2][tid] = c2;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (tid < st) {
      int x = s_best[tid], y = s_best[tid + st];
      if (y >= 0 && (x < 0 || less(y, x))) s_best[tid] = y;
      for (int q = 0; q < 3; ++q) s_c[q][tid] += s_c[q][tid + st];
    }
    __syncthreads();
  }
  if (tid == 0) {
    *out_task = s_best[0];
    counts[0] = s_c[0][0];
    counts[1] = s_c[1][0];
    counts[2] = s_c[2][0];
  }
}

// ------------------------------------------------------------------ plan trace
//
// Winner post-processing (planner.cpp:681-684): every node time of ONE
// explicit plan, for the trace, busy times and in-flight counts of
// evaluate_plan_unchecked(record_trace = true) (evaluate.cpp:78-107,
// sim.cpp:63-195). One block, thread i = stage i; level-synchronous like the
// search evaluators (the unit-time ASAP order of hp_core.cuh stage_level,
// whose doubles are the reference's), with the neighbours' previous-level
// channel state exchanged through shared memory and every op's start / end
// and its send's start / end recorded. nodes: 8 arrays of P*M doubles,
// [F start, F end, B start, B end, SendF start, SendF end, SendB start,
// SendB end] at [stage * M + microbatch]. dur: per stage f, b, sf, sb, dps.
// fin: per stage final stage_free, forward / backward channel ends.
__global__ void __launch_bounds__(256) k_plan_trace(Bufs b, double* dur, double* nodes, double* fin) {
  __shared__ double s_chf[HP_MAX_STAGES], s_chb[HP_MAX_STAGES];
  __shared__ int s_nf[HP_MAX_STAGES], s_nb[HP_MAX_STAGES];
  const Leaf lf = b.leaves[0];
  const int P = lf.P, M = lf.M;
  const bool gpipe = lf.sched == 0;
  const int i = threadIdx.x;
  const size_t PM = (size_t)P * M;
  StageDur d{0.0, 0.0, 0.0, 0.0, 0.0};
  if (i < P) {
    stage_setup(c_consts, lf, b.lg + lf.lg_off, b.layouts + lf.layout_off, b.hop + lf.B_idx * c_consts.n_links, i,
                b.uni[lf.split_off + i], d);
    dur[5 * i + 0] = d.f;
    dur[5 * i + 1] = d.b;
    dur[5 * i + 2] = d.sf;
    dur[5 * i + 3] = d.sb;
    dur[5 * i + 4] = d.dps;
  }
  StageState st;
  stage_init(st);
  const int wb = gpipe ? M : min(P - i, M);
  double* row = nodes + (size_t)i * M;
  for (;;) {
    if (i < P) {
      s_chf[i] = st.chf;
      s_nf[i] = st.nf;
      s_chb[i] = st.chb;
      s_nb[i] = st.nb;
    }
    __syncthreads();
    const double lchf = i > 0 && i < P ? s_chf[i - 1] : 0.0;
    const int lnf = i > 0 && i < P ? s_nf[i - 1] : 0;
    const double rchb = i + 1 < P ? s_chb[i + 1] : 0.0;
    const int rnb = i + 1 < P ? s_nb[i + 1] : 0;
    const bool done = i >= P || stage_done(st, M);
    if (__syncthreads_and(done)) break;
    if (done) continue;
    // stage_level (hp_core.cuh) with every node recorded
    bool want_f;
    if (gpipe) want_f = st.nf < M;
    else want_f = st.nf < wb || (st.nf < M && st.nb > st.nf - wb);
    if (!want_f && st.nb >= M) continue;
    if (want_f) {
      if (i > 0 && !(lnf > st.nf)) continue;            // ready(), sim.cpp:102
      const double start = dmax(st.free_t, i > 0 ? lchf : 0.0);
      const double end = start + d.f;
      st.free_t = end;
      row[st.nf] = start;
      row[PM + st.nf] = end;
      if (i < P - 1) {                                  // sim.cpp:125-134
        const double ss = dmax(end, st.chf);
        const double e = ss + d.sf;
        st.chf = e;
        row[4 * PM + st.nf] = ss;
        row[5 * PM + st.nf] = e;
      }
      st.nf++;
    } else {
      if (i < P - 1 && !(rnb > st.nb)) continue;        // ready(), sim.cpp:103
      const double start = dmax(st.free_t, i < P - 1 ? rchb : 0.0);
      const double end = start + d.b;
      st.free_t = end;
      row[2 * PM + st.nb] = start;
      row[3 * PM + st.nb] = end;
      if (i > 0) {                                      // sim.cpp:135-145
        const double ss = dmax(end, st.chb);
        const double e = ss + d.sb;
        st.chb = e;
        row[6 * PM + st.nb] = ss;
        row[7 * PM + st.nb] = e;
      }
      st.nb++;
    }
  }
  if (i < P) {
    fin[3 * i + 0] = st.free_t;
    fin[3 * i + 1] = st.chf;
    fin[3 * i + 2] = st.chb;
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
  if (!v.empty()) {
    const size_t nb = v.size() * sizeof(T);
    if (char* h = a.stage(nb)) {
      std::memcpy(h, v.data(), nb);
      CK(cudaMemcpyAsync(p, h, nb, cudaMemcpyHostToDevice, a.stream));
    } else {
      CK(cudaMemcpyAsync(p, v.data(), nb, cudaMemcpyHostToDevice, a.stream));
    }
  }
  a.h2d_bytes += static_cast<double>(v.size() * sizeof(T));
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

// The per-thread stack (local memory) the kernels need, reserved once per
// context: without it the driver grows the device's local-memory pool at
// the first launch that needs more and may shrink it again afterwards, a
// device-wide reallocation on the critical path of every search (measured
// as a ~16 ms gap before the climb kernel's first item).
hph::Status reserve_local_memory() {
  size_t want = 0;
  const void* fns[] = {reinterpret_cast<const void*>(hpk::k_hill_async),
                       reinterpret_cast<const void*>(hpk::k_default),
                       reinterpret_cast<const void*>(hpk::k_async_seed),
                       reinterpret_cast<const void*>(hpk::k_seeds)};
  for (const void* f : fns) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, f) == cudaSuccess) want = std::max(want, fa.localSizeBytes);
  }
  size_t cur = 0;
  CK(cudaDeviceGetLimit(&cur, cudaLimitStackSize));
  if (cur < want) CK(cudaDeviceSetLimit(cudaLimitStackSize, want));
  return hph::Status{};
}

// Consts to __constant__ memory, with the group names (encode_plan's
// tie-break) copied to device memory first.
static hph::Status consts_to_device(Arena& a, const hph::Problem& p, Consts& c) {
  // a new search / evaluation: the previous one's staged copies are done
  // (every entry point synchronises its stream before returning)
  a.pinned_used = 0;
  std::vector<char> blob(p.names_blob.begin(), p.names_blob.end());
  char* d_names;
  hph::Status s = upload(a, "names", blob, &d_names);
  if (!s.ok()) return s;
  c.names = d_names;
  CK(cudaMemcpyToSymbolAsync(hpk::c_consts, &c, sizeof c, 0, cudaMemcpyHostToDevice, a.stream));
  return s;
}

// Shared-memory staging of the cost tables for a kernel that can give them
// `limit` bytes of dynamic shared memory (0 = read them from global).
static hpk::StagedTables staged(const hpk::Bufs& b, size_t limit) {
  hpk::StagedTables t{0, 0};
  const size_t lg = (size_t)b.n_lg * sizeof(LeafGroup), hop = (size_t)b.n_hop * sizeof(double);
  if (b.n_lg > 0 && lg % 16 == 0 && hop % 16 == 0 && hop > 0 && lg + hop <= limit) {
    t.lg_bytes = static_cast<unsigned>(lg);
    t.hop_bytes = static_cast<unsigned>(hop);
  }
  return t;
}

static size_t split_total_of(const std::vector<Leaf>& leaves) {
  size_t n = 0;
  for (const Leaf& lf : leaves) n += lf.P;
  return n;
}

static void launch_eval(int cls, const hpk::Bufs& b, const Work* items, const int* n_items,
                        int* next, int grid, cudaStream_t st) {
  switch (cls) {
    case 0: hpk::k_eval<2, true><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 1: hpk::k_eval<4, true><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 2: hpk::k_eval<6, true><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 3: hpk::k_eval<8, true><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 4: hpk::k_eval<1, false><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 5: hpk::k_eval<2, false><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    case 6: hpk::k_eval<3, false><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
    default: hpk::k_eval<8, false><<<grid, 256, 0, st>>>(b, items, n_items, next); break;
  }
}

static int async_grid(int sm_count, int threads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hpk::k_hill_async, threads, 0);
  if (const char* e = std::getenv("HP_ASYNC_BLOCKS")) per_sm = std::min(per_sm, std::atoi(e));  // tuning
  return sm_count * (per_sm > 0 ? per_sm : 1);
}

static hph::Status setup_tables(Arena& a, const hph::Problem& p, const std::vector<int>& my_leaves,
                                hpk::Bufs& b, std::vector<Leaf>& leaves, std::vector<int>& hill_ids,
                                std::vector<int>& exh_ids) {
  cudaStream_t st = a.stream;
  const int G = static_cast<int>(p.groups.size());
  const int nL = static_cast<int>(my_leaves.size());
  Consts c;
  hph::fill_consts(p, c);
  a.h2d_bytes = sizeof c;
  a.d2h_bytes = 0;
  hph::Status s_;
  if (!(s_ = consts_to_device(a, p, c)).ok()) return s_;

  // ---- host tables (split-independent, exact reference order)
  leaves.assign(nL, Leaf{});
  std::vector<LeafGroup> lgs;
  std::vector<int> hist_off(nL), nb_off(nL);
  std::vector<double> hop = hph::hop_table(p);
  int split_total = 0, hist_total = 0, nb_total = 0;
  hill_ids.clear();
  exh_ids.clear();
  // A leaf's G cost rows depend only on (dp, B, tp and nodes per group), so
  // leaves share them: one copy per distinct tuple (C3: ~600 for 63k leaves)
  struct KeyHash {
    size_t operator()(const std::vector<long long>& v) const {
      unsigned long long h = 1469598103934665603ULL;  // FNV-1a over the values
      for (long long x : v) h = (h ^ static_cast<unsigned long long>(x)) * 1099511628211ULL;
      return static_cast<size_t>(h);
    }
  };
  std::unordered_map<std::vector<long long>, int, KeyHash> row_of;
  row_of.reserve(4096);
  std::vector<long long> key(3 + 2 * G);
  for (int k = 0; k < nL; ++k) {
    Leaf& lf = leaves[k];
    lf = hph::device_leaf(p, my_leaves[k]);
    lf.split_off = split_total;
    split_total += lf.P;
    const hph::LeafHost& h = p.leaves[my_leaves[k]];
    key[0] = h.dp;
    key[1] = h.B_idx;
    key[2] = h.B;
    for (int g = 0; g < G; ++g) {
      key[3 + 2 * g] = hph::leaf_tp(p, h, g);
      key[4 + 2 * g] = hph::leaf_nodes(p, h, g);
    }
    auto it = row_of.find(key);
    if (it == row_of.end()) {
      it = row_of.emplace(key, static_cast<int>(lgs.size())).first;
      lgs.resize(lgs.size() + G);
      hph::leaf_rows(p, my_leaves[k], &lgs[lgs.size() - G]);
    }
    lf.lg_off = it->second;
    hist_off[k] = hist_total;
    nb_off[k] = nb_total;
    if (lf.mode == 0) {
      hist_total += 4 * p.model.num_layers;
      nb_total += 2 * (lf.P - 1);
    }
    if (lf.mode == 1) exh_ids.push_back(k);
    else hill_ids.push_back(k);
  }

  b = hpk::Bufs{};
  hph::Status s;
  Leaf* d_leaves;
  LeafGroup* d_lg;
  uint8_t* d_layouts;
  double* d_hop;
  int *d_hist_off, *d_nb_off;
  // padded to whole 16-byte units for the TMA bulk copy into shared memory
  while ((lgs.size() * sizeof(LeafGroup)) % 16) lgs.push_back(LeafGroup{});
  while ((hop.size() * sizeof(double)) % 16) hop.push_back(0.0);
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
  b.n_lg = static_cast<int>(lgs.size());
  b.n_hop = static_cast<int>(hop.size());
  b.hist_off = d_hist_off;
  b.nb_off = d_nb_off;
  if (!(s = scratch(a, "uni", split_total, &b.uni)).ok()) return s;
  if (!(s = scratch(a, "prop", split_total, &b.prop)).ok()) return s;
  if (!(s = scratch(a, "cur", split_total, &b.cur)).ok()) return s;
  if (!(s = scratch(a, "best", split_total, &b.best)).ok()) return s;
  if (!(s = scratch(a, "hist", hist_total, &b.hist)).ok()) return s;
  if (!(s = scratch(a, "tseed", 2 * (size_t)nL, &b.tseed)).ok()) return s;
  if (!(s = scratch(a, "nb", nb_total, &b.nb)).ok()) return s;
  if (!(s = scratch(a, "nb_ids", nb_total, &b.nb_ids)).ok()) return s;
  if (!(s = scratch(a, "lbs", split_total, &b.lbs)).ok()) return s;
  if (!(s = scratch(a, "lbn", split_total, &b.lbn)).ok()) return s;
  if (!(s = scratch(a, "memo_d", hist_total, &b.memo_d)).ok()) return s;
  if (!(s = scratch(a, "hs", nL, &b.hs)).ok()) return s;
  CK(cudaMemsetAsync(b.hs, 0, sizeof(HillState) * std::max(1, nL), st));
  return hph::Status{};
}

// Search-log sink buffers at the arena's current capacities.
static hph::Status log_open(Arena& a, hpk::LogSink& sink) {
  hph::Status s;
  sink = hpk::LogSink{};
  if (!(s = scratch(a, "log_ctr", 2, &sink.ctr)).ok()) return s;
  if (!(s = scratch(a, "log_vals", a.log.val_cap, &sink.vals)).ok()) return s;
  if (!(s = scratch(a, "log_segs", a.log.seg_cap, &sink.segs)).ok()) return s;
  sink.val_cap = a.log.val_cap;
  sink.seg_cap = a.log.seg_cap;
  CK(cudaMemsetAsync(sink.ctr, 0, 2 * sizeof(unsigned long long), a.stream));
  return s;
}

// Reads the segments back and orders them into per-key streams. On overflow
// grows the capacities and flags the search for a re-run.
static hph::Status log_collect(Arena& a, const hpk::LogSink& sink, size_t n_keys) {
  unsigned long long ctr[2];
  CK(cudaMemcpyAsync(ctr, sink.ctr, sizeof ctr, cudaMemcpyDeviceToHost, a.stream));
  CK(cudaStreamSynchronize(a.stream));
  if (ctr[0] > a.log.val_cap || ctr[1] > a.log.seg_cap) {
    a.log.overflow = true;
    a.log.val_cap = std::max(a.log.val_cap, ctr[0] + ctr[0] / 8 + 1024);
    a.log.seg_cap = std::max(a.log.seg_cap, ctr[1] + ctr[1] / 8 + 1024);
    return hph::Status{};
  }
  std::vector<hpk::LogSeg> segs(ctr[1]);
  std::vector<double> vals(ctr[0]);
  if (ctr[1]) CK(cudaMemcpy(segs.data(), sink.segs, sizeof(hpk::LogSeg) * ctr[1], cudaMemcpyDeviceToHost));
  if (ctr[0]) CK(cudaMemcpy(vals.data(), sink.vals, sizeof(double) * ctr[0], cudaMemcpyDeviceToHost));
  a.d2h_bytes += sizeof ctr + sizeof(hpk::LogSeg) * ctr[1] + sizeof(double) * ctr[0];
  std::sort(segs.begin(), segs.end(), [](const hpk::LogSeg& x, const hpk::LogSeg& y) {
    return x.key != y.key ? x.key < y.key : x.seq < y.seq;
  });
  a.log.streams.assign(n_keys, {});
  for (const hpk::LogSeg& g : segs) {
    if (g.key < 0 || static_cast<size_t>(g.key) >= n_keys)
      return hph::Status{HP_INTERNAL, "search log: bad segment key"};
    auto& v = a.log.streams[g.key];
    v.insert(v.end(), vals.begin() + g.off, vals.begin() + g.off + g.n);
  }
  return hph::Status{};
}

hph::Status search_full(Arena& a, const hph::Problem& p, const std::vector<int>& my_leaves,
                        SearchOut& out) {
  cudaStream_t st = a.stream;
  const int nL = static_cast<int>(my_leaves.size());
  hpk::Bufs b;
  std::vector<Leaf> leaves;
  std::vector<int> hill_ids, exh_ids;
  const auto t_setup = std::chrono::steady_clock::now();
  hph::Status s = setup_tables(a, p, my_leaves, b, leaves, hill_ids, exh_ids);
  if (!s.ok()) return s;
  if (std::getenv("HP_DEBUG_TIMING"))
    std::fprintf(stderr, "search_full: setup_tables %.2f ms (host)\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup).count());
  if (a.log.on) {
    a.log.reset();
    a.log.key_of = my_leaves;
    if (!(s = log_open(a, b.log)).ok()) return s;
  }

  // counters: [0..7] items per class, [8..15] next-item per class,
  // [16] n_active, [17] n_next, [18..19] one-off queue count / next
  int* d_ctr;
  if (!(s = scratch(a, "ctr", 32, &d_ctr)).ok()) return s;
  unsigned long long* d_ops;
  if (!(s = scratch(a, "ops", 4, &d_ops)).ok()) return s;
  CK(cudaMemsetAsync(d_ops, 0, 4 * sizeof(unsigned long long), st));
  b.ops = d_ops;
  const int grid = a.sm_count * 8;
  const int T = 128;

  auto eval_launch = [&](int cls, const Work* items, const int* n_items, int* next) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (a.time_evals) {
      a.event_pair(&e0, &e1);
      cudaEventRecord(e0, st);
    }
    launch_eval(cls, b, items, n_items, next, grid, st);
    if (a.time_evals) cudaEventRecord(e1, st);
    out.launches++;
    out.eval_launches++;
  };

  // ---- seeds
  if (nL > 0) {
    hpk::k_seeds<<<(nL + T - 1) / T, T, 0, st>>>(b, nL);
    out.launches++;
  }

  // ---- seed evaluation (uniform + proportional of hill / uniform-only leaves)
  std::vector<std::vector<Work>> seedq(hpk::NCLS);
  for (int k : hill_ids) {
    int cls = hpk::eval_class(leaves[k].P, leaves[k].M, leaves[k].sched == 0);
    int cpw = hpk::class_cpw(cls, leaves[k].P);
    int n = p.uniform_only ? 1 : 2;
    if (cpw >= n) {
      seedq[cls].push_back(Work{k, 0, 0, n, 0, nullptr});
    } else {
      seedq[cls].push_back(Work{k, 0, 0, 1, 0, nullptr});
      if (n == 2) seedq[cls].push_back(Work{k, 0, 1, 1, 0, nullptr});
    }
  }
  auto run_queues = [&](std::vector<std::vector<Work>>& qs, const char* tag) -> hph::Status {
    for (int cls = 0; cls < hpk::NCLS; ++cls) {
      if (qs[cls].empty()) continue;
      Work* d_items;
      std::string nm = std::string(tag) + std::to_string(cls);
      hph::Status s2 = upload(a, nm.c_str(), qs[cls], &d_items);
      if (!s2.ok()) return s2;
      int cnt[2] = {static_cast<int>(qs[cls].size()), 0};
      CK(cudaMemcpyAsync(d_ctr + 18, cnt, sizeof cnt, cudaMemcpyHostToDevice, st));
      eval_launch(cls, d_items, d_ctr + 18, d_ctr + 19);
      CK(cudaStreamSynchronize(st));  // the one-off count slot is reused per queue
    }
    return hph::Status{};
  };
  if (!(s = run_queues(seedq, "seedq")).ok()) return s;

  // ---- hill climb: one asynchronous persistent launch per evaluator class
  int* d_ids;
  std::vector<int> ids(hill_ids.begin(), hill_ids.end());
  if (!(s = upload(a, "hill_ids", ids, &d_ids)).ok()) return s;
  CK(cudaMemsetAsync(d_ctr, 0, 32 * sizeof(int), st));
  int* d_act0;
  if (!(s = scratch(a, "act0", ids.size(), &d_act0)).ok()) return s;
  if (!hill_ids.empty()) {
    hpk::k_hill_init<<<((int)ids.size() + T - 1) / T, T, 0, st>>>(b, d_ids, (int)ids.size(),
                                                                   p.uniform_only ? 1 : 0, d_act0,
                                                                   d_ctr + 16);
    out.launches++;
  }
  std::vector<int> climb;
  size_t n_items = 0;
  for (int k : hill_ids) {
    if (leaves[k].mode != 0) continue;
    climb.push_back(k);
    int cls = hpk::eval_class(leaves[k].P, leaves[k].M, leaves[k].sched == 0);
    // a step's items at the denser of its two possible evaluators (priority
    // items use lat_class): any ring holds at most one step per leaf, so this
    // sum bounds every ring's fill and a ring can never wrap onto an
    // unconsumed item
    int cpw = std::min(hpk::class_cpw(cls, leaves[k].P),
                       hpk::class_cpw(hpk::lat_class(leaves[k].P, cls), leaves[k].P));
    n_items += (2 * (leaves[k].P - 1) + cpw - 1) / cpw;
  }
  // Longest steps first: the seeding order is the initial queue order, so
  // the slowest leaves start early instead of forming the tail.
  std::stable_sort(climb.begin(), climb.end(), [&](int x, int y) {
    return (double)leaves[x].M * leaves[x].P > (double)leaves[y].M * leaves[y].P;
  });
  if (std::getenv("HP_DEBUG_TRACE")) {
    if (!(s = scratch(a, "trace", 1 + 2 * (1ULL << 22), &b.trace)).ok()) return s;
    CK(cudaMemsetAsync(b.trace, 0, sizeof(unsigned long long), st));
    // HP_DEBUG_TRACE_ITEMS=n: item events of every n-th warp of the climb kernel
    b.trace_items = std::getenv("HP_DEBUG_TRACE_ITEMS") ? std::max(1, std::atoi(std::getenv("HP_DEBUG_TRACE_ITEMS"))) : 0;
  }
  // One queue and one persistent kernel for every evaluator class. A leaf
  // has at most one step's items in the rings, so n_items bounds the fill.
  hpk::AsyncQ q{};
  int* d_abort;
  if (!(s = scratch(a, "q_abort", 1, &d_abort)).ok()) return s;
  CK(cudaMemsetAsync(d_abort, 0, sizeof(int), st));
  q.abort = d_abort;
  if (!climb.empty()) {
    if (!(s = scratch(a, "q_pending", nL, &q.pending)).ok()) return s;
    int* d_climb;
    if (!(s = upload(a, "climb_ids", climb, &d_climb)).ok()) return s;
    // unread slots of a ring: its unclaimed items (one step per climbing
    // leaf: <= n_items) + one held ticket per resident warp, + slack
    const size_t qcap = 2 * n_items + (size_t)a.sm_count * 64 + 65536;
    for (int lv = 0; lv < hpk::kRings; ++lv) {
      std::string nm = "q_slots" + std::to_string(lv);
      if (!(s = scratch(a, nm.c_str(), qcap, &q.slots[lv])).ok()) return s;
      nm = "q_seq" + std::to_string(lv);
      if (!(s = scratch(a, nm.c_str(), qcap, &q.seq[lv])).ok()) return s;
      CK(cudaMemsetAsync(q.seq[lv], 0, sizeof(unsigned long long) * qcap, st));
    }
    unsigned long long* d_q;
    if (!(s = scratch(a, "q_ctr", 8, &d_q)).ok()) return s;
    CK(cudaMemsetAsync(d_q, 0, 8 * sizeof(unsigned long long), st));
    q.head[0] = d_q;
    q.head[1] = d_q + 1;
    q.head[2] = d_q + 2;
    q.tail[0] = d_q + 3;
    q.tail[1] = d_q + 4;
    q.tail[2] = d_q + 5;
    q.active = reinterpret_cast<int*>(d_q + 6);
    q.progress = d_q + 7;
    q.cap = qcap;
    // a leaf moves to ring 1 once its climb has run 4096 levels (the third
    // step of a P = 96, M = 1536 climb): continuing climbs go before the
    // first steps still queued, which shortens every long chain. C3 full,
    // 2 alternating runs per value (2^17 -> 4096): 1 GPU 198.1 -> 192.1 ms,
    // 2 GPUs 126.5 -> 121.8, 4 GPUs 93.8 -> 89.5; 0 (one ring for all):
    // 2 GPUs 126.8.
    q.hi_levels = 4096;
    q.r1_thr = -1;  // set below from the grid (one item per SM of backlog)
    if (const char* e = std::getenv("HP_R1_THR")) q.r1_thr = std::max(0, std::atoi(e));  // tuning
    q.r0_thr = -1;
    if (const char* e = std::getenv("HP_R0_THR")) q.r0_thr = std::atoi(e);  // tuning
    if (const char* e = std::getenv("HP_HI_LEVELS")) q.hi_levels = std::atoll(e);  // tuning
    int threads = HP_ASYNC_MAXT;
    if (const char* e = std::getenv("HP_ASYNC_THREADS")) threads = std::atoi(e);  // tuning
    const int grid = async_grid(a.sm_count, threads);
    // C3 full sweep, 1 GPU, 3 alternating A/B runs: 0 -> 236.8 ms, 148 -> 233.8 ms,
    // 300 -> 236.5 ms
    if (q.r1_thr < 0) q.r1_thr = grid;
    q.lat = std::getenv("HP_NO_LAT") ? 0 : 1;  // tuning
    // critical leaves: longest expected climbs (P^2 M) while their neighbour
    // items (~P-1 per step after the screen, one per warp at K = 4) fit the
    // resident warps
    {
      q.lead = (threads >= 128 && !std::getenv("HP_NO_LEAD")) ? 1 : 0;  // tuning
      // A shard of a 4+-GPU sweep ends on its critical climbs, not its bulk:
      // give them half of the SMs alone (C3 on 4 GPUs 128 -> 123 ms; on one
      // GPU the bulk dominates and the reservation costs 242 -> 275 ms).
      q.crit_sms = a.shard_count >= 4 ? grid / 2 : 0;
      if (const char* e = std::getenv("HP_CRIT_SMS")) q.crit_sms = std::min(grid, std::max(0, std::atoi(e)));  // tuning
      if (q.crit_sms > 0) q.lead = 1;
      // ... and those SMs' warps 0-3 serve ring 0 only, so a critical item
      // never waits behind a bulk item there, while warps 4-7 run bulk
      // (C3 on 4 GPUs, 2 alternating runs: mode 0 89.5 ms, 1 87.4, 2 105.0;
      // 2 GPUs with the reservation in mode 1: 124.0 -> 123.2, not adopted)
      q.crit_mode = 1;
      if (const char* e = std::getenv("HP_CRIT_MODE")) q.crit_mode = std::atoi(e);  // tuning
      // rings 1 and 2 need servers: with every SM reserved, warps 4-7 serve
      // them (mode 2 would leave none), and blocks of <= 4 warps have no
      // warps 4-7 at all
      if (q.crit_mode == 2 && q.crit_sms >= grid) q.crit_mode = 1;
      if (threads <= 128) q.crit_mode = 0;
      long long budget = (long long)(q.crit_sms > 0 ? q.crit_sms : grid) * (q.lead ? 4 : threads / 32);
      if (const char* e = std::getenv("HP_CRIT_WARPS")) budget = std::atoll(e);  // tuning
      std::vector<int> byest(climb);
      std::stable_sort(byest.begin(), byest.end(), [&](int x, int y) {
        return (double)leaves[x].P * leaves[x].P * leaves[x].M > (double)leaves[y].P * leaves[y].P * leaves[y].M;
      });
      std::vector<unsigned char> crit(nL, 0);
      long long used = 0;
      for (int k : byest) {
        if (used + leaves[k].P - 1 > budget) break;
        used += leaves[k].P - 1;
        crit[k] = 1;
      }
      unsigned char* d_crit;
      if (!(s = upload(a, "crit", crit, &d_crit)).ok()) return s;
      q.crit = d_crit;
    }
    cudaEvent_t h0 = nullptr, h1 = nullptr;
    if (a.time_evals) {
      a.event_pair(&h0, &h1);
      CK(cudaEventRecord(h0, st));
    }
    const int n = static_cast<int>(climb.size());
    hpk::Bufs bh = b;
    bh.nb_rows = b.log.vals == nullptr ? 1 : 0;  // the screen runs unless the log is recorded
    if (std::getenv("HP_NB_ROWS_OFF")) bh.nb_rows = 0;  // tuning: screened neighbours recompute their durations
    hpk::k_async_seed<<<(n * 32 + T - 1) / T, T, 0, st>>>(bh, q, d_climb, n);
    // one block per SM: up to 160 KB of tables in shared memory
    const hpk::StagedTables tt = staged(bh, std::getenv("HP_NO_STAGE") ? 0 : 160 * 1024);  // (knob: A/B)
    const size_t dsm = tt.lg_bytes + tt.hop_bytes;
    CK(cudaFuncSetAttribute(hpk::k_hill_async, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    const bool dbg_ph = std::getenv("HP_DEBUG_PHASES") != nullptr;  // diagnostics
    if (dbg_ph) {
      static const int on = 1;
      static const unsigned long long z[16] = {};
      CK(cudaMemcpyToSymbolAsync(hpk::c_dbg_phases, &on, sizeof(int), 0, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyToSymbolAsync(hpk::g_phase, z, sizeof z, 0, cudaMemcpyHostToDevice, st));
    }
    hpk::k_hill_async<<<grid, threads, dsm, st>>>(bh, q, tt);
    if (dbg_ph) {
      unsigned long long ph[16];
      CK(cudaMemcpyFromSymbolAsync(ph, hpk::g_phase, sizeof ph, 0, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::fprintf(stderr, "HP_DEBUG_PHASES Mcycles: screen rows %.1f scan %.1f slots %.1f list %.1f | "
                   "step loads+memo %.1f rest %.1f fence %.1f | steps %llu | items %llu: pop %.1f eval %.1f done %.1f\n",
                   ph[0] / 1e6, ph[1] / 1e6, ph[2] / 1e6, ph[3] / 1e6, ph[4] / 1e6, ph[5] / 1e6, ph[6] / 1e6,
                   ph[7], ph[11], ph[8] / 1e6, ph[9] / 1e6, ph[10] / 1e6);
    }
    if (h1) CK(cudaEventRecord(h1, st));
    out.launches += 2;
    out.eval_launches++;
  }
  out.hill_iterations = 0;
  if (b.trace) {
    CK(cudaStreamSynchronize(st));
    unsigned long long n = 0;
    CK(cudaMemcpy(&n, b.trace, sizeof n, cudaMemcpyDeviceToHost));
    n = std::min<unsigned long long>(n, 1ULL << 22);
    std::vector<unsigned long long> tr(2 * n);
    CK(cudaMemcpy(tr.data(), b.trace + 1, sizeof(unsigned long long) * 2 * n, cudaMemcpyDeviceToHost));
    if (FILE* fp = std::fopen(std::getenv("HP_DEBUG_TRACE"), "wb")) {
      std::fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fp);
      std::fclose(fp);
    }
  }
  if (!climb.empty()) {
    int abort_flag = 0;
    CK(cudaMemcpyAsync(&abort_flag, q.abort, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (abort_flag) {
      // ring counters for the report: head/tail per ring, leaves climbing
      unsigned long long ctr[7] = {0, 0, 0, 0, 0, 0, 0};
      cudaMemcpy(ctr, q.head[0], sizeof ctr, cudaMemcpyDeviceToHost);
      char msg[256];
      std::snprintf(msg, sizeof msg,
                    "%s (head %llu/%llu/%llu tail %llu/%llu/%llu active %d)",
                    abort_flag == 2 ? "hill-climb work ring overwrote an unread item"
                                    : "watchdog: hill-climb work queue made no progress for ~35 s",
                    ctr[0], ctr[1], ctr[2], ctr[3], ctr[4], ctr[5], (int)(ctr[6] & 0xffffffffu));
      return hph::Status{HP_INTERNAL, msg};
    }
  }

  // ---- exhaustive leaves: bounded compositions only (memory gate solved
  // analytically), thread-per-candidate for small P, warp segments otherwise
  if (!exh_ids.empty()) {
    const int L = p.model.num_layers;
    std::vector<int> etbl_off(nL, 0);
    size_t etbl_total = 0;
    for (int k : exh_ids) {
      etbl_off[k] = static_cast<int>(etbl_total);
      etbl_total += (size_t)(leaves[k].P + 1) * (L + 1);
    }
    int* d_etbl_off;
    long long* d_etbl;
    int* d_ecap;
    long long* d_feas;
    int* d_exh_ids;
    if (!(s = upload(a, "etbl_off", etbl_off, &d_etbl_off)).ok()) return s;
    if (!(s = scratch(a, "etbl", etbl_total, &d_etbl)).ok()) return s;
    if (!(s = scratch(a, "ecap", split_total_of(leaves), &d_ecap)).ok()) return s;
    if (!(s = scratch(a, "feas", nL, &d_feas)).ok()) return s;
    if (!(s = upload(a, "exh_ids", exh_ids, &d_exh_ids)).ok()) return s;
    b.etbl = d_etbl;
    b.etbl_off = d_etbl_off;
    b.ecap = d_ecap;
    const int ne = static_cast<int>(exh_ids.size());
    hpk::k_exh_prep<<<(ne + T - 1) / T, T, 0, st>>>(b, d_exh_ids, ne, d_feas, d_etbl, d_ecap);
    out.launches++;
    std::vector<long long> feas(nL, 0);
    CK(cudaMemcpyAsync(feas.data(), d_feas, sizeof(long long) * nL, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    a.d2h_bytes += sizeof(long long) * nL;
    if (a.log.on) {  // per-rank times of the exhaustive leaves for the log
      a.log.exh_off.assign(nL, -1);
      long long tot = 0;
      for (int k : exh_ids) {
        a.log.exh_off[k] = tot;
        tot += feas[k];
      }
      long long* d_xo;
      if (!(s = upload(a, "log_exh_off", a.log.exh_off, &d_xo)).ok()) return s;
      if (!(s = scratch(a, "log_exh", (size_t)tot, &b.log.exh)).ok()) return s;
      b.log.exh_off = d_xo;
      a.log.exh.resize(tot);
    }

    // thread path: 1F1B with M >= P and P <= 8
    std::vector<std::vector<hpk::ExhItem>> titems(9);
    std::vector<std::vector<int>> tleaf(9);
    std::vector<int> generic;
    const long long per_item = 32LL * hpk::kExhChunk;
    for (int k : exh_ids) {
      const Leaf& lf = leaves[k];
      if (feas[k] == 0) continue;
      if (lf.sched == HP_1F1B && lf.M >= lf.P && lf.P <= 8) {
        tleaf[lf.P].push_back(k);
        for (long long r = 0; r < feas[k]; r += per_item)
          titems[lf.P].push_back(hpk::ExhItem{k, 0, r, std::min(per_item, feas[k] - r)});
      } else {
        generic.push_back(k);
      }
    }
    size_t nrec = 0;
    for (int P = 1; P <= 8; ++P) nrec += titems[P].size();
    if (nrec > 0) {
      hpk::ExhRec* d_recs;
      if (!(s = scratch(a, "exh_recs", nrec, &d_recs)).ok()) return s;
      std::vector<int> mids, rb, re;
      size_t off = 0;
      for (int P = 1; P <= 8; ++P) {
        if (titems[P].empty()) continue;
        hpk::ExhItem* d_items;
        std::string nm = "exh_items" + std::to_string(P);
        if (!(s = upload(a, nm.c_str(), titems[P], &d_items)).ok()) return s;
        const int ni = static_cast<int>(titems[P].size());
        const int blocks = (ni * 32 + 127) / 128;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (a.time_evals) {
          a.event_pair(&e0, &e1);
          cudaEventRecord(e0, st);
        }
        switch (P) {
          case 1: hpk::k_exh_thread<1><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
          case 2: hpk::k_exh_thread<2><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
          case 3: hpk::k_exh_thread<3><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
          case 4: hpk::k_exh_thread<4><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
          case 5: hpk::k_exh_thread<5><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
          case 6: hpk::k_exh_thread<6><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
          case 7: hpk::k_exh_thread<7><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
          default: hpk::k_exh_thread<8><<<blocks, 128, 0, st>>>(b, d_items, ni, d_recs + off); break;
        }
        if (a.time_evals) cudaEventRecord(e1, st);
        out.launches++;
        out.eval_launches++;
        // items of one leaf are contiguous
        size_t j = 0;
        while (j < titems[P].size()) {
          int leaf = titems[P][j].leaf;
          size_t j2 = j;
          while (j2 < titems[P].size() && titems[P][j2].leaf == leaf) ++j2;
          mids.push_back(leaf);
          rb.push_back(static_cast<int>(off + j));
          re.push_back(static_cast<int>(off + j2));
          j = j2;
        }
        off += titems[P].size();
      }
      int *d_mids, *d_rb, *d_re;
      if (!(s = upload(a, "exh_mids", mids, &d_mids)).ok()) return s;
      if (!(s = upload(a, "exh_rb", rb, &d_rb)).ok()) return s;
      if (!(s = upload(a, "exh_re", re, &d_re)).ok()) return s;
      const int nm = static_cast<int>(mids.size());
      hpk::k_exh_merge<<<(nm + T - 1) / T, T, 0, st>>>(b, d_recs, d_rb, d_re, d_mids, nm);
      out.launches++;
    }

    // generic path: warp segments over bounded ranks, in chunks
    if (!generic.empty()) {
      const long long kChunk = 1 << 24;
      double* d_x;
      if (!(s = scratch(a, "xbuf", kChunk, &d_x)).ok()) return s;
      b.xbuf = d_x;
      size_t e = 0;
      long long pos = 0;
      while (e < generic.size()) {
        std::vector<std::vector<Work>> q(hpk::NCLS);
        std::vector<hpk::ExhSpan> spans;
        long long used = 0;
        while (e < generic.size() && used < kChunk) {
          int k = generic[e];
          const Leaf& lf = leaves[k];
          long long total = feas[k];
          long long take = std::min(total - pos, kChunk - used);
          int cls = hpk::eval_class(lf.P, lf.M, lf.sched == 0);
          int cpw = hpk::class_cpw(cls, lf.P);
          for (long long j = 0; j < take; j += cpw)
            q[cls].push_back(Work{k, 2, pos + j, (int)std::min<long long>(cpw, take - j), (int)(used + j), nullptr});
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
    hpk::k_exh_fix<<<(ne + T - 1) / T, T, 0, st>>>(b, d_exh_ids, ne, d_feas);
    out.launches++;
  }

  if (a.log.on) {
    if (!(s = log_collect(a, b.log, my_leaves.size())).ok()) return s;
    a.log.tseed.resize(2 * (size_t)nL);
    if (nL) CK(cudaMemcpy(a.log.tseed.data(), b.tseed, sizeof(double) * 2 * nL, cudaMemcpyDeviceToHost));
    if (!a.log.exh.empty())
      CK(cudaMemcpy(a.log.exh.data(), b.log.exh, sizeof(double) * a.log.exh.size(), cudaMemcpyDeviceToHost));
    a.d2h_bytes += sizeof(double) * (2.0 * nL + a.log.exh.size());
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
  unsigned long long ops[4] = {0, 0, 0, 0};
  CK(cudaMemcpy(ops, d_ops, sizeof ops, cudaMemcpyDeviceToHost));
  out.eval_fp64_ops = static_cast<double>(ops[0]);
  out.dev_simulated = static_cast<long long>(ops[1]);
  out.dev_aborted = static_cast<long long>(ops[2]);
  out.dev_screened = static_cast<long long>(ops[3]);
  if (a.time_evals) out.eval_ms = a.drain_events();
  a.d2h_bytes += sizeof(int) + sizeof counts + sizeof ops;
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
    a.d2h_bytes += sizeof hs + sizeof(int) * lf.P;
  }
  out.h2d_bytes = a.h2d_bytes;
  out.d2h_bytes = a.d2h_bytes;
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
  hph::Status s_;
  c.n_B = n;
  if (!(s_ = consts_to_device(a, p, c)).ok()) return s_;
  std::vector<Leaf> leaves(n);
  std::vector<LeafGroup> lgs;
  std::vector<uint8_t> layouts;
  std::vector<int> splits;
  std::vector<double> hop((size_t)n * p.links.size());
  std::vector<std::vector<Work>> q(hpk::NCLS);
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
    lf.sched = pl.schedule;
    for (size_t l = 0; l < p.links.size(); ++l) hop[(size_t)k * p.links.size() + l] = hph::hop_time(p, (int)l, B);
    for (int i = 0; i < P; ++i) {
      const hp_stage& s = pl.stages[i];
      layouts.push_back(static_cast<uint8_t>(i));
      splits.push_back(s.layer_end - s.layer_begin);
      lgs.push_back(hph::leaf_group(p, s.group, s.tp_degree, B, s.dp_degree, s.nodes_used));
    }
    q[hpk::eval_class(P, lf.M, lf.sched == HP_GPIPE)].push_back(Work{k, 0, 0, 1, 0, nullptr});
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
  for (int cls = 0; cls < hpk::NCLS; ++cls) {
    if (q[cls].empty()) continue;
    Work* d_items;
    std::string nm = "e_q" + std::to_string(cls);
    if (!(s = upload(a, nm.c_str(), q[cls], &d_items)).ok()) return s;
    int cnt[2] = {static_cast<int>(q[cls].size()), 0};
    CK(cudaMemcpyAsync(d_ctr, cnt, sizeof cnt, cudaMemcpyHostToDevice, st));
    launch_eval(cls, b, d_items, d_ctr, d_ctr + 1, a.sm_count * 8, st);
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaGetLastError());
  std::vector<double> t(2 * (size_t)n);
  CK(cudaMemcpyAsync(t.data(), b.tseed, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int k = 0; k < n; ++k) out_times[k] = t[2 * (size_t)k];
  return hph::Status{};
}


// Node times of one explicit plan on the GPU (k_plan_trace), for the winner
// post-processing of hp_evaluate_plan_full (hp_eval.cpp).
hph::Status plan_node_times(Arena& a, const hph::Problem& p, const hp_plan& pl, PlanNodes& out) {
  cudaStream_t st = a.stream;
  Consts c;
  hph::fill_consts(p, c);
  hph::Status s_;
  c.n_B = 1;
  if (!(s_ = consts_to_device(a, p, c)).ok()) return s_;
  const int P = pl.n_stages;
  const long long M = pl.micro_batches_per_dp_replica;
  const int64_t B = pl.micro_batch_size > 0 ? pl.micro_batch_size : p.train.micro_batch_size;
  std::vector<Leaf> leaves(1);
  Leaf& lf = leaves[0];
  lf.task = -1;
  lf.P = P;
  lf.M = static_cast<int>(M);
  lf.dp = pl.stages[0].dp_degree;
  lf.B = B;
  lf.B_idx = 0;
  lf.layout_off = 0;
  lf.split_off = 0;
  lf.lg_off = 0;
  lf.mode = 3;
  lf.sched = pl.schedule;
  std::vector<LeafGroup> lgs;
  std::vector<uint8_t> layouts;
  std::vector<int> counts;
  std::vector<double> hop(p.links.size());
  for (size_t l = 0; l < p.links.size(); ++l) hop[l] = hph::hop_time(p, (int)l, B);
  for (int i = 0; i < P; ++i) {
    const hp_stage& s = pl.stages[i];
    layouts.push_back(static_cast<uint8_t>(i));
    counts.push_back(s.layer_end - s.layer_begin);
    lgs.push_back(hph::leaf_group(p, s.group, s.tp_degree, B, s.dp_degree, s.nodes_used));
  }
  hpk::Bufs b{};
  hph::Status s;
  Leaf* d_leaves;
  LeafGroup* d_lg;
  uint8_t* d_layouts;
  double* d_hop;
  int* d_counts;
  if (!(s = upload(a, "t_leaves", leaves, &d_leaves)).ok()) return s;
  if (!(s = upload(a, "t_lg", lgs, &d_lg)).ok()) return s;
  if (!(s = upload(a, "t_layouts", layouts, &d_layouts)).ok()) return s;
  if (!(s = upload(a, "t_hop", hop, &d_hop)).ok()) return s;
  if (!(s = upload(a, "t_counts", counts, &d_counts)).ok()) return s;
  b.leaves = d_leaves;
  b.lg = d_lg;
  b.layouts = d_layouts;
  b.hop = d_hop;
  b.uni = d_counts;
  const size_t PM = (size_t)P * (size_t)M;
  double *d_dur, *d_nodes, *d_fin;
  if (!(s = scratch(a, "t_dur", 5 * (size_t)P, &d_dur)).ok()) return s;
  if (!(s = scratch(a, "t_nodes", 8 * PM, &d_nodes)).ok()) return s;
  if (!(s = scratch(a, "t_fin", 3 * (size_t)P, &d_fin)).ok()) return s;
  const int threads = ((P + 31) / 32) * 32;
  hpk::k_plan_trace<<<1, threads, 0, st>>>(b, d_dur, d_nodes, d_fin);
  CK(cudaGetLastError());
  out.P = P;
  out.M = M;
  out.dur.resize(5 * (size_t)P);
  out.nodes.resize(8 * PM);
  out.fin.resize(3 * (size_t)P);
  CK(cudaMemcpyAsync(out.dur.data(), d_dur, sizeof(double) * out.dur.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out.nodes.data(), d_nodes, sizeof(double) * out.nodes.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out.fin.data(), d_fin, sizeof(double) * out.fin.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return hph::Status{};
}

}  // namespace hpd

// ---------------------------------------------------------------- roofline
//
// Microbenchmarks for the FP64 roofline denominator (MEASURED_PEAKS.json has
// no FP64 figure). k_peak_dadd: 8 independent DADD chains per thread, full
// occupancy. k_peak_mix: 4 independent copies of the evaluator's node update
// st = max(a, r); a = st + d; c = max(a, c) + s (4 algorithmic add/max ops).
namespace hpk {

__global__ void k_peak_dadd(double* out, int iters, double y) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = x[k] + y;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == -1.0) out[threadIdx.x] = s;
}

__global__ void k_peak_mix(double* out, int iters, double d, double sd) {
  double a[4], c[4], r[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = threadIdx.x * 1e-9 + k;
    c[k] = k * 0.5;
    r[k] = k * 0.25;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double st = dmax(a[k], r[k]);
      a[k] = st + d;
      c[k] = dmax(a[k], c[k]) + sd;
      r[k] = c[(k + 1) & 3];
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += a[k] + c[k];
  if (s == -1.0) out[threadIdx.x] = s;
}

}  // namespace hpk

extern "C" int hp_fp64_peak(int device, double* dadd_ops_per_s, double* mix_ops_per_s) {
  if (cudaSetDevice(device) != cudaSuccess) return HP_CUDA;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d_out = nullptr;
  if (cudaMalloc(&d_out, 1024 * sizeof(double)) != cudaSuccess) return HP_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float best_add = 1e30f, best_mix = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    hpk::k_peak_dadd<<<blocks, threads>>>(d_out, iters, 1e-12);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best_add = ms < best_add ? ms : best_add;
    cudaEventRecord(e0);
    hpk::k_peak_mix<<<blocks, threads>>>(d_out, iters, 1e-12, 2e-12);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best_mix = ms < best_mix ? ms : best_mix;
  }
  double n = (double)blocks * threads * iters;
  if (dadd_ops_per_s) *dadd_ops_per_s = n * 8 / (best_add * 1e-3);
  if (mix_ops_per_s) *mix_ops_per_s = n * 16 / (best_mix * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_out);
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_CUDA;
}

namespace hpd {

// Default (time-bound-pruned) mode over whole tasks `my_tasks` (reference
// order). When !have_bound the probe pass runs first (planner.cpp:640-651)
// over the same tasks; its min is the global bound (a sharded caller passes
// the all-reduced min instead).
hph::Status search_default(Arena& a, const hph::Problem& p, const std::vector<int>& my_tasks,
                           bool have_bound, double bound, bool probe_only, SearchOut& out) {
  cudaStream_t st = a.stream;
  std::vector<int> my_leaves;
  std::vector<hpk::TaskDev> tasks;
  std::vector<int> task_ids;  // device task position -> global task
  int best_total = 0;
  for (int ti : my_tasks) {
    const hph::Task& t = p.tasks[ti];
    hpk::TaskDev td;
    td.leaf_begin = static_cast<int>(my_leaves.size());
    for (int li = t.leaf_begin; li < t.leaf_end; ++li) my_leaves.push_back(li);
    td.leaf_end = static_cast<int>(my_leaves.size());
    td.pp = t.pp;
    td.best_off = best_total;
    best_total += t.pp;
    if (td.leaf_end > td.leaf_begin) {
      tasks.push_back(td);
      task_ids.push_back(ti);
    }
  }
  hpk::Bufs b;
  std::vector<Leaf> leaves;
  std::vector<int> hill_ids, exh_ids;
  hph::Status s = setup_tables(a, p, my_leaves, b, leaves, hill_ids, exh_ids);
  if (!s.ok()) return s;
  const int nT = static_cast<int>(tasks.size());
  out.global_bound = have_bound ? bound : std::numeric_limits<double>::infinity();
  if (nT == 0) return hph::Status{};
  hpk::TaskDev* d_tasks;
  if (!(s = upload(a, "d_tasks", tasks, &d_tasks)).ok()) return s;
  hpk::TaskRes* d_res;
  int* d_tbest;
  if (!(s = scratch(a, "d_tres", nT, &d_res)).ok()) return s;
  if (!(s = scratch(a, "d_tbest", best_total, &d_tbest)).ok()) return s;
  // Tasks run longest expected first (sum over leaves of P*M: the cost of a
  // simulation, plus the gating of the leaf); the order is free, since the
  // reduction (k_final_tasks) and the log are keyed by task.
  std::vector<int> order(nT);
  std::vector<double> est(nT, 0.0);
  for (int k = 0; k < nT; ++k) {
    order[k] = k;
    for (int j = tasks[k].leaf_begin; j < tasks[k].leaf_end; ++j)
      est[k] += (double)leaves[j].P * (double)leaves[j].M + 64.0 * leaves[j].P * leaves[j].P;
  }
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return est[x] > est[y]; });
  int* d_order;
  if (!(s = upload(a, "d_order", order, &d_order)).ok()) return s;
  const int threads = hpk::DEF_THREADS;
  const hpk::StagedTables tt = staged(b, std::getenv("HP_NO_STAGE") ? 0 : 80 * 1024);  // (knob: A/B)
  const size_t dsm = tt.lg_bytes + tt.hop_bytes;
  // (always set: the default cap on dynamic shared memory is 48 KB minus the
  // kernel's static shared memory)
  CK(cudaFuncSetAttribute(hpk::k_default, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hpk::k_default, threads, dsm);
  if (std::getenv("HP_DEBUG_LAUNCH"))
    std::fprintf(stderr, "k_default: tasks %d leaves %zu rows %d hop %d dsm %zu per_sm %d\n", nT, my_leaves.size(),
                 b.n_lg, b.n_hop, dsm, per_sm);
  const int blocks = std::min(nT, a.sm_count * std::max(1, per_sm));
  hpk::DefScratch sc;
  sc.CH = hpk::DEF_CH;
  const size_t nb = (size_t)blocks;
  const size_t nl = std::max<size_t>(1, my_leaves.size());
  hpk::DefSeeds sd;
  if (!(s = scratch(a, "sd_flag", 2 * nl, &sd.flag)).ok()) return s;
  if (!(s = scratch(a, "sd_low", 2 * nl, &sd.low)).ok()) return s;
  if (!(s = scratch(a, "sd_done", 2 * nl, &sd.done)).ok()) return s;
  if (!(s = scratch(a, "sd_xmem", nl, &sd.xmem)).ok()) return s;
  if (!(s = scratch(a, "sd_xfeas", nl, &sd.xfeas)).ok()) return s;
  if (!(s = scratch(a, "sd_xmin", nl, &sd.xmin)).ok()) return s;
  if (!(s = scratch(a, "sc_ids", nb * sc.CH, &sc.ids)).ok()) return s;
  if (!(s = scratch(a, "sc_lower", nb * sc.CH, &sc.lower)).ok()) return s;
  if (!(s = scratch(a, "sc_times", nb * sc.CH, &sc.times)).ok()) return s;
  if (!(s = scratch(a, "sc_flag", nb * sc.CH, &sc.flag)).ok()) return s;
  if (!(s = scratch(a, "sc_dec", nb * sc.CH, &sc.dec)).ok()) return s;
  int* d_next;
  if (!(s = scratch(a, "d_next", 4, &d_next)).ok()) return s;
  unsigned long long* d_ops;
  if (!(s = scratch(a, "ops", 4, &d_ops)).ok()) return s;
  CK(cudaMemsetAsync(d_ops, 0, 4 * sizeof(unsigned long long), st));
  b.ops = d_ops;
  // the global bound as the bit pattern of a non-negative double: the probe
  // pass folds every task's first simulated seed into it with atomicMin, the
  // main pass reads it on the device (no host round trip in between)
  unsigned long long* d_gb;
  if (!(s = scratch(a, "d_gb", 1, &d_gb)).ok()) return s;
  {
    double g0 = have_bound ? bound : std::numeric_limits<double>::infinity();
    CK(cudaMemcpyAsync(d_gb, &g0, sizeof g0, cudaMemcpyHostToDevice, st));
  }

  const char* dbg_tasks = std::getenv("HP_DEBUG_TASKS");  // per-task cycle records (diagnostics)
  if (dbg_tasks) {
    if (!(s = scratch(a, "dbg_tasks", 16 * (size_t)nT, &b.trace)).ok()) return s;
    CK(cudaMemsetAsync(b.trace, 0, sizeof(unsigned long long) * 16 * nT, st));
  }
  if (!have_bound) {
    CK(cudaMemsetAsync(d_next, 0, sizeof(int), st));
    hpk::k_default<<<blocks, threads, dsm, st>>>(b, d_tasks, d_order, nT, d_next, d_res, d_tbest, sc, sd, 0, d_gb,
                                                 1, p.uniform_only ? 1 : 0, tt);
    out.launches++;
    out.eval_launches++;
    if (probe_only) {
      double gb = 0.0;
      CK(cudaMemcpyAsync(&gb, d_gb, sizeof gb, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      a.d2h_bytes += sizeof gb;
      out.global_bound = gb;
      return hph::Status{};
    }
  }
  CK(cudaMemsetAsync(d_next, 0, sizeof(int), st));
  if (a.log.on) {
    a.log.reset();
    a.log.key_of = task_ids;
    if (!(s = log_open(a, b.log)).ok()) return s;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (a.time_evals) {
    a.event_pair(&e0, &e1);
    cudaEventRecord(e0, st);
  }
  // the probe pass computed every leaf's seeds (and simulated some)
  hpk::k_default<<<blocks, threads, dsm, st>>>(b, d_tasks, d_order, nT, d_next, d_res, d_tbest, sc, sd,
                                               have_bound ? 0 : 1, d_gb, 0, p.uniform_only ? 1 : 0, tt);
  if (a.time_evals) cudaEventRecord(e1, st);
  out.launches++;
  out.eval_launches++;
  int* d_bt;
  long long* d_counts;
  if (!(s = scratch(a, "d_bt", 1, &d_bt)).ok()) return s;
  if (!(s = scratch(a, "d_counts3", 3, &d_counts)).ok()) return s;
  hpk::k_final_tasks<<<1, 1024, 0, st>>>(b, d_res, d_tasks, d_tbest, nT, d_bt, d_counts);
  out.launches++;
  CK(cudaGetLastError());
  int bt = -1;
  long long counts[3];
  unsigned long long ops[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(&bt, d_bt, sizeof bt, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(counts, d_counts, sizeof counts, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ops, d_ops, sizeof ops, cudaMemcpyDeviceToHost, st));
  if (!have_bound) CK(cudaMemcpyAsync(&out.global_bound, d_gb, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (a.time_evals) out.eval_ms = a.drain_events();
  if (a.log.on && !(s = log_collect(a, b.log, tasks.size())).ok()) return s;
  if (dbg_tasks) {
    std::vector<unsigned long long> rec(16 * (size_t)nT);
    CK(cudaMemcpy(rec.data(), b.trace, sizeof(unsigned long long) * rec.size(), cudaMemcpyDeviceToHost));
    if (FILE* fp = std::fopen(dbg_tasks, "wb")) {
      for (int k = 0; k < nT; ++k) {
        std::fprintf(fp, "%d %d", task_ids[k], tasks[k].pp);
        for (int q = 0; q < 8; ++q) std::fprintf(fp, " %llu", rec[8 * (size_t)k + q]);
        for (int q = 0; q < 8; ++q) std::fprintf(fp, " %llu", rec[8 * ((size_t)nT + k) + q]);
        std::fprintf(fp, "\n");
      }
      std::fclose(fp);
    }
  }
  out.eval_fp64_ops = static_cast<double>(ops[0]);
  out.dev_simulated = static_cast<long long>(ops[1]);
  out.dev_aborted = static_cast<long long>(ops[2]);
  out.dev_screened = static_cast<long long>(ops[3]);
  out.simulated = counts[0];
  out.pruned = counts[1] + counts[2];
  out.pruned_mem = counts[1];
  out.pruned_bound = counts[2];
  out.has_best = bt >= 0;
  if (out.has_best) {
    hpk::TaskRes r;
    CK(cudaMemcpy(&r, d_res + bt, sizeof r, cudaMemcpyDeviceToHost));
    out.best_time = r.best_time;
    out.best_leaf = my_leaves[r.best_leaf];
    out.best_split.resize(tasks[bt].pp);
    CK(cudaMemcpy(out.best_split.data(), d_tbest + tasks[bt].best_off, sizeof(int) * tasks[bt].pp,
                  cudaMemcpyDeviceToHost));
    a.d2h_bytes += sizeof r + sizeof(int) * tasks[bt].pp;
  }
  a.d2h_bytes += sizeof bt + sizeof counts + sizeof ops;
  out.h2d_bytes = a.h2d_bytes;
  out.d2h_bytes = a.d2h_bytes;
  return hph::Status{};
}

}  // namespace hpd
