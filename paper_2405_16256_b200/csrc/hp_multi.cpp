// hp_multi.cpp — multi-GPU search inside the C ABI (hp_multi_*): the
// reference parallelises search() over `jobs` threads (planner.cpp:612-664);
// here one host thread drives each GPU of the box, every GPU searches one
// shard of the candidate space (hp_search with shard_index = rank), and the
// two cross-shard exchanges of the search run as NCCL collectives over
// NVLink / NVSwitch:
//   * default mode: ncclAllReduce(MIN) of the shards' probe minima — the
//     global bound of planner.cpp:640-651 (a plain min of doubles, exact);
//   * the result: ncclAllGather of the fixed-size hp_result records, then the
//     exact better_than reduction (planner.cpp:178-200, 656-664) on the host.
// NCCL is loaded at run time (dlopen of libnccl.so.2: the one torch bundles
// when torch is in the process, else the system one), so the library stays
// loadable without it; only hp_multi_create needs it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hetplan_b200.h"
#include "hp_host.hpp"

namespace {

struct Nccl {
  void* so = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;

  bool load(std::string& err) {
    if (so) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (so) break;
    }
    if (!so) {
      err = std::string("NCCL not found (dlopen libnccl.so.2): ") + dlerror();
      return false;
    }
    init_all = reinterpret_cast<decltype(init_all)>(dlsym(so, "ncclCommInitAll"));
    destroy = reinterpret_cast<decltype(destroy)>(dlsym(so, "ncclCommDestroy"));
    all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(so, "ncclAllReduce"));
    all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(so, "ncclAllGather"));
    error_string = reinterpret_cast<decltype(error_string)>(dlsym(so, "ncclGetErrorString"));
    if (!init_all || !destroy || !all_reduce || !all_gather || !error_string) {
      err = "NCCL library lacks a required symbol";
      return false;
    }
    return true;
  }
};

Nccl g_nccl;

}  // namespace

struct hp_multi {
  std::vector<int> devices;
  std::vector<hp_ctx*> ctx;
  std::vector<ncclComm_t> comm;
  std::vector<cudaStream_t> stream;
  std::vector<void*> dbuf;  // per device: [n * sizeof(hp_result)] gather target + 1 double
  std::vector<hp_result> per;
  std::string err;
};

namespace {

constexpr size_t kRec = sizeof(hp_result);

hp_status set_err(hp_multi* m, hp_status st, const std::string& msg) {
  m->err = msg;
  return st;
}

}  // namespace

extern "C" {

int hp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

hp_status hp_multi_create(hp_multi** out, const int32_t* devices, int32_t n) {
  if (!out || n < 1 || !devices) return HP_INTERNAL;
  *out = nullptr;
  hp_multi* m = new hp_multi();
  m->devices.assign(devices, devices + n);
  std::string err;
  if (!g_nccl.load(err)) {
    *out = m;
    return set_err(m, HP_NCCL, err);
  }
  m->ctx.assign(n, nullptr);
  m->stream.assign(n, nullptr);
  m->dbuf.assign(n, nullptr);
  for (int r = 0; r < n; ++r) {
    if (hp_create(&m->ctx[r], devices[r]) != HP_OK) {
      *out = m;
      return set_err(m, HP_CUDA, "hp_create failed on device " + std::to_string(devices[r]));
    }
    cudaSetDevice(devices[r]);
    if (cudaStreamCreateWithFlags(&m->stream[r], cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&m->dbuf[r], kRec * (n + 1) + 2 * sizeof(double)) != cudaSuccess) {
      *out = m;
      return set_err(m, HP_CUDA, "stream / buffer allocation failed on device " + std::to_string(devices[r]));
    }
  }
  m->comm.assign(n, nullptr);
  // NCCL prints its version banner on stdout at initialisation when
  // NCCL_DEBUG is set; a library must not write on the host program's stdout
  // (the CLI's report goes there), so fd 1 points at stderr for the call
  std::fflush(stdout);
  const int saved = dup(1);
  if (saved >= 0) dup2(2, 1);
  ncclResult_t nr = g_nccl.init_all(m->comm.data(), n, m->devices.data());
  std::fflush(stdout);
  if (saved >= 0) {
    dup2(saved, 1);
    close(saved);
  }
  *out = m;
  if (nr != ncclSuccess) return set_err(m, HP_NCCL, std::string("ncclCommInitAll: ") + g_nccl.error_string(nr));
  return HP_OK;
}

void hp_multi_destroy(hp_multi* m) {
  if (!m) return;
  for (size_t r = 0; r < m->ctx.size(); ++r) {
    cudaSetDevice(m->devices[r]);
    if (r < m->comm.size() && m->comm[r]) g_nccl.destroy(m->comm[r]);
    if (m->dbuf[r]) cudaFree(m->dbuf[r]);
    if (m->stream[r]) cudaStreamDestroy(m->stream[r]);
    if (m->ctx[r]) hp_destroy(m->ctx[r]);
  }
  delete m;
}

const char* hp_multi_last_error(const hp_multi* m) { return m ? m->err.c_str() : ""; }

hp_status hp_search_multi(hp_multi* m, const hp_problem* problem, int32_t flags, hp_result* result,
                          hp_result* per_device) {
  if (!m || !result) return HP_INTERNAL;
  const int n = static_cast<int>(m->devices.size());
  if (m->comm.size() != static_cast<size_t>(n) || !m->comm[0]) return set_err(m, HP_NCCL, "no NCCL communicators");
  hph::Problem p;
  hph::Status vs = hph::load_problem(problem, p);
  if (!vs.ok()) return set_err(m, vs.code, vs.msg);
  const bool pruning = p.pruning;
  std::vector<hp_status> st(n, HP_OK);
  std::vector<std::string> why(n);
  std::vector<std::vector<unsigned char>> gathered(n, std::vector<unsigned char>(kRec * n));
  m->per.assign(n, hp_result{});
  auto worker = [&](int r) {
    cudaSetDevice(m->devices[r]);
    hp_ctx* ctx = m->ctx[r];
    cudaStream_t s = m->stream[r];
    unsigned char* dbase = static_cast<unsigned char*>(m->dbuf[r]);
    double* dbound = reinterpret_cast<double*>(dbase + kRec * (n + 1));
    hp_search_opts opts{r, n, 0, flags, 0.0};
    if (pruning) {
      // probe pass per shard, then the global bound (planner.cpp:640-651);
      // every rank reaches the collective even after a local failure
      double b = std::numeric_limits<double>::infinity();
      st[r] = hp_probe(ctx, problem, &opts, &b);
      if (st[r] != HP_OK) why[r] = hp_last_error(ctx);
      cudaMemcpyAsync(dbound, &b, sizeof b, cudaMemcpyHostToDevice, s);
      ncclResult_t nr = g_nccl.all_reduce(dbound, dbound + 1, 1, ncclFloat64, ncclMin, m->comm[r], s);
      cudaMemcpyAsync(&b, dbound + 1, sizeof b, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (nr != ncclSuccess && st[r] == HP_OK) {
        st[r] = HP_NCCL;
        why[r] = std::string("ncclAllReduce: ") + g_nccl.error_string(nr);
      }
      opts.have_global_bound = 1;
      opts.global_bound = b;
    }
    hp_result& mine = m->per[r];
    std::memset(&mine, 0, sizeof mine);
    if (st[r] == HP_OK) {
      st[r] = hp_search(ctx, problem, &opts, &mine);
      if (st[r] != HP_OK) why[r] = hp_last_error(ctx);
    }
    // one all-gather of the fixed-size records (planner.cpp:656-664)
    cudaMemcpyAsync(dbase + kRec * n, &mine, kRec, cudaMemcpyHostToDevice, s);
    ncclResult_t nr = g_nccl.all_gather(dbase + kRec * n, dbase, kRec, ncclUint8, m->comm[r], s);
    cudaMemcpyAsync(gathered[r].data(), dbase, kRec * n, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (nr != ncclSuccess && st[r] == HP_OK) {
      st[r] = HP_NCCL;
      why[r] = std::string("ncclAllGather: ") + g_nccl.error_string(nr);
    }
  };
  std::vector<std::thread> th;
  for (int r = 0; r < n; ++r) th.emplace_back(worker, r);
  for (auto& t : th) t.join();
  for (int r = 0; r < n; ++r)
    if (st[r] != HP_OK) return set_err(m, st[r], why[r]);
  // exact reduction of the gathered records (rank 0's copy; every rank holds
  // the same bytes): counts add up, the best is better_than's minimum
  std::vector<hp_result> recs(n);
  for (int r = 0; r < n; ++r) std::memcpy(&recs[r], gathered[0].data() + kRec * r, kRec);
  hp_result red;
  std::memset(&red, 0, sizeof red);
  for (int r = 0; r < n; ++r) {
    const hp_result& x = recs[r];
    red.candidates_simulated += x.candidates_simulated;
    red.candidates_pruned += x.candidates_pruned;
    for (int k = 0; k < HP_REASON_COUNT; ++k) red.reason_counts[k] += x.reason_counts[k];
    red.leaves += x.leaves;
    red.tasks = x.tasks;
    red.gpu_launches += x.gpu_launches;
    red.eval_launches += x.eval_launches;
    red.eval_ms += x.eval_ms;
    red.eval_fp64_ops += x.eval_fp64_ops;
    red.h2d_bytes += x.h2d_bytes;
    red.d2h_bytes += x.d2h_bytes;
    red.device_ms = std::max(red.device_ms, x.device_ms);
    red.host_ms = std::max(red.host_ms, x.host_ms);
    red.global_bound = x.global_bound;
    red.device_simulated += x.device_simulated;
    red.device_aborted += x.device_aborted;
    red.device_screened += x.device_screened;
    if (x.has_best &&
        (!red.has_best || hph::compare_plans(p, x.best_time_s, x.best_plan, red.best_time_s, red.best_plan) < 0)) {
      red.has_best = 1;
      red.best_time_s = x.best_time_s;
      red.best_pp = x.best_pp;
      red.best_plan = x.best_plan;
    }
  }
  *result = red;
  if (per_device) std::memcpy(per_device, recs.data(), kRec * n);
  return HP_OK;
}

hp_status hp_multi_search_log(hp_multi* m, hp_log_entry* entries, uint64_t entry_cap, char* text, uint64_t text_cap,
                              uint64_t* n_entries, uint64_t* text_bytes) {
  if (!m) return HP_INTERNAL;
  // shards own whole tasks (default mode) or whole leaves (full mode): the
  // global log is the stable merge of the shards' logs by (task, leaf)
  struct Part {
    std::vector<hp_log_entry> e;
    std::vector<char> t;
  };
  std::vector<Part> parts(m->ctx.size());
  uint64_t total = 0, tbytes = 0;
  for (size_t r = 0; r < m->ctx.size(); ++r) {
    uint64_t ne = 0, nb = 0;
    hp_status s = hp_search_log(m->ctx[r], nullptr, 0, nullptr, 0, &ne, &nb);
    if (s != HP_OK) return set_err(m, s, hp_last_error(m->ctx[r]));
    parts[r].e.resize(ne);
    parts[r].t.resize(nb);
    s = hp_search_log(m->ctx[r], parts[r].e.data(), ne, parts[r].t.data(), nb, &ne, &nb);
    if (s != HP_OK) return set_err(m, s, hp_last_error(m->ctx[r]));
    total += ne;
    tbytes += nb;
  }
  if (n_entries) *n_entries = total;
  if (text_bytes) *text_bytes = tbytes;
  if (!entries && !text) return HP_OK;
  if ((entries && entry_cap < total) || (text && text_cap < tbytes))
    return set_err(m, HP_BAD_CONFIG, "search log: buffer too small");
  std::vector<std::pair<size_t, size_t>> order;  // (part, index)
  order.reserve(total);
  for (size_t r = 0; r < parts.size(); ++r)
    for (size_t k = 0; k < parts[r].e.size(); ++k) order.push_back({r, k});
  std::stable_sort(order.begin(), order.end(), [&](const auto& x, const auto& y) {
    const hp_log_entry& a = parts[x.first].e[x.second];
    const hp_log_entry& b = parts[y.first].e[y.second];
    return a.task != b.task ? a.task < b.task : a.leaf < b.leaf;
  });
  std::vector<uint64_t> base(parts.size(), 0);
  for (size_t r = 1; r < parts.size(); ++r) base[r] = base[r - 1] + parts[r - 1].t.size();
  if (text)
    for (size_t r = 0; r < parts.size(); ++r)
      if (!parts[r].t.empty()) std::memcpy(text + base[r], parts[r].t.data(), parts[r].t.size());
  if (entries)
    for (size_t k = 0; k < order.size(); ++k) {
      hp_log_entry e = parts[order[k].first].e[order[k].second];
      e.candidate += base[order[k].first];
      e.reason += base[order[k].first];
      entries[k] = e;
    }
  return HP_OK;
}

}  // extern "C"
