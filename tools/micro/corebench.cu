// Core-loop microbenchmark: the evaluator's steady-state level (K stages per
// lane, F/B by parity, neighbour channel values exchanged by __shfl_sync)
// on synthetic data, to separate the loop's own ceiling from the rest.
#include <cstdio>
#include <type_traits>
#include <cuda_runtime.h>

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }

template <int K>
__global__ void core(double* out, int levels, double fd, double bd, double sd) {
  const int lane = threadIdx.x & 31;
  double f[K], bw[K], sf[K], fr[K], chf[K], chb[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    f[r] = fd * (1 + r); bw[r] = bd * (2 + r); sf[r] = sd; fr[r] = 0; chf[r] = 0; chb[r] = 0;
  }
  const int src_l = (lane + 31) & 31, src_r = (lane + 1) & 31;
  const double sb0 = sd;
  auto level = [&](auto par_tag) {
    constexpr int PAR = decltype(par_tag)::value;
    const double lchf = __shfl_sync(0xffffffffu, chf[K - 1], src_l);
    const double rchb = __shfl_sync(0xffffffffu, chb[0], src_r);
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (((PAR - r) & 1) == 0) {
        const double recv = r == 0 ? lchf : chf[r > 0 ? r - 1 : 0];
        fr[r] = dmax(fr[r], recv) + f[r];
        chf[r] = dmax(fr[r], chf[r]) + sf[r];
      } else {
        const double recv = r == K - 1 ? rchb : chb[r < K - 1 ? r + 1 : 0];
        fr[r] = dmax(fr[r], recv) + bw[r];
        chb[r] = dmax(fr[r], chb[r]) + (r == 0 ? sb0 : sf[r > 0 ? r - 1 : 0]);
      }
    }
  };
  for (int t = 0; t < levels; t += 2) {
    level(std::integral_constant<int, 0>{});
    level(std::integral_constant<int, 1>{});
  }
  double v = 0;
#pragma unroll
  for (int r = 0; r < K; ++r) v = dmax(v, fr[r] + chf[r] + chb[r]);
  if (v == -1.0) out[threadIdx.x] = v;
}

template <int K>
void run(int blocks_per_sm, int threads) {
  double* o; cudaMalloc(&o, 8192);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int levels = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    core<K><<<sms * blocks_per_sm, threads>>>(o, levels, 1e-3, 2e-3, 3e-4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = ms < best ? ms : best;
  }
  double ops = (double)sms * blocks_per_sm * threads * levels * K * 4;
  printf("core K=%d warps/SM=%2d : %6.2f T alg-ops/s (%.1f upd/clk/SM) %.1f cyc/level/warp\n", K,
         blocks_per_sm * threads / 32, ops / best / 1e9, ops / 4 / best * 1e3 / sms / 1.965e9,
         best * 1e-3 * 1.965e9 / levels);
}

int main() {
  // latency: one warp per SM, then one per SM sub-partition
  run<2>(1, 32); run<4>(1, 32); run<6>(1, 32); run<8>(1, 32);
  run<2>(1, 128); run<4>(1, 128); run<6>(1, 128); run<8>(1, 128);
  for (int w : {2, 4, 8}) { run<2>(w, 128); run<4>(w, 128); run<6>(w, 128); run<8>(w, 128); }
  return 0;
}
