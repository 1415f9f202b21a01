// Microbenchmark: node update fr = max(fr, r) + d; c = max(fr, c) + s with
// different formulations of the double max on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double max_sel(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double max_pmov(double a, double b) {
  double r = a;
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, %2;\n\t@p mov.b64 %0, %2;\n\t}" : "+d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ double max_i64(double a, double b) {
  long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return __longlong_as_double(x < y ? y : x);
}
__device__ __forceinline__ double max_fmax(double a, double b) { return fmax(a, b); }

template <int V>
__device__ __forceinline__ double mx(double a, double b) {
  if (V == 0) return max_sel(a, b);
  if (V == 1) return max_pmov(a, b);
  if (V == 2) return max_i64(a, b);
  return max_fmax(a, b);
}

template <int V, int CH>
__global__ void k(double* out, int iters, double d, double s) {
  double fr[CH], c[CH], r[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) { fr[k] = threadIdx.x * 1e-9 + k; c[k] = k * 0.5; r[k] = k * 0.25; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      fr[k] = mx<V>(fr[k], r[k]) + d;
      c[k] = mx<V>(fr[k], c[k]) + s;
    }
#pragma unroll
    for (int k = 0; k < CH; ++k) r[k] = c[(k + 1) % CH];
  }
  double t = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) t += fr[k] + c[k];
  if (t == -1.0) out[threadIdx.x] = t;
}

template <int V, int CH>
void run(const char* name, int blocks_per_sm, int threads) {
  double* o; cudaMalloc(&o, 8192);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<V, CH><<<sms * blocks_per_sm, threads>>>(o, iters, 1e-12, 2e-12);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = ms < best ? ms : best;
  }
  double ops = (double)sms * blocks_per_sm * threads * iters * CH * 4;
  printf("%-8s CH=%d warps/SM=%2d : %6.2f T alg-ops/s  (%.1f upd/clk/SM @1.965GHz)\n", name, CH,
         blocks_per_sm * threads / 32, ops / best / 1e9, ops / 4 / best * 1e3 / sms / 1.965e9);
  cudaFree(o);
}

int main() {
  for (int occ : {4, 8}) {
    run<0, 6>("sel", occ, 128); run<1, 6>("pmov", occ, 128); run<2, 6>("i64", occ, 128); run<3, 6>("fmax", occ, 128);
  }
  run<0, 6>("sel", 16, 128); run<1, 6>("pmov", 16, 128);
  run<0, 12>("sel", 4, 128); run<1, 12>("pmov", 4, 128);
  return 0;
}
