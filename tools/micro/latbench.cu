// Dependent-latency microbenchmark (one warp): DADD chain, DSETP+FSEL max
// chain, max+add node update, SHFL of a double, to size the evaluator's
// per-level critical path on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }

__global__ void lat(double* out, long long* cyc, double a, double d, int n) {
  const int lane = threadIdx.x;
  double x = a + lane, y = a * 0.5 + lane, z = a;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + d;
  t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  // max chain: x = max(x, y) ; y alternates
  t0 = clock64();
  for (int i = 0; i < n; ++i) { z = dmax(z, y); y = y + 0.0; z = z * 1.0; }
  t1 = clock64();
  if (lane == 0) cyc[1] = t1 - t0;
  // node update: z = max(z, y) + d
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = dmax(z, y) + d;
  t1 = clock64();
  if (lane == 0) cyc[2] = t1 - t0;
  // shfl chain of a double
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = __shfl_sync(0xffffffffu, y, (lane + 1) & 31);
  t1 = clock64();
  if (lane == 0) cyc[3] = t1 - t0;
  // shfl + node update + add (one level of the boundary stage)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double r = __shfl_sync(0xffffffffu, x, (lane + 31) & 31);
    x = (dmax(z, r) + d) + d;
    z = x;
  }
  t1 = clock64();
  if (lane == 0) cyc[4] = t1 - t0;
  out[lane] = x + y + z;
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 8 * 8);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(o, c, 1.0, 1e-3, n);
  long long h[8];
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  printf("cycles per iteration: dadd %.1f | max (DSETP+FSEL, + DMUL filler) %.1f | max+add %.1f | shfl.f64 %.1f | shfl+max+add+add %.1f\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n);
  return 0;
}
