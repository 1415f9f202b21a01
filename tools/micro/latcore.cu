// Latency of one 1F1B core level for a lone warp (the critical climb's
// evaluator, K stages per lane, hp_kernels.cu eval_item_fast MODE 2):
// cycles per level for the product's level structure, and for variants
// that isolate the cross-lane exchange.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o latcore latcore.cu
#include <cstdio>
#include <type_traits>
#include <cuda_runtime.h>

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }

// EX: 0 = shuffle at odd levels (product), 1 = no exchange (lanes independent),
//     2 = exchange through shared memory
template <int K, int EX>
__device__ void core(double* out, long long* cyc, int levels, double fd, double bd, double sd) {
  __shared__ double sl[32], sr[32];
  const int lane = threadIdx.x & 31;
  double f[K], bw[K], sf[K], fr[K], chf[K], chb[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    f[r] = fd * (1 + r); bw[r] = bd * (2 + r); sf[r] = sd; fr[r] = 0; chf[r] = 0; chb[r] = 0;
  }
  const int src_l = (lane + 31) & 31, src_r = (lane + 1) & 31;
  const double sb0 = sd;
  double xl = 0, xr = 0;
  auto op = [&](auto par_tag, int r) {
    constexpr int PAR = decltype(par_tag)::value;
    if (((PAR - r) & 1) == 0) {
      const double recv = r == 0 ? xl : chf[r > 0 ? r - 1 : 0];
      const double nfr = dmax(fr[r], recv) + f[r];
      fr[r] = nfr;
      chf[r] = nfr + sf[r];
    } else {
      const double recv = r == K - 1 ? xr : chb[r < K - 1 ? r + 1 : 0];
      const double nfr = dmax(fr[r], recv) + bw[r];
      fr[r] = nfr;
      chb[r] = nfr + (r == 0 ? sb0 : sf[r > 0 ? r - 1 : 0]);
    }
  };
  auto level = [&](auto par_tag) {
    constexpr int PAR = decltype(par_tag)::value;
    if (PAR == 1) {
      op(par_tag, 0);
      op(par_tag, K - 1);
      if (EX == 0) {
        xl = __shfl_sync(0xffffffffu, chf[K - 1], src_l);
        xr = __shfl_sync(0xffffffffu, chb[0], src_r);
      } else if (EX == 1) {
        xl = chf[K - 1];
        xr = chb[0];
      } else {
        sl[lane] = chf[K - 1];
        sr[lane] = chb[0];
        __syncwarp();
        xl = sl[src_l];
        xr = sr[src_r];
      }
#pragma unroll
      for (int r = 1; r < K - 1; ++r) op(par_tag, r);
    } else {
#pragma unroll
      for (int r = 0; r < K; ++r) op(par_tag, r);
      if (EX == 2) __syncwarp();
    }
  };
  const long long c0 = clock64();
#pragma unroll 4
  for (int t = 0; t < levels; t += 2) {
    level(std::integral_constant<int, 0>{});
    level(std::integral_constant<int, 1>{});
  }
  const long long c1 = clock64();
  double v = 0;
#pragma unroll
  for (int r = 0; r < K; ++r) v = dmax(v, fr[r] + chf[r] + chb[r]);
  if (v == -1.0) out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

template <int K, int EX>
__global__ void core_k(double* out, long long* cyc, int levels, double fd, double bd, double sd) {
  core<K, EX>(out, cyc, levels, fd, bd, sd);
}

// convergence variants of the same loop: V 1: an early exit on threadIdx
// (as the climb kernel's reserved-SM warps 4-7); 2: the same condition
// broadcast from lane 0 first; 3: a lane-0-only block before the loop
template <int K, int V>
__global__ void core_v(double* out, long long* cyc, int levels, double fd, double bd, double sd, int* flag) {
  if (V == 1 && threadIdx.x >= 32 && *flag) return;
  if (V == 2 && __shfl_sync(0xffffffffu, (int)(threadIdx.x >= 32 && *flag), 0)) return;
  if (V == 3 && (threadIdx.x & 31) == 0) atomicAdd(flag, 0);
  core<K, 0>(out, cyc, levels, fd, bd, sd);
}

template <int K, int V>
void run_v(const char* name) {
  double* o; cudaMalloc(&o, 8192);
  long long* c; cudaMalloc(&c, 8);
  int* fl; cudaMalloc(&fl, 4); cudaMemset(fl, 0, 4);
  const int levels = 1 << 16;
  long long best = 1LL << 62;
  for (int rep = 0; rep < 3; ++rep) {
    core_v<K, V><<<1, 32>>>(o, c, levels, 1e-3, 2e-3, 3e-4, fl);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (h < best) best = h;
  }
  printf("K=%d %-34s %6.1f cycles/level\n", K, name, (double)best / levels);
}

// warps 1.. of the block: the climb kernel's idle warps polling the rings
// (volatile global loads + __nanosleep), next to the timed warp 0
__global__ void pollers(volatile unsigned long long* ctr, int* stop) {
  unsigned ns = 32;
  while (!*(volatile int*)stop) {
    unsigned long long a = ctr[0], b = ctr[1];
    if (a == 12345 && b == 678) ctr[2] = a;
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

// mode 0: loads + sleep up to cap ns; 1: sleep only; 2: loads only
template <int K>
__global__ void core_with_pollers(double* out, long long* cyc, int levels, volatile unsigned long long* ctr, int* stop,
                                  int mode, unsigned cap) {
  if (threadIdx.x >= 32) {
    unsigned ns = 32;
    while (!*(volatile int*)stop) {
      if (mode != 1) {
        unsigned long long a = ctr[0], b = ctr[1];
        if (a == 12345 && b == 678) ctr[2] = a;
      }
      if (mode != 2) __nanosleep(ns);
      if (ns < cap) ns <<= 1;
    }
    return;
  }
  core<K, 0>(out, cyc, levels, 1e-3, 2e-3, 3e-4);
  if (threadIdx.x == 0) atomicExch(stop, 1);
}

template <int K, int EX>
void run(const char* name) {
  double* o; cudaMalloc(&o, 8192);
  long long* c; cudaMalloc(&c, 8);
  const int levels = 1 << 16;
  long long best = 1LL << 62;
  for (int rep = 0; rep < 3; ++rep) {
    core_k<K, EX><<<1, 32>>>(o, c, levels, 1e-3, 2e-3, 3e-4);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (h < best) best = h;
  }
  printf("K=%d %-22s %6.1f cycles/level\n", K, name, (double)best / levels);
}

template <int K>
void run_polled(int threads, int mode = 0, unsigned cap = 256) {
  double* o; cudaMalloc(&o, 8192);
  long long* c; cudaMalloc(&c, 8);
  unsigned long long* ctr; cudaMalloc(&ctr, 64); cudaMemset(ctr, 0, 64);
  int* stop; cudaMalloc(&stop, 4);
  const int levels = 1 << 16;
  long long best = 1LL << 62;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(stop, 0, 4);
    core_with_pollers<K><<<1, threads>>>(o, c, levels, ctr, stop, mode, cap);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (h < best) best = h;
  }
  printf("K=%d shuffle + %d polling warps (mode %d, cap %u ns)  %6.1f cycles/level\n", K, threads / 32 - 1, mode, cap,
         (double)best / levels);
}

int main() {
  run_v<4, 1>("early exit on threadIdx"); run_v<4, 2>("early exit, broadcast condition");
  run_v<4, 3>("lane-0 block before the loop");
  run<4, 0>("shuffle (product)"); run<4, 1>("no exchange"); run<4, 2>("shared memory");
  run<6, 0>("shuffle (product)"); run<6, 1>("no exchange");
  run<8, 0>("shuffle (product)"); run<8, 1>("no exchange");
  run<2, 0>("shuffle (product)"); run<2, 1>("no exchange");
  return 0;
}
