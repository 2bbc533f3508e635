// Microbenchmark (experiment support, not product code): per-SM throughput of LDS.64, SHFL.32,
// DFMA and their mixes on the B200, to decide how k_wave exchanges x-neighbours and history.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub scripts/ubench_smem.cu && /tmp/ub
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 4096;

template <int MODE>
__global__ void __launch_bounds__(256) kern(unsigned long long* out, double* dout, int salt) {
  __shared__ double sm[2048];
  const int t = threadIdx.x;
  for (int i = t; i < 2048; i += blockDim.x) sm[i] = i * 0.5 + salt;
  __syncthreads();
  unsigned a0 = t, a1 = t * 3;
  double d0 = t, d1 = t + 1, d2 = t + 2, d3 = t + 3, d4 = t + 4, d5 = t + 5, d6 = t + 6, d7 = t + 7;
  const double c = 1.0000001, e = 1e-9;
  int off = (t & 255);
  for (int it = 0; it < IT; ++it) {
    if (MODE == 0 || MODE == 2 || MODE == 4 || MODE == 5) {        // LDS.64 x2
      const double v = sm[(off + it * 7) & 2047];
      const double w = sm[(off + it * 13 + 512) & 2047];
      unsigned long long u = __double_as_longlong(v) ^ __double_as_longlong(w);
      a0 ^= (unsigned)u;
      a1 += (unsigned)(u >> 32);
    }
    if (MODE == 1 || MODE == 2) {                                  // SHFL.32 x4
      a0 ^= __shfl_down_sync(0xffffffffu, a1, 1);
      a1 += __shfl_up_sync(0xffffffffu, a0, 1);
      a0 ^= __shfl_down_sync(0xffffffffu, a1 + it, 1);
      a1 += __shfl_up_sync(0xffffffffu, a0 + it, 1);
    }
    if (MODE == 3 || MODE == 4 || MODE == 5) {                     // DFMA x8 (x16 in mode 5)
      d0 = fma(d0, c, e); d1 = fma(d1, c, e); d2 = fma(d2, c, e); d3 = fma(d3, c, e);
      d4 = fma(d4, c, e); d5 = fma(d5, c, e); d6 = fma(d6, c, e); d7 = fma(d7, c, e);
      if (MODE == 5) {
        d0 = fma(d0, c, e); d1 = fma(d1, c, e); d2 = fma(d2, c, e); d3 = fma(d3, c, e);
        d4 = fma(d4, c, e); d5 = fma(d5, c, e); d6 = fma(d6, c, e); d7 = fma(d7, c, e);
      }
    }
    if (MODE == 6) {                                              // STS.64 x1 + LDS.64 x2 (exchange)
      sm[(off + it) & 2047] = d0 + it;
      const double v = sm[(off + 1 + it) & 2047], w = sm[(off + 2047 + it) & 2047];
      d0 = v - w;
    }
  }
  out[blockIdx.x * blockDim.x + t] = a0 ^ a1;
  dout[blockIdx.x * blockDim.x + t] = d0 + d1 + d2 + d3 + d4 + d5 + d6 + d7;
}

template <int MODE>
void run(const char* name, int per_iter_ops, int nthreads, int ctas_per_sm) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * ctas_per_sm;
  unsigned long long* o;
  double* d;
  cudaMalloc(&o, (size_t)grid * nthreads * 8);
  cudaMalloc(&d, (size_t)grid * nthreads * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) kern<MODE><<<grid, nthreads>>>(o, d, w);
  cudaEventRecord(a);
  kern<MODE><<<grid, nthreads>>>(o, d, 7);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warps_per_sm = (double)ctas_per_sm * nthreads / 32;
  const double cycles = ms * 1e-3 * clk * 1e3;   // at the nominal max clock
  const double winstr = warps_per_sm * IT;       // iterations per SM (warp-level)
  printf("%-28s %8.3f ms  %6.3f SM-cycles per warp-iteration (%d ops)  err=%s\n", name, ms,
         cycles / winstr, per_iter_ops, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("LDS.64 x2", 2, 256, 4);
  run<1>("SHFL.32 x4", 4, 256, 4);
  run<2>("LDS.64 x2 + SHFL.32 x4", 6, 256, 4);
  run<3>("DFMA x8", 8, 256, 4);
  run<4>("DFMA x8 + LDS.64 x2", 10, 256, 4);
  run<5>("DFMA x16 + LDS.64 x2", 18, 256, 4);
  run<6>("STS.64 + LDS.64 x2", 3, 256, 4);
  return 0;
}
