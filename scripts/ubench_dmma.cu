// Microbenchmark (experiment support, not product code): fp64 tensor-core (DMMA, mma.sync
// m8n8k4 f64) throughput on the B200, against plain DFMA -- decides how the N3 DST contraction
// is written. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubm scripts/ubench_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 1024;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int NACC>
__global__ void __launch_bounds__(256) k(double* out, const double* in) {
  const int t = threadIdx.x;
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = in[t & 31], b = in[32 + (t & 31)];
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + t] = s;
}

template <int NACC>
void run(int ctas_per_sm) {
  int nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int grid = nsm * ctas_per_sm;
  double *o, *in;
  cudaMalloc(&o, (size_t)grid * 256 * 8);
  cudaMalloc(&in, 64 * 8);
  cudaMemset(in, 0, 64 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<NACC><<<grid, 256>>>(o, in);
  cudaEventRecord(e0);
  k<NACC><<<grid, 256>>>(o, in);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * (double)NACC * IT * (grid * 256 / 32);
  printf("DMMA m8n8k4, %d independent accumulators/warp, %d CTAs/SM: %.1f TFLOP/s  (%s)\n", NACC,
         ctas_per_sm, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4>(2);
  run<8>(2);
  run<8>(4);
  run<16>(2);
  return 0;
}
