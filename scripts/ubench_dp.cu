// Microbenchmark (experiment support, not product code): DFMA throughput with 2 vs 3 register
// operands (register-file bank pressure) and DFMA dependent-chain latency on the B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubd scripts/ubench_dp.cu && /tmp/ubd
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 2048;

// MODE 0: 8 independent chains d_k = fma(d_k, a_k, b_k) with a_k, b_k distinct REGISTERS
// MODE 1: same with a, b kernel constants (constant-bank operands)
// MODE 2: one dependent chain (latency)
// MODE 3: 4 independent chains, all-register operands
template <int MODE>
__global__ void __launch_bounds__(256) kern(double* out, const double* in) {
  const int t = threadIdx.x;
  double a[8], b[8], d[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = in[k] + t * 1e-9;
    b[k] = in[8 + k] - t * 1e-9;
    d[k] = t + k;
  }
  for (int it = 0; it < IT; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k] = fma(d[k], a[k], b[k]);
    } else if (MODE == 1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k] = fma(d[k], 1.0000001, 1e-9 * (k + 1));
    } else if (MODE == 2) {
#pragma unroll
      for (int k = 0; k < 8; ++k) d[0] = fma(d[0], a[k], b[k]);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k & 3] = fma(d[k & 3], a[k], b[k]);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += d[k];
  out[blockIdx.x * blockDim.x + t] = s;
}

template <int MODE>
void run(const char* name, int threads, int ctas_per_sm) {
  int nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int grid = nsm * ctas_per_sm;
  double *o, *in;
  cudaMalloc(&o, (size_t)grid * threads * 8);
  cudaMalloc(&in, 16 * 8);
  double h[16];
  for (int k = 0; k < 16; ++k) h[k] = 1.0 + 1e-7 * k;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) kern<MODE><<<grid, threads>>>(o, in);
  cudaEventRecord(e0);
  kern<MODE><<<grid, threads>>>(o, in);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * clk * 1e3;
  const double warps_per_smsp = (double)ctas_per_sm * threads / 32 / 4;
  printf("%-40s warps/SMSP %5.2f: %7.3f SMSP-cycles per warp-DFMA (per SMSP, all warps)   %s\n", name,
         warps_per_smsp, cyc / (warps_per_smsp * IT * 8), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("8 chains, 3 register operands", 256, 4);
  run<1>("8 chains, constant operands", 256, 4);
  run<3>("4 chains, 3 register operands", 256, 4);
  run<2>("1 chain (latency), 1 warp/SMSP", 128, 1);
  run<2>("1 chain (latency), 2 warps/SMSP", 256, 1);
  run<0>("8 chains, 3 reg ops, 1 warp/SMSP", 128, 1);
  run<0>("8 chains, 3 reg ops, 2 warps/SMSP", 256, 1);
  return 0;
}
