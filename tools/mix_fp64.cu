// Do DMMA (FP64 tensor core) and DFMA (FP64 ALU) share throughput on sm_100a?
// Runs DMMA-only, DFMA-only and mixed loops; prints TF/s of each pipe.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mix_fp64 tools/mix_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NMMA, int NFMA>
__global__ void mix(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-3, b0 = 0.5;
  double c[4][4] = {};
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NMMA; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[j & 3][0]), "+d"(c[j & 3][1]), "+d"(c[j & 3][2]), "+d"(c[j & 3][3])
                   : "d"(a0), "d"(a1), "d"(b0));
#pragma unroll
    for (int j = 0; j < NFMA; ++j) x[j & 7] = fma(x[j & 7], 0.999, 1e-3);
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) s += c[j][k];
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NMMA, int NFMA>
void run(const char* name, double* out, int sms) {
  const int grid = sms * 2, threads = 256, iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<NMMA, NFMA><<<grid, threads>>>(out, 8);
  cudaEventRecord(e0);
  mix<NMMA, NFMA><<<grid, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)grid * threads / 32;
  const double mma_f = 2.0 * 16 * 8 * 4 * NMMA * iters * warps;
  const double fma_f = 2.0 * NFMA * iters * warps * 32;
  printf("{\"kernel\":\"%s\",\"ms\":%.3f,\"dmma_tflops\":%.2f,\"dfma_tflops\":%.2f,\"total\":%.2f}\n", name, ms,
         mma_f / ms / 1e9, fma_f / ms / 1e9, (mma_f + fma_f) / ms / 1e9);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, p.multiProcessorCount * 2 * 256 * sizeof(double));
  run<8, 0>("dmma_only", out, p.multiProcessorCount);
  run<0, 64>("dfma_only", out, p.multiProcessorCount);
  run<8, 16>("mix_8_16", out, p.multiProcessorCount);
  run<8, 64>("mix_8_64", out, p.multiProcessorCount);
  run<4, 64>("mix_4_64", out, p.multiProcessorCount);
  return 0;
}
