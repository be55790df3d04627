// Microbenchmark: FP64 FFMA pipe and DMMA (mma.sync f64) throughput on sm_100a,
// plus a float64 streaming copy. Used to set the FP64 roofline denominator.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-3, b0 = 0.5;
  double c[4][4];
  for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) c[j][k] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b0));
    }
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) s += c[j][k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main(int argc, char** argv) {
  const double sustain_s = argc > 1 ? atof(argv[1]) : 0.0;  // > 0: also a sustained DMMA run of this length
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu,\"regs_per_sm\":%d}\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double* out; CK(cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int blocksPerSm : {2, 4, 8}) {
    int threads = 256, iters = 4096, grid = sms * blocksPerSm;
    dfma_loop<<<grid, threads>>>(out, 16, 0.999, 1e-3);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<<<grid, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64.0 * iters * (double)grid * threads;
    printf("{\"kernel\":\"dfma\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", blocksPerSm, ms, flops / ms / 1e9);
  }
  for (int blocksPerSm : {2, 4, 8}) {
    int threads = 128, iters = 4096, grid = sms * blocksPerSm;
    dmma_loop<<<grid, threads>>>(out, 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_loop<<<grid, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 4 * 4.0 * iters * (double)grid * (threads / 32);
    printf("{\"kernel\":\"dmma_m16n8k4\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", blocksPerSm, ms, flops / ms / 1e9);
  }
  if (sustain_s > 0) {  // back-to-back launches for sustain_s seconds (the figure for a kernel inside a long step)
    int threads = 128, iters = 4096, grid = sms * 4;
    double flops1 = 2.0 * 16 * 8 * 4 * 4.0 * iters * (double)grid * (threads / 32);
    float ms = 0; long launches = 0;
    cudaEventRecord(e0);
    while (ms < sustain_s * 1e3) {
      for (int k = 0; k < 50; ++k) dmma_loop<<<grid, threads>>>(out, iters);
      launches += 50;
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("{\"kernel\":\"dmma_m16n8k4_sustained\",\"seconds\":%.2f,\"launches\":%ld,\"tflops\":%.2f}\n", ms / 1e3, launches, flops1 * launches / ms / 1e9);
  }
  size_t n = (size_t)1 << 28; // 2 GiB per buffer of doubles
  double2 *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
  cudaMemset(a, 0, n * 8);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_k<<<sms * 8, 512>>>(a, b, n / 2);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\":\"copy_f64\",\"ms\":%.3f,\"gbs\":%.1f}\n", ms, 2.0 * n * 8 / ms / 1e6);
  }
  return 0;
}
