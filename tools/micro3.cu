// DMMA throughput with operands from shared memory (dev aid): per k-step each
// warp loads a0,a1 (A frag) and NT b0's, then issues NT m16n8k4 (A reused).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b0));
}
template <int NT, int CHAINS>
__global__ void k(double* out, int iters) {
  __shared__ double A[32 * 72];
  __shared__ double B[32 * 72];
  for (int i = threadIdx.x; i < 32 * 72; i += blockDim.x) { A[i] = i * 1e-6; B[i] = i * 2e-6; }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double acc[CHAINS][NT][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      const int kk = (4 * ks + t) & 31;
      const double a0 = A[kk * 72 + g + 16 * (w & 3)], a1 = A[kk * 72 + g + 8 + 16 * (w & 3)];
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[ks % CHAINS][j], a0, a1, B[kk * 72 + 8 * j + g]);
    }
  }
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) for (int j = 0; j < NT; ++j) for (int q = 0; q < 4; ++q) s += acc[c][j][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NT, int CHAINS>
void run(int threads, int blocksPerSm, double* o) {
  int iters = 2000, grid = 148 * blocksPerSm;
  k<NT, CHAINS><<<grid, threads>>>(o, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NT, CHAINS><<<grid, threads>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 16 * 8 * 4 * 16.0 * NT * iters * grid * (threads / 32);
  printf("{\"NT\":%d,\"chains\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f}\n", NT, CHAINS, threads / 32 * blocksPerSm, fl / ms / 1e9);
}
int main() {
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  run<7, 1>(256, 1, o); run<7, 2>(256, 1, o); run<7, 2>(512, 1, o); run<7, 2>(256, 2, o);
  run<4, 2>(256, 1, o); run<2, 2>(256, 1, o); run<1, 4>(256, 1, o); run<7, 4>(256, 1, o);
  return 0;
}
