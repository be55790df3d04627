// L2 read bandwidth + DMMA m16n8k4 fragment-layout check (dev aid).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void l2read(const double2* __restrict__ a, size_t n, int passes, double* out) {
  double2 acc = make_double2(0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; ++p)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x + (size_t)p * 7919; i < n + (size_t)p * 7919; i += stride) {
      double2 v = a[i % n];
      acc.x += v.x; acc.y += v.y;
    }
  if (acc.x == 12345.0) out[0] = acc.y;
}
__global__ void mma_check(double* out) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  // A[m][k] = m*10 + k ; B[k][n] = (k+1)*100 + n
  double a0 = g * 10 + t, a1 = (g + 8) * 10 + t, b0 = (t + 1) * 100 + g;
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b0));
  // expected C[m][n] = sum_k A[m][k]*B[k][n]
  auto ref = [](int m, int n) { double s = 0; for (int k = 0; k < 4; ++k) s += (m * 10 + k) * ((k + 1) * 100.0 + n); return s; };
  int bad = 0;
  bad += c0 != ref(g, 2 * t);
  bad += c1 != ref(g, 2 * t + 1);
  bad += c2 != ref(g + 8, 2 * t);
  bad += c3 != ref(g + 8, 2 * t + 1);
  out[lane] = bad;
}
int main() {
  double* o; cudaMalloc(&o, 64 * sizeof(double));
  mma_check<<<1, 32>>>(o);
  double h[32]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < 32; ++i) bad += (int)h[i];
  printf("{\"mma_m16n8k4_layout_mismatches\": %d}\n", bad);
  for (size_t mb : {16, 48, 96, 2048}) {
    size_t n = mb * (1 << 20) / 16;
    double2* a; cudaMalloc(&a, n * 16); cudaMemset(a, 0, n * 16);
    int passes = mb >= 1024 ? 3 : 40;
    l2read<<<148 * 8, 512>>>(a, n, 1, o);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    l2read<<<148 * 8, 512>>>(a, n, passes, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"read_buffer_mb\": %zu, \"gbs\": %.1f}\n", mb, (double)n * 16 * passes / ms / 1e6);
    cudaFree(a);
  }
  return 0;
}
