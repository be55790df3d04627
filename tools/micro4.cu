// DRAM read efficiency vs segment size / stride (dev aid). Each warp reads
// segments of `seg` bytes at stride `stride` bytes; 3 buffers of 8 GB like pass 1.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ c,
                   size_t n, int seg_d, size_t stride_d, double* out) {
  // segment id s -> base = (s % nseg_per_row) * seg_d + (s / nseg_per_row)...: simple: segments laid out at stride
  const size_t nseg = n / stride_d * (stride_d / seg_d);
  double acc = 0;
  const int lane = threadIdx.x & 31;
  const size_t wid = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  const size_t rows = n / stride_d, per_row = stride_d / seg_d;
  for (size_t s = wid; s < nseg; s += nw) {
    // walk segments "column-major": consecutive s -> same offset within row, next row
    const size_t row = s % rows, col = s / rows;
    const size_t base = row * stride_d + col * seg_d;
    for (int k = lane; k < seg_d; k += 32) acc += a[base + k] + b[base + k] + c[base + k];
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  size_t n = (size_t)1 << 30;  // 8 GB per buffer
  double *a, *b, *c, *o;
  cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8); cudaMalloc(&o, 64);
  cudaMemset(a, 0, n * 8); cudaMemset(b, 0, n * 8); cudaMemset(c, 0, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int segs[] = {16, 32, 128, 512};
  size_t strides[] = {1000, 1024, 1 << 20};
  for (int sg : segs) for (size_t st : strides) {
    rd<<<148 * 8, 256>>>(a, b, c, n, sg, st, o);
    cudaEventRecord(e0);
    rd<<<148 * 8, 256>>>(a, b, c, n, sg, st, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"seg_doubles\":%d,\"stride_doubles\":%zu,\"gbs\":%.0f}\n", sg, st, 3.0 * (n / st) * st * 8 / ms / 1e6);
  }
  return 0;
}
