// micro_issue.cu — does an FP64 DMMA in flight leave its scheduler's issue slots to the other warps?
// 8 warps per CTA, one CTA per SM: warps 0-3 (one per scheduler) run mma.sync.m16n8k4.f64 chains from
// registers, warps 4-7 (the second warp of each scheduler) run a second instruction stream: integer
// IMAD chains, FP64 DADD chains, or shared-memory LDS.64.  Each group is timed alone and together.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/micro_issue tools/micro_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// what: bit 0 = warps 0-3 run DMMAs; bits 1.. = stream of warps 4-7: 0 none, 1 IMAD, 2 DADD, 3 LDS.64
__global__ void __launch_bounds__(256, 1) k_probe(int dm, int other, int iters, long long* cyc, double* sink) {
  __shared__ double sm[4096];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 4096; i += 256) sm[i] = 1.0 + 1e-6 * i;
  __syncthreads();
  long long t0 = 0, t1 = 0;
  double out = 0.0;
  if (w < 4) {
    if (dm) {
      double c[6][4] = {};
      const double a0 = 1.0 + 1e-9 * lane, a1 = 1.0 - 1e-9 * lane, b0 = 1e-3;
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 6; ++k) dmma(c[k], a0, a1, b0);
      }
      t1 = clock64();
      for (int k = 0; k < 6; ++k) out += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    }
  } else if (other == 1) {
    unsigned x0 = tid, x1 = tid + 1, x2 = tid + 2, x3 = tid + 3;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {  // 24 dependent-free-ish IMADs per iteration (4 chains)
        x0 = x0 * 1664525u + 1013904223u;
        x1 = x1 * 1664525u + 1013904223u;
        x2 = x2 * 1664525u + 1013904223u;
        x3 = x3 * 1664525u + 1013904223u;
      }
    }
    t1 = clock64();
    out = (double)(x0 ^ x1 ^ x2 ^ x3);
  } else if (other == 2) {
    double x0 = 1.0 + lane, x1 = 2.0, x2 = 3.0, x3 = 4.0;
    const double d = 1e-9 * (lane + 1);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {  // 24 DADDs per iteration (4 chains)
        x0 = __dadd_rn(x0, d);
        x1 = __dadd_rn(x1, d);
        x2 = __dadd_rn(x2, d);
        x3 = __dadd_rn(x3, d);
      }
    }
    t1 = clock64();
    out = x0 + x1 + x2 + x3;
  } else if (other == 3) {
    double x0 = 0, x1 = 0, x2 = 0, x3 = 0;
    const double* p = sm + lane;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {  // 24 LDS.64 per iteration (conflict-free), results folded with integer ops
        const int o = ((it + k) & 15) * 128;
        double v0, v1, v2, v3;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v0) : "r"((unsigned)__cvta_generic_to_shared(p + o)));
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v1) : "r"((unsigned)__cvta_generic_to_shared(p + o + 32)));
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v2) : "r"((unsigned)__cvta_generic_to_shared(p + o + 64)));
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v3) : "r"((unsigned)__cvta_generic_to_shared(p + o + 96)));
        x0 = __longlong_as_double(__double_as_longlong(x0) ^ __double_as_longlong(v0));
        x1 = __longlong_as_double(__double_as_longlong(x1) ^ __double_as_longlong(v1));
        x2 = __longlong_as_double(__double_as_longlong(x2) ^ __double_as_longlong(v2));
        x3 = __longlong_as_double(__double_as_longlong(x3) ^ __double_as_longlong(v3));
      }
    }
    t1 = clock64();
    out = x0 + x1 + x2 + x3;
  }
  if (lane == 0) cyc[blockIdx.x * 8 + w] = t1 - t0;
  if (out == 123.456) sink[0] = out;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, sizeof(long long) * sms * 8);
  cudaMalloc(&sink, 8);
  const int iters = 20000;
  const char* names[4] = {"none", "IMAD x24", "DADD x24", "LDS.64 x24"};
  long long* h = new long long[sms * 8];
  for (int other = 0; other < 4; ++other) {
    for (int dm = 1; dm >= 0; --dm) {
      if (!dm && !other) continue;
      for (int rep = 0; rep < 2; ++rep) {
        k_probe<<<sms, 256>>>(dm, other, iters, cyc, sink);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, cyc, sizeof(long long) * sms * 8, cudaMemcpyDeviceToHost);
      double cd = 0, co = 0;
      for (int b = 0; b < sms; ++b)
        for (int w = 0; w < 8; ++w) (w < 4 ? cd : co) += (double)h[b * 8 + w];
      cd /= sms * 4.0;
      co /= sms * 4.0;
      printf("DMMA warps %s, other warps %-11s:", dm ? "on " : "off", names[other]);
      if (dm) printf("  %.2f clk per m16n8k4 per scheduler (6 chains)", cd / (iters * 6.0));
      if (other) printf("  %.2f clk per %s instruction per scheduler", co / (iters * 24.0), names[other]);
      printf("\n");
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error: %s\n", cudaGetErrorString(e));
  return 0;
}
