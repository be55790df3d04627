// Microbenchmark: DMMA (mma.sync.m16n8k4.f64) throughput when the operands
// come from shared memory, in the pattern of the pass-2 Z products
// (3 products per k-step, 2 A + 1 B LDS.64 each, 2 accumulators per product).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_dmma tools/micro_dmma.cu
// Variants: LDS-fed (as pass 2), half the operands in registers, all in
// registers; 8 or 16 warps per SM; LDS.128 operand pairs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

constexpr int KS = 13, LD = 60, LD2 = 132;

// MODE 0: all operands from smem (pass-2 Z pattern)
// MODE 1: product-1 A and product-3 B in registers (pencil-resident fragments)
// MODE 2: all operands in registers
// MODE 3: LDS.128 pairs (K permuted so a thread's two k-steps are adjacent)
template <int MODE>
__global__ void __launch_bounds__(512) zloop(double* out, int iters) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int i = tid; i < 24000; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const double* U1 = sm;            // [16][LD]
  const double* A1 = sm + 1000;     // [64][LD]
  const double* A2 = sm + 5000;     // [RP][LD2]
  const double* U2 = sm + 13000;    // [8][LD]
  const double* A3 = sm + 14000;    // [RP][LD2]
  const double* U3 = sm + 22000;    // [8][LD]
  double ru1[KS][2], ru3[KS];
  if (MODE == 1 || MODE == 2) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      ru1[ks][0] = U1[g * LD + 4 * ks + t];
      ru1[ks][1] = U1[(g + 8) * LD + 4 * ks + t];
      ru3[ks] = U3[g * LD + 4 * ks + t];
    }
  }
  double z1[4] = {}, z2[4] = {}, z3[4] = {}, y1[4] = {}, y2[4] = {}, y3[4] = {};
  for (int it = 0; it < iters; ++it) {
    const int sh = (it & 1) * 4;  // keep the compiler from hoisting the loads
    if (MODE == 3) {
#pragma unroll
      for (int kp = 0; kp < (KS + 1) / 2; ++kp) {
        const int k = 8 * kp + 2 * t;
        const double2 ua = *reinterpret_cast<const double2*>(U1 + g * LD + k + sh);
        const double2 ub = *reinterpret_cast<const double2*>(U1 + (g + 8) * LD + k + sh);
        const double2 bb = *reinterpret_cast<const double2*>(A1 + (g + 8 * w) * LD + k + sh);
        const double2 u2 = *reinterpret_cast<const double2*>(U2 + g * LD + k + sh);
        const double2 u3 = *reinterpret_cast<const double2*>(U3 + g * LD + k + sh);
        dmma(z1, ua.x, ub.x, bb.x);
        dmma(z2, A2[k * LD2 + g + 16 * w + sh], A2[k * LD2 + g + 8 + 16 * w + sh], u2.x);
        dmma(z3, A3[k * LD2 + g + 16 * w + sh], A3[k * LD2 + g + 8 + 16 * w + sh], u3.x);
        dmma(y1, ua.y, ub.y, bb.y);
        dmma(y2, A2[(k + 1) * LD2 + g + 16 * w + sh], A2[(k + 1) * LD2 + g + 8 + 16 * w + sh], u2.y);
        dmma(y3, A3[(k + 1) * LD2 + g + 16 * w + sh], A3[(k + 1) * LD2 + g + 8 + 16 * w + sh], u3.y);
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int k = 4 * ks + t;
        double(&c1)[4] = (ks & 1) ? y1 : z1;
        double(&c2)[4] = (ks & 1) ? y2 : z2;
        double(&c3)[4] = (ks & 1) ? y3 : z3;
        if (MODE == 2) {
          dmma(c1, ru1[ks][0], ru1[ks][1], ru3[ks]);
          dmma(c2, ru1[ks][1], ru1[ks][0], ru3[ks]);
          dmma(c3, ru1[ks][0], ru3[ks], ru1[ks][1]);
        } else if (MODE == 1) {
          dmma(c1, ru1[ks][0], ru1[ks][1], A1[(g + 8 * w) * LD + k + sh]);
          dmma(c2, A2[k * LD2 + g + 16 * w + sh], A2[k * LD2 + g + 8 + 16 * w + sh], U2[g * LD + k + sh]);
          dmma(c3, A3[k * LD2 + g + 16 * w + sh], A3[k * LD2 + g + 8 + 16 * w + sh], ru3[ks]);
        } else {
          dmma(c1, U1[g * LD + k + sh], U1[(g + 8) * LD + k + sh], A1[(g + 8 * w) * LD + k + sh]);
          dmma(c2, A2[k * LD2 + g + 16 * w + sh], A2[k * LD2 + g + 8 + 16 * w + sh], U2[g * LD + k + sh]);
          dmma(c3, A3[k * LD2 + g + 16 * w + sh], A3[k * LD2 + g + 8 + 16 * w + sh], U3[g * LD + k + sh]);
        }
      }
    }
  }
  double s = 0;
  for (int q = 0; q < 4; ++q) s += z1[q] + z2[q] + z3[q] + y1[q] + y2[q] + y3[q];
  out[blockIdx.x * blockDim.x + tid] = s;
}

template <int MODE>
void run(const char* name, double* out, int threads, int sms) {
  const int ctas_per_sm = 1;
  const int smem = 24000 * 8;
  cudaFuncSetAttribute(zloop<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = sms * ctas_per_sm, iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  zloop<MODE><<<grid, threads, smem>>>(out, 10);
  cudaEventRecord(e0);
  zloop<MODE><<<grid, threads, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = (MODE == 3 ? 2.0 * ((KS + 1) / 2) : (double)KS) * 3.0;
  const double flops = 2.0 * 16 * 8 * 4 * dmmas * iters * grid * (threads / 32);
  printf("{\"kernel\":\"%s\",\"threads\":%d,\"ms\":%.3f,\"tflops\":%.2f,\"err\":\"%s\"}\n", name, threads, ms,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 148 * 512 * sizeof(double));
  const int sms = p.multiProcessorCount;
  for (int th : {256, 512}) {
    run<0>("lds_fed", out, th, sms);
    run<1>("half_regs", out, th, sms);
    run<2>("all_regs", out, th, sms);
    run<3>("lds128_pairs", out, th, sms);
  }
  return 0;
}
