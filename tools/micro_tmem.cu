// micro_tmem.cu — can tensor memory (TMEM) serve as a per-thread operand store for the FP64 DMMA
// products of pass 2?  Measures tcgen05.ld (32x32b, x16 = 8 doubles per thread) throughput per SM
// with 8 warps, alone and interleaved with mma.sync.m16n8k4.f64 in the Z-product pattern
// (5 of the 9 operand doubles per k-step from TMEM, the other 4 from shared memory).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/micro_tmem tools/micro_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__);       \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void tm_ld16(uint32_t (&r)[16], uint32_t taddr) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ double as_double(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

// mode 0: TMEM loads only; 1: Z pattern with all 9 operands from shared memory; 2: Z pattern, 5 from TMEM
// modes 3 / 4 = modes 1 / 2 with the element streams of a pass-2 step in flight: 16 LDG.64 per thread issued
// before the products (64-byte row segments, streaming), consumed after them, then 20 STG.64 per thread
__global__ void __launch_bounds__(256, 1) k_probe(int mode_in, int iters, double* out, long long* cyc,
                                                  const double* __restrict__ src, double* __restrict__ dst,
                                                  long long nsrc) {
  const bool traffic = mode_in >= 3;
  const int mode = traffic ? mode_in - 2 : mode_in;
  extern __shared__ double sm[];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  for (int i = tid; i < 8192; i += 256) sm[i] = 1.0 + 1e-3 * (i % 97);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"l"(
        (uint64_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // this warp's window: lanes 32 (w % 4) .., columns 256 (w / 4) .. + 255
  const uint32_t tw = tbase + ((uint32_t)(32 * (w & 3)) << 16) + 256u * (w >> 2);
  for (int c = 0; c < 256; c += 16) {
    uint32_t r[16];
    for (int k = 0; k < 16; k += 2) {
      const double v = 1.0 + 1e-3 * ((c + k + tid) % 89);
      r[k] = (uint32_t)__double2loint(v);
      r[k + 1] = (uint32_t)__double2hiint(v);
    }
    tm_st16(tw + c, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  double acc[6][4] = {};
  double s = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double ev[16];
    long long eoff[4];
    const bool tr = traffic && (it & 3) == 0;  // one step of the real kernel ~ 4 Z phases
    if (tr) {
      const long long brick = ((long long)it * gridDim.x + blockIdx.x) * 1024 % (nsrc / 4 - 1024);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        eoff[q] = brick + (g + 8 * (q >> 1)) + 16 * ((2 * t + (q & 1)) + 8 * w);
#pragma unroll
        for (int n = 0; n < 4; ++n) ev[4 * q + n] = src[eoff[q] + n * (nsrc / 4)];
      }
    }
    if (mode == 0) {
#pragma unroll
      for (int c = 0; c < 256; c += 16) {
        uint32_t r[16];
        tm_ld16(r, tw + c);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        s += as_double(r[0], r[1]) + as_double(r[14], r[15]);
      }
    } else {
      // 14 k-steps of the Z pattern: 3 DMMAs, operands (a0, a1, b) x 3
#pragma unroll
      for (int ks = 0; ks < 14; ks += 2) {  // two k-steps per 16-register TMEM load (5 doubles each, 10 of 16 used... use 8 + 2 from the next)
        uint32_t r[16] = {};
        if (mode == 2) {
          tm_ld16(r, tw + 16 * (ks / 2));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = 4 * (ks + h) + t;
          double u1a, u1b, a2a, a2b, u3;
          if (mode == 2) {  // pencil-constant operands from TMEM (4 per k-step here; the fifth shares a load in the kernel)
            u1a = as_double(r[8 * h + 0], r[8 * h + 1]);
            u1b = as_double(r[8 * h + 2], r[8 * h + 3]);
            a2a = as_double(r[8 * h + 4], r[8 * h + 5]);
            a2b = as_double(r[8 * h + 6], r[8 * h + 7]);
            u3 = sm[7000 + g * 60 + k];
          } else {
            u1a = sm[g * 60 + k];
            u1b = sm[(g + 8) * 60 + k];
            a2a = sm[1000 + k * 132 + g + 16 * (w & 3)];
            a2b = sm[1000 + k * 132 + g + 8 + 16 * (w & 3)];
            u3 = sm[7000 + g * 60 + k];
          }
          const double a1 = sm[2000 + (g + 8 * (w & 3)) * 60 + k];
          const double u2 = sm[6000 + g * 60 + k];
          const double a3a = sm[3000 + (k & 15) * 132 + g + 16 * (w & 3)];
          const double a3b = sm[3000 + (k & 15) * 132 + g + 8 + 16 * (w & 3)];
          dmma(acc[0 + h], u1a, u1b, a1);
          dmma(acc[2 + h], a2a, a2b, u2);
          dmma(acc[4 + h], a3a, a3b, u3);
        }
      }
    }
    if (tr) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double v = ev[4 * q] + ev[4 * q + 1] + ev[4 * q + 2] + ev[4 * q + 3] + acc[q][0];
#pragma unroll
        for (int n = 0; n < 5; ++n) dst[eoff[q] + n * (nsrc / 4)] = v + n;
      }
    }
  }
  const long long t1 = clock64();
  for (int i = 0; i < 6; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * 256 + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  const int grid = 148, iters = 2000;
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, grid * 256 * sizeof(double)));
  CK(cudaMalloc(&cyc, grid * sizeof(long long)));
  const long long nsrc = 4ll * 64 * 1024 * 1024;  // 4 streams of 512 MB
  double *src, *dst;
  CK(cudaMalloc(&src, nsrc * sizeof(double)));
  CK(cudaMalloc(&dst, (nsrc / 4) * 5 * sizeof(double)));
  CK(cudaMemset(src, 0, nsrc * sizeof(double)));
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      k_probe<<<grid, 256, 160 * 1024>>>(mode, iters, out, cyc, src, dst, nsrc);
      CK(cudaDeviceSynchronize());
    }
    long long h[148];
    CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < grid; ++i) avg += (double)h[i] / grid;
    if (mode == 0) {
      const double bytes = (double)iters * 16 * 64.0 * 256;  // 16 loads x 64 B per thread per iteration
      printf("mode 0 (tcgen05.ld x16 only, 8 warps): %.0f cycles, %.1f B/clk/SM\n", avg, bytes / avg);
    } else {
      const double dm = (double)iters * 14 * 3 * 8;  // DMMAs per CTA
      printf("mode %d (Z pattern, %s%s): %.0f cycles, %.2f clk per DMMA per SM (peak 8), %.0f cycles per step\n", mode,
             (mode == 1 || mode == 3) ? "all operands from shared memory" : "4 of 9 operand doubles from TMEM",
             mode >= 3 ? ", element streams in flight" : "", avg, avg / dm, avg / iters);
    }
  }
  return 0;
}
