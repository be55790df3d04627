// micro5: DRAM efficiency of pass 2's element-stream pattern (no compute).
// A persistent CTA (256 threads, one per SM) walks pencils of B1 (i1) x 8 (i3)
// along i2 in steps of 8; per step it reads 4 tensors and writes 5 over the
// B1 x 8 x 8 brick (the T, Y_1..3 -> E, D, Y_1..3 streams of k_pass2_fused).
// Prints GB/s for B1 = 16, 32, 64 and for a "banded" vs "linear" pencil order.
#include <cstdio>
#include <cuda_runtime.h>

template <int B1>
__global__ void __launch_bounds__(256) k_stream(const double* __restrict__ in0, const double* __restrict__ in1,
                                                const double* __restrict__ in2, const double* __restrict__ in3,
                                                double* o0, double* o1, double* o2, double* o3, double* o4,
                                                int I1, int I2, int I3, int banded) {
  const int n1b = I1 / B1, n3b = I3 / 8, np = n1b * n3b;
  const long S12 = (long)I1 * I2;
  constexpr int EPT = B1 * 64 / 256;  // elements per thread per step
  for (int lin = blockIdx.x; lin < np; lin += gridDim.x) {
    int ib1, ib3;
    if (banded) {
      const int BW = 12, band = lin / (BW * n3b), li = lin - band * BW * n3b;
      const int bw = min(BW, n1b - band * BW);
      ib1 = band * BW + li % bw;
      ib3 = li / bw;
    } else {
      ib1 = lin % n1b;
      ib3 = lin / n1b;
    }
    for (int i2o = 0; i2o < I2; i2o += 8) {
      double v[EPT];
      long off[EPT];
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int e = threadIdx.x + 256 * k;  // e = l1 + B1 * (l2 + 8 * l3)
        const int l1 = e % B1, l2 = (e / B1) % 8, l3 = e / (B1 * 8);
        off[k] = (long)ib1 * B1 + l1 + (long)I1 * (i2o + l2) + S12 * (ib3 * 8 + l3);
        v[k] = in0[off[k]] + in1[off[k]] + in2[off[k]] + in3[off[k]];
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        o0[off[k]] = v[k];
        o1[off[k]] = v[k] + 1.0;
        o2[off[k]] = v[k] + 2.0;
        o3[off[k]] = v[k] + 3.0;
        o4[off[k]] = v[k] + 4.0;
      }
    }
  }
}

template <int B1>
void run(double** b, int I1, int I2, int I3, int banded, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_stream<B1><<<sms, 256>>>(b[0], b[1], b[2], b[3], b[4], b[5], b[6], b[7], b[8], I1, I2, I3, banded);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 9.0 * 8.0 * I1 * (double)I2 * I3;
  printf("{\"B1\": %d, \"banded\": %d, \"ms\": %.3f, \"GBps\": %.1f}\n", B1, banded, ms, bytes / ms / 1e6);
}

int main() {
  const int I1 = 1024, I2 = 512, I3 = 1024;  // 0.5 G elements, 4 GB per tensor
  const size_t n = (size_t)I1 * I2 * I3;
  double* b[9];
  for (int k = 0; k < 9; ++k) {
    cudaMalloc(&b[k], n * 8);
    cudaMemset(b[k], 0, n * 8);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int banded = 0; banded < 2; ++banded) {
    run<16>(b, I1, I2, I3, banded, sms);
    run<32>(b, I1, I2, I3, banded, sms);
    run<64>(b, I1, I2, I3, banded, sms);
  }
  run<16>(b, I1, I2, I3, 1, 2 * sms);
  run<16>(b, I1, I2, I3, 1, 4 * sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
