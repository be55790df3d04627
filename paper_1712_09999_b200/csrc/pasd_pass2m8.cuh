// pasd_pass2m8.cuh — fused pass 2 (refold, E/Y/residual, next Procrustes
// products) for order-3 tensors, 8 x 8 x 8 bricks on mma.sync.m8n8k4.f64
// (SASS DMMA.8x8x4), two CTAs per SM.
//
// Same mathematics as k_pass2_fused (pasd_pass2.cuh; reference
// proj/src/pasd.cpp:189-228 and linops.cpp:98).  The 16-row variant needs
// ~215 KB of shared memory and 240 registers, so one CTA per SM serialises
// staging, the elementwise step and the tensor-core products behind block
// barriers.  Here the brick is 8 (i1) x 8 (i2) x 8 (i3) with m8n8k4 tiles,
// the A slices are stored unpadded with an XOR swizzle (conflict-free
// fragment reads), and the CTA fits in ~113 KB / 128 registers: two CTAs per
// SM interleave their phases.  Cost: per-element A-slice traffic R(1/8+1/8)
// instead of R(1/16+1/8), served from L2.
#pragma once
#include "pasd_pass2.cuh"

namespace pasd {

constexpr int M8_THREADS = 256;
#ifndef PASD_M8_CTAS
#define PASD_M8_CTAS 2  // resident CTAs per SM (register budget 65536 / (256 x CTAS))
#endif
constexpr int M8_CTAS = PASD_M8_CTAS;
constexpr int M8_B = 8;  // brick edge

__device__ __forceinline__ void dmma8(double (&c)[2], double a0, double b0) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a0), "d"(b0));
}

// A-slice layout: row r holds 64 doubles (a 8 x 8 column block); element
// (r, c) lives at r*64 + (c ^ (4 * (r & 3))).  Fragment reads of the form
// (rows k0+t, cols b+g) and (rows 8m+g, cols k0+t) hit 16 distinct banks per
// half-warp.
__device__ __forceinline__ int sw(int r, int c) { return r * 64 + (c ^ ((r & 3) << 2)); }
// UM rows: (l, r) at l*LDU + (r ^ (4 * (l & 3))), LDU = RP rounded up to 16 so
// the XOR stays inside the row.
template <int RP>
__device__ __forceinline__ int swu(int l, int r) { return l * ((RP + 15) / 16 * 16) + (r ^ ((l & 3) << 2)); }
// exchange layouts (strides chosen for their write / read patterns)
__device__ __forceinline__ int z8x(int l1, int l2, int l3) { return l1 + 10 * l2 + 82 * l3; }
__device__ __forceinline__ int g28x(int l1, int l2, int l3) { return l1 + 12 * l2 + 96 * l3; }
__device__ __forceinline__ int g38x(int l1, int l2, int l3) { return l1 + 10 * l2 + 84 * l3; }

template <int RP>
struct M8Layout {
  static constexpr int A = RP * 64;
  static constexpr int oA1 = 0, oA2 = A, oA3 = 2 * A;
  static constexpr int LDU = (RP + 15) / 16 * 16;
  static constexpr int oU1 = 3 * A, oU2 = oU1 + 8 * LDU, oU3 = oU2 + 8 * LDU;
  static constexpr int oZ = oU3 + 8 * LDU;
  static constexpr int oG2 = oZ + 656;
  static constexpr int oG3 = oG2 + 768;
  static constexpr int oRed = oG3 + 672;
  static constexpr int total = oRed + 64;
  static constexpr size_t bytes = sizeof(double) * (size_t)total;
};

// EL: storage type of T, E, D, Y_n (float in the fp32 mode; arithmetic in fp64)
template <int RP, class EL = double>
__global__ void __launch_bounds__(M8_THREADS, M8_CTAS) k_pass2_m8(const Pass2Args a, const Ctl* ctl) {
  if (ctl->done) return;
  using L = M8Layout<RP>;
  constexpr int KS = RP / 4;   // k-steps of the Z products
  constexpr int NT = RP / 8;   // n-tiles of Wt_1 / m-tiles of Wt_2^T, Wt_3^T
  extern __shared__ double sm[];
  const ModeDev& m1 = a.m[0];
  const ModeDev& m2 = a.m[1];
  const ModeDev& m3 = a.m[2];
  const int R1 = m1.R, R2 = m2.R, R3 = m3.R;
  const int64_t I1 = m1.I, I2 = m2.I, I3 = m3.I;
  double* A1s = sm + L::oA1;
  double* A2s = sm + L::oA2;
  double* A3s = sm + L::oA3;
  double* U1s = sm + L::oU1;
  double* U2s = sm + L::oU2;
  double* U3s = sm + L::oU3;
  double* Zx = sm + L::oZ;
  double* G2x = sm + L::oG2;
  double* G3x = sm + L::oG3;
  double* red = sm + L::oRed;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;

  const EL* __restrict__ T = reinterpret_cast<const EL*>(a.T);
  EL* __restrict__ Enew = reinterpret_cast<EL*>(ctl->ecur ? a.E0 : a.E1);
  EL* __restrict__ Dp = reinterpret_cast<EL*>(a.D);
  EL* const Yp[3] = {reinterpret_cast<EL*>(a.Y[0]), reinterpret_cast<EL*>(a.Y[1]), reinterpret_cast<EL*>(a.Y[2])};
  const double mu = ctl->mu;
  const double inv_mu = __ddiv_rn(1.0, mu);                // pasd.cpp:170
  const double inv_n = __ddiv_rn(1.0, 3.0);                // pasd.cpp:204
  const double tau = __ddiv_rn(1.0, __dmul_rn(mu, 3.0));   // pasd.cpp:205
  const double cand = __dmul_rn(ctl->rho, mu);
  const double mu_next = (ctl->mu_max < cand) ? ctl->mu_max : cand;
  const double inv_mu_next = __ddiv_rn(1.0, mu_next);

  double* W2c = a.W2part + (int64_t)blockIdx.x * I2 * R2;  // per-CTA Wt_2 partial
  for (int64_t idx = tid; idx < I2 * R2; idx += M8_THREADS) W2c[idx] = 0.0;
  // zero everything once: padding rows/cols (r >= R_n) are never written by staging
  for (int idx = tid; idx < L::oZ; idx += M8_THREADS) sm[idx] = 0.0;

  double worst[3] = {0.0, 0.0, 0.0};
  double gsq[3] = {0.0, 0.0, 0.0};
  int bad = 0;
  const int64_t S12 = I1 * I2;
  const int ksz = (max(R1, max(R2, R3)) + 3) / 4;  // Z k-steps that touch a nonzero rank row
  const bool al1 = (I1 % 2) == 0;
#if PASD_P2_TIMING
  unsigned long long ph_acc[12] = {};
  long long ph_t = clock64();
#endif

  // Work items: pencil x i2 segment (segments keep small tensors, where the
  // pencil count is near the CTA count, from ending on a partial wave).
  const int64_t seg_len = (((I2 + M8_B - 1) / M8_B + a.nseg - 1) / a.nseg) * M8_B;
  for (int item = blockIdx.x; item < a.npencils * a.nseg; item += gridDim.x) {
    const int seg = item / a.npencils, lin = item - seg * a.npencils;
    const int64_t i2b = seg * seg_len, i2e = imin64(I2, i2b + seg_len);
    int ib1, ib3;
    {  // banded order: concurrent pencils form ~12 x 25 patches of (i1, i3) blocks
      const int BW = 12;
      const int band = lin / (BW * a.n3b), lin_in = lin - band * BW * a.n3b;
      const int bw = min(BW, a.n1b - band * BW);
      ib1 = band * BW + lin_in % bw;
      ib3 = lin_in / bw;
    }
    const int pen = ib1 + a.n1b * ib3 + a.npencils * seg;  // index of the Wt_1 / Wt_3 partials
    const int64_t i1o = (int64_t)ib1 * M8_B, i3o = (int64_t)ib3 * M8_B;
    const int nv1 = (int)imin64(M8_B, I1 - i1o);
    __syncthreads();
    // ---- pencil-resident: A_2 (I1, R2, I3) slice rows (r, l3) of 8 i1; UM_1, UM_3 rows ----
    {
      const int c = tid & 3;  // 16-byte piece of an 8-double run
      const int v = nv1 - 2 * c, nbc = v >= 2 ? 16 : (v == 1 ? 8 : 0);
      for (int row = tid >> 2; row < 8 * R2; row += M8_THREADS / 4) {
        const int l3 = row & 7, r = row >> 3;
        const int nb = (i3o + l3 < I3) ? nbc : 0;
        double* dst = A2s + sw(r, 8 * l3 + 2 * c);
        const double* src = m2.A + i1o + 2 * c + I1 * ((int64_t)r + (int64_t)R2 * (i3o + l3));
        if (al1)
          cp_async16(dst, nb ? src : m2.A, nb);
        else {
          cp_async8(dst, nb >= 8 ? src : m2.A, nb >= 8);
          cp_async8(dst + 1, nb >= 16 ? src + 1 : m2.A, nb >= 16);
        }
      }
    }
    for (int idx = tid; idx < 8 * R1; idx += M8_THREADS) {
      const int l1 = idx & 7, r = idx >> 3;
      const bool v = l1 < nv1;
      cp_async8(U1s + swu<RP>(l1, r), v ? m1.UM + m1.ioff + i1o + l1 + m1.Ifull * r : m1.UM, v);
    }
    for (int idx = tid; idx < 8 * R3; idx += M8_THREADS) {
      const int l3 = idx & 7, r = idx >> 3;
      const bool v = i3o + l3 < I3;
      cp_async8(U3s + swu<RP>(l3, r), v ? m3.UM + m3.ioff + i3o + l3 + m3.Ifull * r : m3.UM, v);
    }
    double w1acc[NT][2];  // Wt_1 (8 i1 x R1) over this warp's columns (i3 = w)
#pragma unroll
    for (int j = 0; j < NT; ++j) w1acc[j][0] = w1acc[j][1] = 0.0;
    double w3acc[2][2] = {};  // Wt_3^T m-tiles (w-4) and (w), warps 4..7

    // Per-step staging with per-thread address bases hoisted out of the copy
    // loops (the swizzle term is fixed per thread, so a thread's copies are
    // a constant stride apart in shared memory).
    auto stage_step = [&](int64_t i2o) {
      {  // A_1 (R1, I2, I3): column (i2, i3) holds R1 contiguous values; thread -> column c, rows r0 + 4k
        const int c = tid >> 2, l2 = c & 7, l3 = c >> 3, r0 = tid & 3;
        const int64_t i2 = i2o + l2, i3 = i3o + l3;
        const bool colok = i2 < I2 && i3 < I3;
        const double* src = colok ? m1.A + (int64_t)R1 * (i2 + I2 * i3) + r0 : m1.A;
        const int sst = colok ? 4 : 0;
        const unsigned d0 = smem_u32(A1s + sw(r0, c));
#pragma unroll
        for (int k = 0; k < RP / 4; ++k)
          if (r0 + 4 * k < R1) cp8s(d0 + 8u * 256u * k, src + k * sst, colok ? 8 : 0);
      }
      {  // A_3 (I1, I2, R3): rows (r, l2) of 8 consecutive i1; thread -> piece c, l2, rows r = tid/32 + 8k
        const int c = tid & 3, l2 = (tid >> 2) & 7, rb = tid >> 5;
        const int v = nv1 - 2 * c, nbc = v >= 2 ? 16 : (v == 1 ? 8 : 0);
        const int nb = (i2o + l2 < I2) ? nbc : 0;
        const double* src = nb ? m3.A + i1o + 2 * c + I1 * (i2o + l2) + S12 * (int64_t)rb : m3.A;
        const int64_t sst = nb ? 8 * S12 : 0;
        const unsigned d0 = smem_u32(A3s + sw(rb, 8 * l2 + 2 * c));
        if (al1) {
#pragma unroll
          for (int k = 0; k < (RP + 7) / 8; ++k)
            if (rb + 8 * k < R3) cp16s(d0 + 8u * 512u * k, src + k * sst, nb);
        } else {
          const int n0 = nb >= 8 ? 8 : 0, n1 = nb >= 16 ? 8 : 0;
#pragma unroll
          for (int k = 0; k < (RP + 7) / 8; ++k)
            if (rb + 8 * k < R3) {
              cp8s(d0 + 8u * 512u * k, n0 ? src + k * sst : m3.A, n0);
              cp8s(d0 + 8u * 512u * k + 8u, n1 ? src + k * sst + 1 : m3.A, n1);
            }
        }
      }
      {  // UM_2 rows of the step: thread -> (l2, r = tid / 8 + 32 k)
        const int l2 = tid & 7, rb = tid >> 3;
        const bool v = i2o + l2 < I2;
        const double* src = v ? m2.UM + m2.ioff + i2o + l2 + m2.Ifull * rb : m2.UM;
        const int64_t sst = v ? 32 * m2.Ifull : 0;
        const unsigned d0 = smem_u32(U2s + swu<RP>(l2, rb));
#pragma unroll
        for (int k = 0; k < (RP + 31) / 32; ++k)
          if (rb + 32 * k < R2) cp8s(d0 + 8u * 32u * k, src + k * sst, v ? 8 : 0);
      }
    };
    // this thread's 2 elements: i1 = g, i2 = 2t + p, i3 = w
    double tv[2], yv[3][2];
    bool inb[2];
    int64_t off[2];
    auto load_elems = [&](int64_t i2o) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int64_t i1 = i1o + g, i2 = i2o + 2 * t + p, i3 = i3o + w;
        inb[p] = i1 < I1 && i2 < I2 && i3 < I3;
        off[p] = i1 + I1 * i2 + S12 * i3;
        tv[p] = inb[p] ? T[off[p]] : 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) yv[n][p] = inb[p] ? (double)Yp[n][off[p]] : 0.0;
      }
    };
    stage_step(i2b);
    load_elems(i2b);

    for (int64_t i2o = i2b; i2o < i2e; i2o += M8_B) {
      P2T(0);
      cp_async_wait_all();
      P2T(1);
      __syncthreads();
      P2T(2);
      // ---- Z products: three 8x8 tiles per warp, 2 chains each ----
      double z1[2] = {0, 0}, z2[2] = {0, 0}, z3[2] = {0, 0};
      {
        double y1[2] = {0, 0}, y2[2] = {0, 0}, y3[2] = {0, 0};
        // k-steps past max R_n only multiply zero padding; ksz is KS - 1 or KS
        // (RP = max R_n rounded up to 8), so the first KS - 1 run branch-free
        auto zstep = [&](int ks) {
          const int k = 4 * ks + t;
          double(&c1)[2] = (ks & 1) ? y1 : z1;
          double(&c2)[2] = (ks & 1) ? y2 : z2;
          double(&c3)[2] = (ks & 1) ? y3 : z3;
          dmma8(c1, U1s[swu<RP>(g, k)], A1s[sw(k, g + 8 * w)]);  // rows i1, cols i2 at i3 = w
          dmma8(c2, A2s[sw(k, g + 8 * w)], U2s[swu<RP>(g, k)]);  // rows i1, cols i2 at i3 = w
          dmma8(c3, A3s[sw(k, g + 8 * w)], U3s[swu<RP>(g, k)]);  // rows i1, cols i3 at i2 = w
        };
#pragma unroll
        for (int ks = 0; ks < KS - 1; ++ks) zstep(ks);
        if (ksz == KS) zstep(KS - 1);
        z1[0] += y1[0]; z1[1] += y1[1];
        z2[0] += y2[0]; z2[1] += y2[1];
        z3[0] += y3[0]; z3[1] += y3[1];
      }
      Zx[z8x(g, w, 2 * t)] = z3[0];
      Zx[z8x(g, w, 2 * t + 1)] = z3[1];
      P2T(3);
      __syncthreads();
      P2T(4);
      // ---- elementwise (reference op order, no FMA contraction) ----
      double g1v[2];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int l2 = 2 * t + p;
        const double zz[3] = {z1[p], z2[p], Zx[z8x(g, l2, w)]};
        const double tt = tv[p];
        double zt[3], h = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          zt[n] = __dsub_rn(tt, zz[n]);
          h = __dadd_rn(h, __dadd_rn(zt[n], __dmul_rn(yv[n][p], inv_mu)));  // pasd.cpp:202
        }
        const double e = PASD_P2_SOFTSEL ? soft_sel(__dmul_rn(h, inv_n), tau) : soft(__dmul_rn(h, inv_n), tau);  // pasd.cpp:208
        double gn[3];
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          const double r = __dsub_rn(zt[n], e);                       // pasd.cpp:220
          const double ynew = __dadd_rn(yv[n][p], __dmul_rn(mu, r));  // pasd.cpp:221
#if PASD_P2_SOFTSEL
          // entries outside the tensor have T = Y_n = Z_n = 0, so r = 0 there: only the store is guarded
          const double ar = fabs(r);
          worst[n] = ar > worst[n] ? ar : worst[n];
          bad |= !isfinite(r);
          if (inb[p]) Yp[n][off[p]] = (EL)ynew;
#else
          if (inb[p]) {
            const double ar = fabs(r);
            if (ar > worst[n]) worst[n] = ar;
            bad |= !isfinite(r);
            Yp[n][off[p]] = (EL)ynew;
          }
#endif
          gn[n] = inb[p] ? g_elem(tt, e, ynew, inv_mu_next) : 0.0;
          gsq[n] = fma(gn[n], gn[n], gsq[n]);
        }
        if (inb[p]) {
          Enew[off[p]] = (EL)e;
          Dp[off[p]] = (EL)__dsub_rn(tt, e);  // next pass 1 reads D = T - E
        }
        g1v[p] = gn[0];
        G2x[g28x(g, l2, w)] = gn[1];
        G3x[g38x(g, l2, w)] = gn[2];
      }
      const bool more = i2o + M8_B < i2e;
      if (more) load_elems(i2o + M8_B);  // next step's T, Y in flight during the Wt products
      P2T(5);
      __syncthreads();
      P2T(6);
      // ---- Wt_1: A operand = own G_1 (cols permuted: lane t supplies i2 = 2t + p) ----
#pragma unroll
      for (int p = 0; p < 2; ++p) {
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma8(w1acc[j], g1v[p], A1s[sw(8 * j + g, 8 * w + 2 * t + p)]);
      }
      // ---- Wt_3^T (warps 4..7, m-tiles w-4 and w): K = (i1, i2) = 64, kept per pencil ----
      double w2acc[2][2] = {};
      double w2old[2][2] = {};
      if (w >= 4) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int mt = (w - 4) + 4 * h;
          if (mt < NT) {
            double acc[2][2] = {};
#pragma unroll
            for (int ks = 0; ks < 16; ++ks) {
              const int k = 4 * ks + t;
              dmma8(acc[ks & 1], A3s[sw(8 * mt + g, k)], G3x[g38x(k & 7, k >> 3, g)]);
            }
            w3acc[h][0] += acc[0][0] + acc[1][0];
            w3acc[h][1] += acc[0][1] + acc[1][1];
          }
        }
      } else {
        // ---- Wt_2^T (warps 0..3, m-tiles w and w+4): K = (i1, i3) = 64, flushed per step ----
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int mt = w + 4 * h;
          if (mt < NT) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int r = 8 * mt + g;
              const int64_t i2 = i2o + 2 * t + q;
              if (r < R2 && i2 < I2) w2old[h][q] = W2c[i2 * R2 + r];
            }
            double acc[2][2] = {};
#pragma unroll
            for (int ks = 0; ks < 16; ++ks) {
              const int k = 4 * ks + t;
              dmma8(acc[ks & 1], A2s[sw(8 * mt + g, k)], G2x[g28x(k & 7, g, k >> 3)]);
            }
            w2acc[h][0] = acc[0][0] + acc[1][0];
            w2acc[h][1] = acc[0][1] + acc[1][1];
          }
        }
      }
      P2T(7);
      __syncthreads();  // A1s / A3s / U2s free: stage the next step under the Wt_2 flush
      P2T(8);
      if (more) stage_step(i2o + M8_B);
      P2T(9);
      if (w < 4) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int mt = w + 4 * h;
          if (mt < NT) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int r = 8 * mt + g;
              const int64_t i2 = i2o + 2 * t + q;
              if (r < R2 && i2 < I2) W2c[i2 * R2 + r] = w2old[h][q] + w2acc[h][q];
            }
          }
        }
      }
      P2T(10);
    }
    // ---- end of pencil: Wt_1 (sum of the 8 warps' column sets) and Wt_3 ----
    __syncthreads();
    double* wred = A1s;  // 8 warps x 8 x RP doubles <= A1s + A2s
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      wred[(w * 8 + g) * RP + 8 * j + 2 * t] = w1acc[j][0];
      wred[(w * 8 + g) * RP + 8 * j + 2 * t + 1] = w1acc[j][1];
    }
    __syncthreads();
    double* w1out = a.W1p + (int64_t)pen * 8 * R1;
    for (int idx = tid; idx < 8 * R1; idx += M8_THREADS) {
      const int l1 = idx / R1, r = idx - l1 * R1;
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s += wred[(ww * 8 + l1) * RP + r];
      w1out[idx] = s;
    }
    if (w >= 4) {
      double* w3out = a.W3p + (int64_t)pen * 8 * R3;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int mt = (w - 4) + 4 * h;
        if (mt < NT) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int r = 8 * mt + g;
            if (r < R3) w3out[(2 * t + q) * R3 + r] = w3acc[h][q];
          }
        }
      }
    }
    __syncthreads();
    // restore zero padding clobbered by the reduction scratch (rows >= R1 of A1s, A2s)
    for (int idx = tid; idx < 2 * L::A; idx += M8_THREADS) {
      const int r = (idx % L::A) / 64;
      const int Rn = idx < L::A ? R1 : R2;
      if (r >= Rn) sm[idx] = 0.0;
    }
  }
#if PASD_P2_TIMING
  P2T(11);
  if (tid == 0)
    for (int k = 0; k < 12; ++k) atomicAdd(&g_p2_phase[k], ph_acc[k]);
#endif
  for (int n = 0; n < 3; ++n) {
    const double wv = block_reduce(worst[n], MaxOp(), red);
    const double gv = block_reduce(gsq[n], AddOp(), red);
    if (tid == 0) {
      a.resid_part[(int64_t)blockIdx.x * PASD_MAX_ORDER + n] = wv;
      a.gpart[blockIdx.x * 3 + n] = gv;
    }
  }
  int* redi = reinterpret_cast<int*>(red + 32);
  const int b = block_reduce(bad, OrOp(), redi);
  if (tid == 0) a.bad_part[blockIdx.x] = b;
  __syncthreads();  // the block reductions above are done with `red`
  if (a.finish_ticket && last_cta(a.finish_ticket, reinterpret_cast<int*>(red + 48)))
    finish_body(const_cast<Ctl*>(ctl), a.resid_part, a.bad_part, gridDim.x, a.history, nullptr, red);
}

template <int RP>
void launch_m8(const Pass2Args& a, const Ctl* ctl, int grid, cudaStream_t st, bool f32 = false) {
  if constexpr (RP <= 24) {  // float storage (fp32 mode) where this kernel is the default
    if (f32) {
      k_pass2_m8<RP, float><<<grid, M8_THREADS, M8Layout<RP>::bytes, st>>>(a, ctl);
      return;
    }
  }
  k_pass2_m8<RP><<<grid, M8_THREADS, M8Layout<RP>::bytes, st>>>(a, ctl);
}
template <int RP>
void setup_m8() {
  cudaFuncSetAttribute(k_pass2_m8<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)M8Layout<RP>::bytes);
  if constexpr (RP <= 24)
    cudaFuncSetAttribute(k_pass2_m8<RP, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)M8Layout<RP>::bytes);
}
// Measured on B200 (profiles/): the 8x8x8 two-CTA variant wins for R <= 24
// (C1: 0.122 vs 0.129 ms, C2: 0.516 vs 0.565 ms per iteration), the 16x8x8
// variant from R = 32 on (C4: 3.04 vs 3.09 ms; C3, C5).
inline bool m8_supported(int rp) { return rp <= 24; }
inline void m8_setup(int rp) {
  switch (rp) {
    case 8: setup_m8<8>(); break;
    case 16: setup_m8<16>(); break;
    case 24: setup_m8<24>(); break;
    case 32: setup_m8<32>(); break;
    case 40: setup_m8<40>(); break;
    case 48: setup_m8<48>(); break;
    default: setup_m8<56>(); break;
  }
}
inline void m8_launch(int rp, const Pass2Args& a, const Ctl* ctl, int grid, cudaStream_t st, bool f32 = false) {
  switch (rp) {
    case 8: launch_m8<8>(a, ctl, grid, st, f32); break;
    case 16: launch_m8<16>(a, ctl, grid, st, f32); break;
    case 24: launch_m8<24>(a, ctl, grid, st, f32); break;
    case 32: launch_m8<32>(a, ctl, grid, st); break;
    case 40: launch_m8<40>(a, ctl, grid, st); break;
    case 48: launch_m8<48>(a, ctl, grid, st); break;
    default: launch_m8<56>(a, ctl, grid, st); break;
  }
}

}  // namespace pasd
