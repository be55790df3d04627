// pasd_pass2ts.cuh — fused pass 2 (pasd_pass2.cuh) as two warp teams per CTA.
//
// Same mathematics, brick walk, shared-memory slice layouts, bulk-staged slices
// (k_retile) and partial-sum layouts as k_pass2_fused (reference:
// proj/src/pasd.cpp:189-228, linops.cpp:98), and bit-identical results: every
// product keeps its k order and its partial-sum tree.  What changes is who runs
// what.  ncu's per-instruction samples of k_pass2_fused showed each warp's
// timeline to be serial — a DMMA.8x8x4 holds its warp for 16 cycles, the
// operand loads of a k-step wait ~120 cycles behind the other warps' loads, the
// elementwise phase issues no DMMA at all — with only two warps per scheduler,
// all in the same phase.  Here 16 warps form two teams that are in different
// phases at any time:
//   team A (warps 0-7): T / Y_n element loads, Z_1 and Z_2 products (their
//     accumulators are the element layout), the elementwise phase, E / D / Y_n
//     stores; G_1, G_2, G_3 of the step go to shared memory.
//   team B (warps 8-15): the Z_3 products (exchanged through shared memory in
//     the fused kernel too), and all Wt products: Wt_2 of the previous step
//     while team A runs the elementwise phase (two G_2 buffers), then Wt_3 and
//     Wt_1 of this step, releasing the A_3 / A_1 slices for the next bulk copy.
// Hand-offs are named barriers (arrive on one side, sync on the other):
// "Z_3 ready" (B -> A) and "G ready" (A -> B).  128 registers per thread.
#pragma once
#include "pasd_pass2.cuh"

namespace pasd {

#ifndef PASD_P2_TS
#define PASD_P2_TS 1  // compile k_pass2_ts in; selected at run time with PASD_P2_TS=1 in the environment
                      // (measured slower than k_pass2_fused: see DESIGN.md "Pass 2, round 2")
#endif
constexpr int TS_THREADS = 512;

// G_1 exchange: read as the B operand of Wt_1 (l1 = g, l2 = t + c: conflict-free), written (l1 = g, l2 = 2t: 2-way)
__device__ __forceinline__ int g1x(int l1, int l2, int l3) { return l1 + 20 * l2 + 164 * l3; }
__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int RP>
struct P2TsLayout {
  using F = P2Layout<RP, false>;
  static constexpr int RM = F::RM;
  static constexpr int LD1 = F::LD1, LD2 = F::LD2, LD3 = F::LD3, LDU = F::LDU;  // = the tiled copies (k_retile)
  static constexpr int oA1 = 0;
  static constexpr int oA2 = oA1 + 64 * LD1;
  static constexpr int oA3 = oA2 + RP * LD2;
  static constexpr int oU1 = oA3 + RP * LD3;
  static constexpr int oU2 = oU1 + 16 * LDU;
  static constexpr int oU3 = oU2 + 8 * LDU;
  static constexpr int oZ3 = oU3 + 8 * LDU;
  static constexpr int oG1 = oZ3 + 8 * 182;
  static constexpr int oG2 = oG1 + 8 * 164;      // two buffers (step parity)
  static constexpr int oG3 = oG2 + 2 * 8 * 160;
  static constexpr int oX2 = oG3 + 8 * 180;      // Wt_2 K-half exchange
  static constexpr int oRed = oX2 + 512;
  static constexpr int total = oRed + 64;
  static constexpr size_t bytes = sizeof(double) * (size_t)total;
  static_assert((RM - RP) * LD3 <= total - oU1, "M-tile overrun must stay inside shared memory");
  static_assert(4 * 32 * 12 <= 8 * 182 + 8 * 164, "end-of-pencil exchange fits in Z3s + G1s");
};

template <int RP>
constexpr bool ts_fits() {
  return P2TsLayout<RP>::bytes <= 227u * 1024u;
}

#if PASD_P2_TIMING
#define TST(k)                                          \
  do {                                                  \
    if (lane == 0 && w == 0) {                          \
      const long long now_ = clock64();                 \
      ph_acc[k] += (unsigned long long)(now_ - ph_t);   \
      ph_t = now_;                                      \
    }                                                   \
  } while (0)
#else
#define TST(k) do {} while (0)
#endif
template <int RP, class EL = double>
__global__ void __launch_bounds__(TS_THREADS, 1) k_pass2_ts(const Pass2Args a, const Ctl* ctl) {
  if (ctl->done) return;
  using L = P2TsLayout<RP>;
  constexpr int KS = RP / 4;
  constexpr int MT = L::RM / 16;
  constexpr unsigned kBytesA1 = 64u * L::LD1 * 8u, kBytesA2 = (unsigned)RP * L::LD2 * 8u,
                     kBytesA3 = (unsigned)RP * L::LD3 * 8u, kBytesU2 = 8u * L::LDU * 8u;
  constexpr int BAR_Z3 = 8, BAR_G = 9;  // named barriers (1..4: Wt_2 K-half pairs)
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
  double* Z3s = sm + L::oZ3;
  double* G1s = sm + L::oG1;
  double* G2s = sm + L::oG2;
  double* G3s = sm + L::oG3;
  double* X2s = sm + L::oX2;
  double* red = sm + L::oRed;
  uint64_t* full_s = reinterpret_cast<uint64_t*>(red + 57);
  uint64_t* full_p = reinterpret_cast<uint64_t*>(red + 58);
  int* rel3 = reinterpret_cast<int*>(red + 59);
  int* rel1 = rel3 + 1;
  unsigned phs = 0, php = 0;
  const int tid = threadIdx.x, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const bool teamB = tid >= 256;  // warp-uniform
  const int w = (tid >> 5) & 7;   // warp within its team

  const EL* __restrict__ T = reinterpret_cast<const EL*>(a.T);
  EL* __restrict__ Enew = reinterpret_cast<EL*>(ctl->ecur ? a.E0 : a.E1);
  EL* __restrict__ Dp = reinterpret_cast<EL*>(a.D);
  EL* const Yp[3] = {reinterpret_cast<EL*>(a.Y[0]), reinterpret_cast<EL*>(a.Y[1]), reinterpret_cast<EL*>(a.Y[2])};
  const double mu = ctl->mu;
  const double inv_mu = __ddiv_rn(1.0, mu);               // pasd.cpp:170
  const double inv_n = __ddiv_rn(1.0, 3.0);               // pasd.cpp:204
  const double tau = __ddiv_rn(1.0, __dmul_rn(mu, 3.0));  // pasd.cpp:205
  const double cand = __dmul_rn(ctl->rho, mu);
  const double mu_next = (ctl->mu_max < cand) ? ctl->mu_max : cand;
  const double inv_mu_next = __ddiv_rn(1.0, mu_next);

  const bool w2s = a.nw2 == 2 * (int)gridDim.x;  // one Wt_2 partial per K-half (no exchange)
  const int NW2 = w2s ? 2 : 1;
  double* W2c = a.W2part + (int64_t)blockIdx.x * NW2 * I2 * R2;
  for (int64_t idx = tid; idx < NW2 * I2 * R2; idx += TS_THREADS) W2c[idx] = 0.0;
  const int mt = w & 3, kh = w >> 2;  // team B: m-tile and K-half of the Wt_2 / Wt_3 products
  double* W2k = W2c + (w2s ? (int64_t)kh * I2 * R2 : 0);
  for (int idx = tid; idx < L::total - L::oU1; idx += TS_THREADS) U1s[idx] = 0.0;  // UM rows, exchange buffers, red
  __syncthreads();
  if (tid == 0) {
    mbar_init_n(full_s, 3);
    mbar_init_n(full_p, 1);
    *rel3 = 0;
    *rel1 = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double worst[3] = {0.0, 0.0, 0.0};
  double gsq[3] = {0.0, 0.0, 0.0};
  int bad = 0;
  const int64_t S12 = I1 * I2;
  const int ksz = (max(R1, max(R2, R3)) + 3) / 4;  // Z k-steps that touch a nonzero rank row
#if PASD_P2_TIMING
  unsigned long long ph_acc[12] = {};
  long long ph_t = clock64();
#endif

  const int64_t seg_len = (((I2 + P2_B2 - 1) / P2_B2 + a.nseg - 1) / a.nseg) * P2_B2;
  for (int item = blockIdx.x; item < a.npencils * a.nseg; item += gridDim.x) {
    const int seg = item / a.npencils, lin = item - seg * a.npencils;
    const int64_t i2b = seg * seg_len, i2e = imin64(I2, i2b + seg_len);
    int ib1, ib3;
    {  // banded pencil order (see k_pass2_fused)
      const int BW = PASD_P2_BW;
      const int band = lin / (BW * a.n3b), lin_in = lin - band * BW * a.n3b;
      const int bw = min(BW, a.n1b - band * BW);
      ib1 = band * BW + lin_in % bw;
      ib3 = lin_in / bw;
    }
    const int pen = ib1 + a.n1b * ib3 + a.npencils * seg;
    const int64_t i1o = (int64_t)ib1 * P2_B1, i3o = (int64_t)ib3 * P2_B3;
    const int nv1 = (int)imin64(16, I1 - i1o);
    if (i2b >= i2e) {  // empty i2 segment (the segment count does not divide the steps): zero partials, no staging
      for (int idx = tid; idx < 16 * R1; idx += TS_THREADS) a.W1p[(int64_t)pen * 16 * R1 + idx] = 0.0;
      for (int idx = tid; idx < 8 * R3; idx += TS_THREADS) a.W3p[(int64_t)pen * 8 * R3 + idx] = 0.0;
      continue;
    }
    __syncthreads();  // previous pencil fully done with shared memory
    auto issue_a3 = [&](int64_t i2o_) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(full_s, kBytesA3);
      bulk_load(A3s, a.At3 + ((int64_t)ib1 * a.n2b + i2o_ / P2_B2) * (RP * L::LD3), kBytesA3, full_s);
    };
    auto issue_a1 = [&](int64_t i2o_) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(full_s, kBytesA1);
      bulk_load(A1s, a.At1 + ((int64_t)ib3 * a.n2b + i2o_ / P2_B2) * (64 * L::LD1), kBytesA1, full_s);
    };
    auto issue_u2 = [&](int64_t i2o_) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(full_s, kBytesU2);
      bulk_load(U2s, a.U2t + (i2o_ / P2_B2) * (8 * L::LDU), kBytesU2, full_s);
    };
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(full_p, kBytesA2);
      bulk_load(A2s, a.At2 + ((int64_t)ib3 * a.n1b + ib1) * (RP * L::LD2), kBytesA2, full_p);
      issue_a3(i2b);
      issue_a1(i2b);
      issue_u2(i2b);
    }
    // pencil-resident UM_1 / UM_3 rows
    for (int idx = tid; idx < 16 * R1; idx += TS_THREADS) {
      const int l1 = idx & 15, r = idx >> 4;
      const bool v = l1 < nv1;
      cp_async8(U1s + l1 * L::LDU + r, v ? m1.UM + m1.ioff + i1o + l1 + m1.Ifull * r : m1.UM, v);
    }
    for (int idx = tid; idx < 8 * R3; idx += TS_THREADS) {
      const int l3 = idx & 7, r = idx >> 3;
      const bool v = i3o + l3 < I3;
      cp_async8(U3s + l3 * L::LDU + r, v ? m3.UM + m3.ioff + i3o + l3 + m3.Ifull * r : m3.UM, v);
    }
    cp_async_wait_all();
    __syncthreads();  // UM rows visible to both teams

    // team B, warp (mt, kh): Wt_3^T m-tile mt over K-half kh, and Wt_1^T (R_1 x 16 i1) m-tile mt over the
    // column half kh (two n-tiles of 8 i1)
    double w1acc[2][4] = {};
    double w3acc[4] = {0.0, 0.0, 0.0, 0.0};

    if (!teamB) {
      // =========================== team A ===========================
      for (int64_t i2o = i2b; i2o < i2e; i2o += P2_B2) {
        const bool more = i2o + P2_B2 < i2e;
        // this thread's 4 elements: (i1 = g, g+8) x (i2 = 2t, 2t+1) at i3 = w
        double tv[4], yv[3][4];
        bool inb[4];
        int64_t off[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t i1 = i1o + g + 8 * (q >> 1), i2 = i2o + 2 * t + (q & 1), i3 = i3o + w;
          inb[q] = i1 < I1 && i2 < I2 && i3 < I3;
          off[q] = i1 + I1 * i2 + S12 * i3;
          tv[q] = inb[q] ? (double)T[off[q]] : 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) yv[n][q] = inb[q] ? (double)Yp[n][off[q]] : 0.0;
        }
        TST(0);  // A0: pencil set-up / element-load issue
        mbar_wait(full_s, phs);  // this step's A_1, A_3, UM_2 slices
        phs ^= 1;
        if (i2o == i2b) {
          mbar_wait(full_p, php);  // the pencil's A_2 slice
          php ^= 1;
        }
        TST(1);  // A1: wait for the slices
        // ---- Z_1, Z_2 products ----
        double z1[4] = {0, 0, 0, 0}, z2[4] = {0, 0, 0, 0};
        {
          double y1[4] = {0, 0, 0, 0}, y2[4] = {0, 0, 0, 0};
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            if (ks >= ksz) break;
            const int k = 4 * ks + t;
            dmma((ks & 1) ? y1 : z1, U1s[g * L::LDU + k], U1s[(g + 8) * L::LDU + k], A1s[(g + 8 * w) * L::LD1 + k]);
            dmma((ks & 1) ? y2 : z2, A2s[k * L::LD2 + g + 16 * w], A2s[k * L::LD2 + g + 8 + 16 * w],
                 U2s[g * L::LDU + k]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            z1[q] += y1[q];
            z2[q] += y2[q];
          }
        }
        TST(2);  // A2: Z_1, Z_2
        bar_sync_n(BAR_Z3, TS_THREADS);  // Z_3 of this step is in Z3s; every team-A warp is done with UM_2
        TST(3);  // A3: wait for Z_3
        if (more && tid == 0) issue_u2(i2o + P2_B2);
        // ---- elementwise (reference op order, no FMA contraction) ----
        double* G2w = G2s + ((int)((i2o - i2b) >> 3) & 1) * (8 * 160);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int l1 = g + 8 * (q >> 1), l2 = 2 * t + (q & 1);
          const double zz[3] = {z1[q], z2[q], Z3s[zx(l1, l2, w)]};
          const double tt = tv[q];
          double zt[3], h = 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            zt[n] = __dsub_rn(tt, zz[n]);
            h = __dadd_rn(h, __dadd_rn(zt[n], __dmul_rn(yv[n][q], inv_mu)));  // pasd.cpp:202
          }
          const double e = soft(__dmul_rn(h, inv_n), tau);  // pasd.cpp:208
          double gn[3];
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            const double r = __dsub_rn(zt[n], e);                       // pasd.cpp:220
            const double ynew = __dadd_rn(yv[n][q], __dmul_rn(mu, r));  // pasd.cpp:221
            if (inb[q]) {
              const double ar = fabs(r);
              if (ar > worst[n]) worst[n] = ar;
              bad |= !isfinite(r);
              Yp[n][off[q]] = (EL)ynew;
            }
            gn[n] = inb[q] ? g_elem(tt, e, ynew, inv_mu_next) : 0.0;  // next G_n
            gsq[n] = fma(gn[n], gn[n], gsq[n]);
          }
          if (inb[q]) {
            Enew[off[q]] = (EL)e;
            Dp[off[q]] = (EL)__dsub_rn(tt, e);  // next pass 1 reads D = T - E
          }
          G1s[g1x(l1, l2, w)] = gn[0];
          G2w[g2x(l1, l2, w)] = gn[1];
          G3s[g3x(l1, l2, w)] = gn[2];
        }
        bar_arrive_n(BAR_G, TS_THREADS);  // G_1..3 of this step are in shared memory
        TST(4);  // A4: elementwise
      }
    } else {
      // =========================== team B ===========================
      double w2old[4], acc2[4];
      // Wt_2^T of the step at i2p (m-tile mt, K-half kh), K = (i1, i3); G_2 from buffer G2b
      auto wt2 = [&](int64_t i2p, const double* G2b) {
        if (mt < MT) {
          if (w2s || kh == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int r = 16 * mt + g + 8 * (q >> 1);
              const int64_t i2 = i2p + 2 * t + (q & 1);
              w2old[q] = (r < R2 && i2 < I2) ? W2k[i2 * R2 + r] : 0.0;
            }
          }
          double acc[3][4] = {};
          acc2[0] = acc2[1] = acc2[2] = acc2[3] = 0.0;
          const double* rowa = A2s + (16 * mt + g) * L::LD2 + 64 * kh;
          const double* rowb = rowa + 8 * L::LD2;
#pragma unroll
          for (int ks = 0; ks < 16; ++ks) {
            const int k = 64 * kh + 4 * ks + t;
            double(&c)[4] = (ks & 3) == 0 ? acc2 : acc[(ks & 3) - 1];
            dmma(c, rowa[4 * ks + t], rowb[4 * ks + t], G2b[g2x(k & 15, g, k >> 4)]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) acc2[q] += (acc[0][q] + acc[1][q]) + acc[2][q];
          if (!w2s) {
            if (kh == 1) {
#pragma unroll
              for (int q = 0; q < 4; ++q) X2s[(mt * 32 + lane) * 4 + q] = acc2[q];
            }
            bar_sync_n(1 + mt, 64);  // the two K-half warps of m-tile mt
          }
          if (w2s || kh == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int r = 16 * mt + g + 8 * (q >> 1);
              const int64_t i2 = i2p + 2 * t + (q & 1);
              const double v = w2s ? acc2[q] : (acc2[q] + X2s[(mt * 32 + lane) * 4 + q]);
              if (r < R2 && i2 < I2) W2k[i2 * R2 + r] = w2old[q] + v;
            }
          }
          // (the pair's next exchange comes after a BAR_G / block barrier that this read precedes)
        }
      };
      for (int64_t i2o = i2b; i2o < i2e; i2o += P2_B2) {
        const bool more = i2o + P2_B2 < i2e;
        const int gpar = (int)((i2o - i2b) >> 3) & 1;
        TST(5);  // B5: loop top / pencil set-up
        mbar_wait(full_s, phs);
        phs ^= 1;
        if (i2o == i2b) {
          mbar_wait(full_p, php);
          php ^= 1;
        }
        TST(6);  // B6: wait for the slices
        // ---- Z_3 products: (16 i1 x 8 i3) tile at i2 = w ----
        {
          double z3[4] = {0, 0, 0, 0}, y3[4] = {0, 0, 0, 0};
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            if (ks >= ksz) break;
            const int k = 4 * ks + t;
            dmma((ks & 1) ? y3 : z3, A3s[k * L::LD3 + g + 16 * w], A3s[k * L::LD3 + g + 8 + 16 * w],
                 U3s[g * L::LDU + k]);
          }
          Z3s[zx(g, w, 2 * t)] = z3[0] + y3[0];
          Z3s[zx(g, w, 2 * t + 1)] = z3[1] + y3[1];
          Z3s[zx(g + 8, w, 2 * t)] = z3[2] + y3[2];
          Z3s[zx(g + 8, w, 2 * t + 1)] = z3[3] + y3[3];
        }
        bar_arrive_n(BAR_Z3, TS_THREADS);
        TST(7);  // B7: Z_3
        // ---- Wt_2 of the previous step, while team A runs the elementwise phase ----
        if (i2o > i2b) wt2(i2o - P2_B2, G2s + (gpar ^ 1) * (8 * 160));
        TST(8);  // B8: Wt_2 of the previous step
        bar_sync_n(BAR_G, TS_THREADS);  // G_1..3 of this step
        TST(9);  // B9: wait for G
        auto release = [&](int* cnt, auto&& issue) {
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            const int old = atomicAdd(cnt, 1);
            if ((old & 7) == 7 && more) issue(i2o + P2_B2);
          }
        };
        // ---- Wt_3^T (m-tile mt, K-half kh), K = (i1, i2) ----
        if (mt < MT) {
          double acc[3][4] = {};
          const double* rowa = A3s + (16 * mt + g) * L::LD3 + 64 * kh;
          const double* rowb = rowa + 8 * L::LD3;
          const double* gcol = G3s + 180 * g;
#pragma unroll
          for (int ks = 0; ks < 16; ++ks) {
            const int k = 64 * kh + 4 * ks + t;
            double(&c)[4] = (ks & 3) == 0 ? w3acc : acc[(ks & 3) - 1];
            dmma(c, rowa[4 * ks + t], rowb[4 * ks + t], gcol[(k & 15) + 22 * (k >> 4)]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) w3acc[q] += (acc[0][q] + acc[1][q]) + acc[2][q];
        }
        release(rel3, issue_a3);
        TST(10);  // B10: Wt_3
        // ---- Wt_1^T (m-tile mt of r, column half kh): the A_1 slice as the A operand, G_1 as B ----
        // (rows r >= RP of the last m-tile read past their column: they feed output rows that are not stored)
        if (mt < MT) {
          double acc[2][4] = {};
          const double* cola = A1s + (32 * kh + t) * L::LD1 + 16 * mt + g;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int c = 32 * kh + 4 * ks + t;  // column (l2, l3) = (c & 7, c >> 3)
            const double a0 = cola[4 * ks * L::LD1], a1 = cola[4 * ks * L::LD1 + 8];
            dmma((ks & 1) ? acc[0] : w1acc[0], a0, a1, G1s[g1x(g, c & 7, c >> 3)]);
            dmma((ks & 1) ? acc[1] : w1acc[1], a0, a1, G1s[g1x(g + 8, c & 7, c >> 3)]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            w1acc[0][q] += acc[0][q];
            w1acc[1][q] += acc[1][q];
          }
        }
        release(rel1, issue_a1);
        TST(11);  // B11: Wt_1
      }
      {  // drain: Wt_2 of the pencil's last step
        const int64_t i2l = i2b + ((i2e - i2b - 1) / P2_B2) * P2_B2;
        wt2(i2l, G2s + ((int)((i2l - i2b) >> 3) & 1) * (8 * 160));
      }
    }
    // ---- end of pencil: combine the K-halves of Wt_3 and Wt_1, store the pencil's partials ----
    __syncthreads();
    double* xch = Z3s;  // 4 m-tiles x 32 lanes x 12 doubles (Z3s + G1s are free now)
    if (teamB && kh == 1 && mt < MT) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xch[(mt * 32 + lane) * 12 + q] = w3acc[q];
        xch[(mt * 32 + lane) * 12 + 4 + q] = w1acc[0][q];
        xch[(mt * 32 + lane) * 12 + 8 + q] = w1acc[1][q];
      }
    }
    __syncthreads();
    if (teamB && kh == 0 && mt < MT) {
      double* w3out = a.W3p + (int64_t)pen * 8 * R3;
      double* w1out = a.W1p + (int64_t)pen * 16 * R1;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = 16 * mt + g + 8 * (q >> 1), c = 2 * t + (q & 1);
        if (r < R3) w3out[c * R3 + r] = w3acc[q] + xch[(mt * 32 + lane) * 12 + q];
        if (r < R1) {
          w1out[c * R1 + r] = w1acc[0][q] + xch[(mt * 32 + lane) * 12 + 4 + q];
          w1out[(c + 8) * R1 + r] = w1acc[1][q] + xch[(mt * 32 + lane) * 12 + 8 + q];
        }
      }
    }
  }
#if PASD_P2_TIMING
  if (lane == 0 && w == 0)
    for (int k = 0; k < 12; ++k) atomicAdd(&g_p2_phase[k], ph_acc[k]);
#endif
  // ---- per-CTA residual / NaN / ||G||^2 partials (team B contributes identities) ----
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
  __syncthreads();
  if (a.finish_ticket && last_cta(a.finish_ticket, reinterpret_cast<int*>(red + 48)))
    finish_body(const_cast<Ctl*>(ctl), a.resid_part, a.bad_part, gridDim.x, a.history, nullptr, red);
}

template <int RP>
void ts_setup_rp() {
  if constexpr (ts_fits<RP>()) {
    cudaFuncSetAttribute(k_pass2_ts<RP, double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)P2TsLayout<RP>::bytes);
    cudaFuncSetAttribute(k_pass2_ts<RP, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)P2TsLayout<RP>::bytes);
  }
}
template <int RP>
void ts_launch_rp(bool f32, const Pass2Args& a, const Ctl* ctl, int grid, cudaStream_t st) {
  if constexpr (ts_fits<RP>()) {
    if (f32)
      k_pass2_ts<RP, float><<<grid, TS_THREADS, P2TsLayout<RP>::bytes, st>>>(a, ctl);
    else
      k_pass2_ts<RP, double><<<grid, TS_THREADS, P2TsLayout<RP>::bytes, st>>>(a, ctl);
  }
}
// padded ranks k_pass2_ts serves (those the 16 x 8 x 8 kernel serves by default and that fit in 227 KB)
inline bool ts_supported(int rp) { return rp >= 32 && rp <= 56; }
inline void ts_setup(int rp) {
  switch (rp) {
    case 32: ts_setup_rp<32>(); break;
    case 40: ts_setup_rp<40>(); break;
    case 48: ts_setup_rp<48>(); break;
    case 56: ts_setup_rp<56>(); break;
    default: break;
  }
}
inline void ts_launch(int rp, bool f32, const Pass2Args& a, const Ctl* ctl, int grid, cudaStream_t st) {
  switch (rp) {
    case 32: ts_launch_rp<32>(f32, a, ctl, grid, st); break;
    case 40: ts_launch_rp<40>(f32, a, ctl, grid, st); break;
    case 48: ts_launch_rp<48>(f32, a, ctl, grid, st); break;
    case 56: ts_launch_rp<56>(f32, a, ctl, grid, st); break;
    default: break;
  }
}

}  // namespace pasd
