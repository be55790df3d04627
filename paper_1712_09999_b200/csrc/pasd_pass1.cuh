// pasd_pass1.cuh — pass 1 of a PASD iteration on the FP64 tensor cores:
//   A_n = U_n^T G_(n),  G_n = (T - E) + Y_n / mu          (proj/src/pasd.cpp:77,178-186)
// reading D = T - E (kept resident by the update pass, same rounded value) and Y_n.
// for one mode n, directly on the strided tensor (no unfolding copy,
// tensor.cpp:98-113).  As a GEMM: A (J x R) = G (J x I) * U (I x R), with
// kappa = unfolding column, K = I_n, N = R_n <= 64.
//
// Persistent CTAs (one per SM, 8 warps) walk tiles of 128 columns kappa; K runs
// over i in chunks of 16.  Raw T, E, Y_n chunks and the U chunk stream into a
// 3-stage cp.async ring in shared memory (16-byte copies along the contiguous
// index), so ~150 KB per SM is in flight while the DMMAs of the current chunk
// run.  G is formed inside the DMMA A-fragment load (each G value feeds exactly
// one fragment), warp w owns kappa rows 16w..16w+15 and all RP/8 n-tiles.
// Tiles never cross an outer index q (for modes with inner > 1 a tile is 128
// consecutive p at fixed q), so every staged row is one contiguous run.
#pragma once
#include "pasd_pass2.cuh"

namespace pasd {

// 64 columns x 16 i per chunk, double-buffered, two CTAs per SM: one CTA's
// DMMAs overlap the other's loads (a single CTA serialised them: measured
// 4.6 ms compute-only + 4.6 ms load-only -> 7.6 ms combined per C5 mode).
#ifndef PASD_P1_MT
#define PASD_P1_MT 128
#endif
constexpr int P1_MT = PASD_P1_MT;  // kappa columns per tile
#ifndef PASD_P1_KC
#define PASD_P1_KC 16
#endif
constexpr int P1_KC = PASD_P1_KC;  // i rows per chunk
#ifndef PASD_P1_NST
#define PASD_P1_NST 2
#endif
constexpr int P1_NST = PASD_P1_NST;  // pipeline stages
constexpr int P1_THREADS = 256;

template <int RP, bool CONTIG>
struct P1Layout {
  // CONTIG (mode 1): raw[kappa][i] rows of 16 i;  else raw[i][kappa] rows of 128 kappa.
  static constexpr int LDR = CONTIG ? (P1_KC + 4) : (P1_MT + 4);
  static constexpr int RAW = CONTIG ? P1_MT * LDR : P1_KC * LDR;  // doubles per tensor per stage
  static constexpr int LDU = RP + 4;
  static constexpr int USZ = P1_KC * LDU;
  static constexpr int STAGE = 2 * RAW + USZ;  // D, Y_n, U chunk
  static constexpr size_t bytes = sizeof(double) * (size_t)P1_NST * STAGE;
};

template <int RP, bool CONTIG>
__global__ void __launch_bounds__(P1_THREADS, 2) k_pass1(ModeDev m, const double* __restrict__ D,
                                                        const double* __restrict__ Y, const Ctl* ctl) {
  if (ctl->done) return;
  using L = P1Layout<RP, CONTIG>;
  constexpr int MTILES = P1_MT / 16;                 // m16 tiles of kappa rows (4)
  constexpr int NSPLIT = (P1_THREADS / 32) / MTILES;  // warps sharing an m-tile (2): split the n-tiles
  constexpr int NTALL = RP / 8;
  constexpr int NT = (NTALL + NSPLIT - 1) / NSPLIT;  // n-tiles per warp
  extern __shared__ double p1sm[];
  const double inv_mu = __ddiv_rn(1.0, ctl->mu);  // pasd.cpp:170
  const int tid = threadIdx.x, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int w = (tid >> 5) % MTILES, jbase = ((tid >> 5) / MTILES) * NT;  // m-tile, first n-tile
  const int64_t I = m.I, inner = m.inner;
  const int R = m.R;
  // tiles: CONTIG -> 128 consecutive kappa; else (q, p-block of 128)
  const int64_t pblocks = CONTIG ? 1 : (inner + P1_MT - 1) / P1_MT;
  const int64_t ntiles = CONTIG ? (m.J + P1_MT - 1) / P1_MT : pblocks * m.outer;
  const int nchunk = (int)((I + P1_KC - 1) / P1_KC);
  const bool al = CONTIG ? (I % 2 == 0) : (inner % 2 == 0);  // 16-byte aligned rows
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * nchunk;  // (tile, chunk) work items of this CTA

  auto stage_ptr = [&](int s) { return p1sm + (size_t)s * L::STAGE; };
  // issue the cp.async copies of work item `it` into stage s
  auto issue = [&](int64_t it, int s) {
    if (it >= total) return;
    const int64_t tile = blockIdx.x + (it / nchunk) * gridDim.x;
    const int64_t i0 = (it % nchunk) * P1_KC;
    double* st = stage_ptr(s);
    if (CONTIG) {
      // 128 columns kappa, 16 consecutive i each (contiguous): row = column
      const int64_t k0 = tile * P1_MT;
      const int ni = (int)imin64(P1_KC, I - i0);
      if (al) {
        const int c = tid & 7;  // 16-byte chunk of the 16-double row
        const int v = ni - 2 * c, nbc = v >= 2 ? 16 : (v == 1 ? 8 : 0);
#pragma unroll
        for (int k = 0; k < P1_MT / (P1_THREADS / 8); ++k) {
          const int j = (tid >> 3) + (P1_THREADS / 8) * k;
          const int64_t kap = k0 + j;
          const int nb = kap < m.J ? nbc : 0;
          const int64_t off = kap * I + i0 + 2 * c;
          const int d = j * L::LDR + 2 * c;
          cp_async16(st + d, nb ? D + off : D, nb);
          cp_async16(st + L::RAW + d, nb ? Y + off : D, nb);
        }
      } else {
        for (int idx = tid; idx < P1_MT * P1_KC; idx += P1_THREADS) {
          const int j = idx / P1_KC, c = idx % P1_KC;
          const int64_t kap = k0 + j;
          const bool ok = kap < m.J && c < ni;
          const int64_t off = kap * I + i0 + c;
          const int d = j * L::LDR + c;
          cp_async8(st + d, ok ? D + off : D, ok);
          cp_async8(st + L::RAW + d, ok ? Y + off : D, ok);
        }
      }
    } else {
      const int64_t q = tile / pblocks, p0 = (tile % pblocks) * P1_MT;
      const int np = (int)imin64(P1_MT, inner - p0);
      const int ni = (int)imin64(P1_KC, I - i0);
      const int64_t off0 = p0 + inner * (i0 + I * q);
      if (al) {
        // P1_MT/2 16-byte chunks per row; thread -> (chunk c, rows rsub + RG k)
        constexpr int CPR = P1_MT / 2, RG = P1_THREADS / CPR;
        const int c = tid % CPR, rsub = tid / CPR;
        const int v = np - 2 * c, nbc = v >= 2 ? 16 : (v == 1 ? 8 : 0);
#pragma unroll
        for (int k = 0; k < P1_KC / RG; ++k) {
          const int ii = rsub + RG * k;
          const int nb = ii < ni ? nbc : 0;
          const int64_t off = off0 + inner * ii + 2 * c;
          const int d = ii * L::LDR + 2 * c;
          cp_async16(st + d, nb ? D + off : D, nb);
          cp_async16(st + L::RAW + d, nb ? Y + off : D, nb);
        }
      } else {
        for (int idx = tid; idx < P1_KC * P1_MT; idx += P1_THREADS) {
          const int ii = idx / P1_MT, c = idx % P1_MT;
          const bool ok = ii < ni && c < np;
          const int64_t off = off0 + inner * ii + c;
          const int d = ii * L::LDR + c;
          cp_async8(st + d, ok ? D + off : D, ok);
          cp_async8(st + L::RAW + d, ok ? Y + off : D, ok);
        }
      }
    }
    double* us = st + 2 * L::RAW;
    for (int idx = tid; idx < P1_KC * RP; idx += P1_THREADS) {
      const int i = idx % P1_KC, r = idx / P1_KC;
      const bool ok = r < R && i0 + i < I;
      cp_async8(us + i * L::LDU + r, ok ? m.U + m.ioff + (i0 + i) + m.Ifull * r : m.U, ok);
    }
  };

  // even / odd k-steps in separate accumulators (two independent DMMA chains
  // per n-tile) only when a warp has few n-tiles; NT >= 4 chains already keep
  // the tensor pipe busy and the registers are needed by the staging.
  constexpr bool TWO = NT < 4;
  double acc[NT][4], acb[TWO ? NT : 1][4];
  int64_t it = 0;
  for (int s = 0; s < P1_NST - 1; ++s) {
    issue(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (; it < total; ++it) {
    const int s = (int)(it % P1_NST);
    const int ci = (int)(it % nchunk);
    if (ci == 0) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
        if (TWO) acb[TWO ? j : 0][0] = acb[TWO ? j : 0][1] = acb[TWO ? j : 0][2] = acb[TWO ? j : 0][3] = 0.0;
      }
    }
    asm volatile("cp.async.wait_group %0;" ::"n"(P1_NST - 2) : "memory");
    __syncthreads();  // stage s complete for all threads; stage of item it-1 free
    issue(it + P1_NST - 1, (int)((it + P1_NST - 1) % P1_NST));
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* st = stage_ptr(s);
    const double* Ds = st;
    const double* Ys = st + L::RAW;
    const double* Us = st + 2 * L::RAW;
#pragma unroll
    for (int ks = 0; ks < P1_KC / 4; ++ks) {
      const int k = 4 * ks + t;
      const int r0 = 16 * w + g, r1 = r0 + 8;
      const int o0 = CONTIG ? r0 * L::LDR + k : k * L::LDR + r0;
      const int o1 = CONTIG ? r1 * L::LDR + k : k * L::LDR + r1;
      const double a0 = __dadd_rn(Ds[o0], __dmul_rn(Ys[o0], inv_mu));  // g_elem on D
      const double a1 = __dadd_rn(Ds[o1], __dmul_rn(Ys[o1], inv_mu));
#pragma unroll
      for (int j = 0; j < NT; ++j)
        if (jbase + j < NTALL) dmma((TWO && (ks & 1)) ? acb[TWO ? j : 0] : acc[j], a0, a1, Us[k * L::LDU + 8 * (jbase + j) + g]);
    }
    if (ci == nchunk - 1) {  // tile done: write A
      const int64_t tile = blockIdx.x + (it / nchunk) * gridDim.x;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          if (TWO) acc[j][q4] += acb[TWO ? j : 0][q4];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int row = 16 * w + g + 8 * (q4 >> 1);
          const int r = 8 * (jbase + j) + 2 * t + (q4 & 1);
          if (r >= R) continue;
          if (CONTIG) {
            const int64_t kap = tile * P1_MT + row;
            if (kap < m.J) m.A[r + (int64_t)R * kap] = acc[j][q4];
          } else {
            const int64_t q = tile / pblocks, p = (tile % pblocks) * P1_MT + row;
            if (p < inner) m.A[p + inner * ((int64_t)r + (int64_t)R * q)] = acc[j][q4];
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int RP, bool CONTIG>
void launch_p1(const ModeDev& m, const double* D, const double* Y, const Ctl* ctl,
               int grid, cudaStream_t st) {
  using L = P1Layout<RP, CONTIG>;
  static bool attr = false;  // idempotent attribute set
  if (!attr) {
    cudaFuncSetAttribute(k_pass1<RP, CONTIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes);
    attr = true;
  }
  k_pass1<RP, CONTIG><<<grid, P1_THREADS, L::bytes, st>>>(m, D, Y, ctl);
}

template <bool CONTIG>
void launch_p1_rp(const ModeDev& m, const double* D, const double* Y,
                  const Ctl* ctl, int grid, cudaStream_t st) {
  switch ((m.R + 7) / 8 * 8) {
    case 8: launch_p1<8, CONTIG>(m, D, Y, ctl, grid, st); break;
    case 16: launch_p1<16, CONTIG>(m, D, Y, ctl, grid, st); break;
    case 24: launch_p1<24, CONTIG>(m, D, Y, ctl, grid, st); break;
    case 32: launch_p1<32, CONTIG>(m, D, Y, ctl, grid, st); break;
    case 40: launch_p1<40, CONTIG>(m, D, Y, ctl, grid, st); break;
    case 48: launch_p1<48, CONTIG>(m, D, Y, ctl, grid, st); break;
    case 56: launch_p1<56, CONTIG>(m, D, Y, ctl, grid, st); break;
    default: launch_p1<64, CONTIG>(m, D, Y, ctl, grid, st); break;
  }
}

inline int pass1_grid(const ModeDev& m, int sms) {
  const int64_t ntiles =
      m.inner == 1 ? (m.J + P1_MT - 1) / P1_MT : ((m.inner + P1_MT - 1) / P1_MT) * m.outer;
  return (int)imin64(ntiles, 2 * sms);
}

inline void launch_contract_A_mma(const ModeDev& m, const double* D, const double* Y, const Ctl* ctl, int sms, cudaStream_t st) {
  const int grid = pass1_grid(m, sms);
  if (m.inner == 1)
    launch_p1_rp<true>(m, D, Y, ctl, grid, st);
  else
    launch_p1_rp<false>(m, D, Y, ctl, grid, st);
}

}  // namespace pasd
