// pasd_pass1.cuh — pass 1 of a PASD iteration on the FP64 tensor cores:
//   A_n = U_n^T G_(n),  G_n = (T - E) + Y_n / mu          (proj/src/pasd.cpp:77,178-186)
// reading D = T - E (kept resident by the update pass, same rounded value) and Y_n.
// for one mode n, directly on the strided tensor (no unfolding copy,
// tensor.cpp:98-113).  As a GEMM: A (J x R) = G (J x I) * U (I x R), with
// kappa = unfolding column, K = I_n, N = R_n <= 64.
//
// Persistent CTAs (two per SM, 8 warps each) walk tiles of 128 columns kappa;
// K runs over i in chunks of PASD_P1_KCC.  The D and Y_n chunks and the U chunk
// stream into a PASD_P1_NSTC-deep cp.async ring in shared memory (16-byte
// copies along the contiguous index) while the DMMAs of the current chunk run,
// and one CTA's DMMAs overlap the other's loads.  G = D + Y_n / mu is formed
// inside the DMMA A-fragment load (each G value feeds exactly one fragment);
// warp w owns kappa rows 16w..16w+15 and all RP/8 n-tiles.
// A tile is 128 consecutive p at fixed q (every staged row one contiguous run),
// or, where that wastes a mostly empty p-block per q, 128 consecutive unfolding
// columns spanning two q (p1_cross).
#pragma once
#include "pasd_pass2.cuh"

namespace pasd {

// 128 columns x 16 i per chunk, double-buffered, two CTAs per SM: one CTA's
// DMMAs overlap the other's loads.  Warp w owns kappa rows 16w..16w+15 and
// all n-tiles, so every G value is formed once.
// (64-column tiles at 4 CTAs per SM measured slower: 13.5-14.1 vs 12.6 ms per C5 iteration.)
#ifndef PASD_P1_MT
#define PASD_P1_MT 128
#endif
#ifndef PASD_P1_CTAS
#define PASD_P1_CTAS 2
#endif
constexpr int P1_MT = PASD_P1_MT;           // kappa columns per tile (16 per warp)
constexpr int P1_THREADS = 2 * P1_MT;       // one warp per 16-column m-tile
constexpr int P1_CTAS = PASD_P1_CTAS;       // resident CTAs per SM
#ifndef PASD_P1_KCC
#define PASD_P1_KCC 8
#endif
#ifndef PASD_P1_NSTC
#define PASD_P1_NSTC 3
#endif
#ifndef PASD_P1_KCS
#define PASD_P1_KCS 8
#endif
#ifndef PASD_P1_NSTS
#define PASD_P1_NSTS 4
#endif
// chunk depth (i rows) and pipeline stages at two CTAs per SM.  Mode 1
// (CONTIG) stages KC consecutive i per column, the strided modes 1 KB rows of
// 128 kappa.  Measured at C5 (KC/NST): strided 16/2 -> 8/4 takes each strided
// mode from 4.7 to 4.2 ms (8/3, 8/5 in between; 4/6, 4/8 slower); mode 1
// 16/2 -> 8/3 saves 0.4 ms (8/4 no longer fits two CTAs per SM).
template <bool CONTIG>
struct P1Cfg {
  static constexpr int KC = CONTIG ? PASD_P1_KCC : PASD_P1_KCS;
  static constexpr int NST = CONTIG ? PASD_P1_NSTC : PASD_P1_NSTS;
};

template <int RP, bool CONTIG, class EL = double>
struct P1Layout {
  // CONTIG (mode 1): raw[kappa][i] rows of 16 i;  else raw[i][kappa] rows of 128 kappa.
  // Pitches are 4 mod 16 doubles (float storage: 12 / 136 floats): the fragment
  // reads (row g, col t) hit distinct banks per half-warp.
  static constexpr int KC = P1Cfg<CONTIG>::KC, NST = P1Cfg<CONTIG>::NST;
  static constexpr int ES = sizeof(EL);
  static constexpr int LDR = CONTIG ? (KC + 4) : (P1_MT + (ES == 8 ? 4 : 8));
  static constexpr int RAW = CONTIG ? P1_MT * LDR : KC * LDR;  // elements per tensor per stage
  static constexpr int LDU = KC + 4;                           // U chunk (float64) as [r][i]
  static constexpr int USZ = RP * LDU;
  static constexpr int UOFF = 2 * RAW * ES;                    // byte offset of the U chunk
  static constexpr int STAGE = UOFF + 8 * USZ;                 // bytes: D, Y_n, U chunk
  static_assert(UOFF % 16 == 0 && STAGE % 16 == 0, "16-byte aligned stages");
  static constexpr size_t bytes = (size_t)NST * STAGE;
};

// Pair of consecutive elements (16 bytes of float64, 8 of float32): one cp.async.
template <class EL>
__device__ __forceinline__ void cp_pair(unsigned s, const void* g, bool ok) {
  if constexpr (sizeof(EL) == 8)
    cp16z(s, g, ok);
  else
    cp8z(s, g, ok);
}
// One element (ok = false: zero fill).
template <class EL>
__device__ __forceinline__ void cp_one(unsigned s, const void* g, bool ok) {
  if constexpr (sizeof(EL) == 8) {
    cp8s(s, g, ok ? 8 : 0);
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(g), "r"(ok ? 4 : 0) : "memory");
  }
}

// Strided modes whose inner extent leaves a mostly empty last 128-wide p-block
// per q (> 5% of the tiles' width wasted: C1-C3, inner = 100, 200, 400) use
// "crossing" tiles instead: 128 consecutive unfolding columns kappa = p + inner q
// that may span two q.  (Measured: crossing tiles everywhere cost 7% at C5,
// inner = 1000, so the q-aligned p-blocks stay where their waste is small.)
__host__ __device__ inline bool p1_cross(int64_t inner) {
  const int64_t pb = (inner + P1_MT - 1) / P1_MT;
  return inner > 1 && (pb * P1_MT - inner) * 20 > pb * P1_MT;
}
__host__ __device__ inline int64_t p1_ntiles(const ModeDev& m) {
  if (m.inner == 1 || p1_cross(m.inner)) return (m.J + P1_MT - 1) / P1_MT;
  return ((m.inner + P1_MT - 1) / P1_MT) * m.outer;
}

// Work-item cursor: (tile, chunk) advanced without 64-bit divisions.  For
// strided modes a tile is (q, p-block); `p0` / `q` track it incrementally.
struct P1Cursor {
  int64_t tile, q, pb;  // tile index, outer index, p-block
  int chunk;
};

// EL: storage type of D and Y_n (float in the fp32 mode); G is formed in fp64.
template <int RP, bool CONTIG, bool CROSS = false, class EL = double>
__global__ void __launch_bounds__(P1_THREADS, P1_CTAS) k_pass1(ModeDev m, const EL* __restrict__ D,
                                                        const EL* __restrict__ Y, const Ctl* ctl) {
  if (ctl->done) return;
  using L = P1Layout<RP, CONTIG, EL>;
  constexpr unsigned ES = sizeof(EL);
  constexpr int NT = RP / 8;  // n-tiles per warp
  constexpr int P1_KC = L::KC, P1_NST = L::NST;
  extern __shared__ double p1sm[];
  const double inv_mu = __ddiv_rn(1.0, ctl->mu);  // pasd.cpp:170
  const int tid = threadIdx.x, lane = tid & 31, g = lane >> 2, t = lane & 3, w = tid >> 5;
  const int64_t I = m.I, inner = m.inner;
  const int R = m.R;
  const int64_t pblocks = CONTIG ? 1 : (inner + P1_MT - 1) / P1_MT;
  constexpr bool cross = !CONTIG && CROSS;  // compile-time: the q-aligned kernels carry no trace of it
  const int64_t ntiles = (CONTIG || cross) ? (m.J + P1_MT - 1) / P1_MT : pblocks * m.outer;
  const int nchunk = (int)((I + P1_KC - 1) / P1_KC);
  const bool al = CONTIG ? (I % 2 == 0) : (inner % 2 == 0);        // 16-byte aligned tensor rows
  const bool alu = (m.Ifull % 2 == 0) && (m.ioff % 2 == 0);         // 16-byte aligned U columns
  const int64_t gq = gridDim.x / pblocks, gpb = gridDim.x % pblocks;  // tile stride as (q, p-block)
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(p1sm));

  auto advance = [&](P1Cursor& c) {
    if (++c.chunk == nchunk) {
      c.chunk = 0;
      c.tile += gridDim.x;
      if (!CONTIG) {
        c.q += gq;
        c.pb += gpb;
        if (c.pb >= pblocks) {
          c.pb -= pblocks;
          ++c.q;
        }
      }
    }
  };
  // issue the cp.async copies of the work item at cursor c into stage s
  auto issue = [&](const P1Cursor& c, int s) {
    if (c.tile >= ntiles) return;
    const int64_t i0 = (int64_t)c.chunk * P1_KC;
    const unsigned st = sbase + (unsigned)(s * L::STAGE);
    const int ni = (int)imin64(P1_KC, I - i0);
    if (CONTIG) {
      // 128 columns kappa, 16 consecutive i each (contiguous): row = column
      const int64_t k0 = c.tile * P1_MT;
      if (al) {
        constexpr int CPR = P1_KC / 2, RPP = P1_THREADS / CPR;  // 16-byte chunks per row, rows per pass
        const int cc = tid % CPR;  // 16-byte chunk of the KC-double row
        const int v = ni - 2 * cc, nbc = v >= 2 ? 16 : (v == 1 ? 8 : 0);
        const int j0 = tid / CPR;
        const int64_t off0 = (k0 + j0) * I + i0 + 2 * cc;
#pragma unroll
        for (int k = 0; k < P1_MT / RPP; ++k) {
          const int j = j0 + RPP * k;
          const int nb = (k0 + j < m.J) ? nbc : 0;
          const int64_t off = off0 + (int64_t)RPP * k * I;
          const unsigned d = st + ES * (unsigned)(j * L::LDR + 2 * cc);
          cp_pair<EL>(d, nb ? D + off : D, nb != 0);  // even I: chunks wholly in or out
          cp_pair<EL>(d + ES * L::RAW, nb ? Y + off : D, nb != 0);
        }
      } else {
        for (int idx = tid; idx < P1_MT * P1_KC; idx += P1_THREADS) {
          const int j = idx / P1_KC, cc = idx % P1_KC;
          const bool ok = k0 + j < m.J && cc < ni;
          const int64_t off = (k0 + j) * I + i0 + cc;
          const unsigned d = st + ES * (unsigned)(j * L::LDR + cc);
          cp_one<EL>(d, ok ? D + off : D, ok);
          cp_one<EL>(d + ES * L::RAW, ok ? Y + off : D, ok);
        }
      }
    } else if (cross) {
      // crossing tile: each column chunk locates its own (p, q)
      if (al) {
        constexpr int CPR = P1_MT / 2, RG = P1_THREADS / CPR;
        const int cc = tid % CPR, rsub = tid / CPR;
        const int64_t kap = c.tile * P1_MT + 2 * cc;
        const bool cok = kap < m.J;
        const int64_t q = kap / inner;
        const int64_t off0 = (kap - q * inner) + inner * (i0 + I * q);
#pragma unroll
        for (int k = 0; k < P1_KC / RG; ++k) {
          const int ii = rsub + RG * k;
          const bool ok = cok && ii < ni;  // even inner: a 16-byte chunk never straddles q
          const int64_t off = off0 + inner * ii;
          const unsigned d = st + ES * (unsigned)(ii * L::LDR + 2 * cc);
          cp_pair<EL>(d, ok ? D + off : D, ok);
          cp_pair<EL>(d + ES * L::RAW, ok ? Y + off : D, ok);
        }
      } else {
        for (int idx = tid; idx < P1_KC * P1_MT; idx += P1_THREADS) {
          const int ii = idx / P1_MT, cc = idx % P1_MT;
          const int64_t kap = c.tile * P1_MT + cc;
          const bool ok = ii < ni && kap < m.J;
          const int64_t q = kap / inner;
          const int64_t off = (kap - q * inner) + inner * (i0 + ii + I * q);
          const unsigned d = st + ES * (unsigned)(ii * L::LDR + cc);
          cp_one<EL>(d, ok ? D + off : D, ok);
          cp_one<EL>(d + ES * L::RAW, ok ? Y + off : D, ok);
        }
      }
    } else {
      const int64_t p0 = c.pb * P1_MT;
      const int np = (int)imin64(P1_MT, inner - p0);
      const int64_t off0 = p0 + inner * (i0 + I * c.q);
      if (al) {
        // MT/2 16-byte chunks per row; thread -> (chunk cc, rows rsub + RG k)
        constexpr int CPR = P1_MT / 2, RG = P1_THREADS / CPR;
        const int cc = tid % CPR, rsub = tid / CPR;
        const int v = np - 2 * cc, nbc = v >= 2 ? 16 : (v == 1 ? 8 : 0);
#pragma unroll
        for (int k = 0; k < P1_KC / RG; ++k) {
          const int ii = rsub + RG * k;
          const int nb = ii < ni ? nbc : 0;
          const int64_t off = off0 + inner * ii + 2 * cc;
          const unsigned d = st + ES * (unsigned)(ii * L::LDR + 2 * cc);
          cp_pair<EL>(d, nb ? D + off : D, nb != 0);  // even inner: chunks wholly in or out
          cp_pair<EL>(d + ES * L::RAW, nb ? Y + off : D, nb != 0);
        }
      } else {
        for (int idx = tid; idx < P1_KC * P1_MT; idx += P1_THREADS) {
          const int ii = idx / P1_MT, cc = idx % P1_MT;
          const bool ok = ii < ni && cc < np;
          const int64_t off = off0 + inner * ii + cc;
          const unsigned d = st + ES * (unsigned)(ii * L::LDR + cc);
          cp_one<EL>(d, ok ? D + off : D, ok);
          cp_one<EL>(d + ES * L::RAW, ok ? Y + off : D, ok);
        }
      }
    }
    // U chunk as [r][i] (16 consecutive i of column r are contiguous in U)
    const unsigned us = st + (unsigned)L::UOFF;
    const double* ub = m.U + m.ioff + i0;
    if (alu) {
      constexpr int PAIRS = P1_KC / 2, RSTEP = P1_THREADS / PAIRS;
      const int ip = tid % PAIRS;
      const int v = ni - 2 * ip, nbc = v >= 2 ? 16 : (v == 1 ? 8 : 0);
#pragma unroll
      for (int k = 0; k < (RP + RSTEP - 1) / RSTEP; ++k) {
        const int r = tid / PAIRS + RSTEP * k;
        if (r < RP) {
          const int nb = r < R ? nbc : 0;
          cp16s(us + 8u * (unsigned)(r * L::LDU + 2 * ip), nb ? ub + 2 * ip + m.Ifull * r : m.U, nb);
        }
      }
    } else {
      for (int idx = tid; idx < P1_KC * RP; idx += P1_THREADS) {
        const int i = idx & (P1_KC - 1), r = idx / P1_KC;
        const bool ok = r < R && i < ni;
        cp8s(us + 8u * (unsigned)(r * L::LDU + i), ok ? ub + i + m.Ifull * r : m.U, ok ? 8 : 0);
      }
    }
  };

  // few n-tiles: even / odd k-steps in separate accumulators (independent chains)
  constexpr bool TWO = NT < 4;
  double acc[NT][4], acb[TWO ? NT : 1][4];
  P1Cursor cur{(int64_t)blockIdx.x, (int64_t)blockIdx.x / pblocks, (int64_t)blockIdx.x % pblocks, 0};
  P1Cursor nxt = cur;
  for (int s = 0; s < P1_NST - 1; ++s) {
    issue(nxt, s);
    advance(nxt);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t it = 0; cur.tile < ntiles; ++it) {
    const int s = (int)(it % P1_NST);
    if (cur.chunk == 0) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
        if (TWO) acb[TWO ? j : 0][0] = acb[TWO ? j : 0][1] = acb[TWO ? j : 0][2] = acb[TWO ? j : 0][3] = 0.0;
      }
    }
    asm volatile("cp.async.wait_group %0;" ::"n"(P1_NST - 2) : "memory");
    __syncthreads();  // stage s complete for all threads; stage of item it-1 free
    issue(nxt, (int)((it + P1_NST - 1) % P1_NST));
    advance(nxt);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const char* st = reinterpret_cast<const char*>(p1sm) + (size_t)s * L::STAGE;
    const EL* Ds = reinterpret_cast<const EL*>(st);
    const EL* Ys = Ds + L::RAW;
    const double* Us = reinterpret_cast<const double*>(st + L::UOFF);
#pragma unroll
    for (int ks = 0; ks < P1_KC / 4; ++ks) {
      const int k = 4 * ks + t;
      const int r0 = 16 * w + g, r1 = r0 + 8;
      const int o0 = CONTIG ? r0 * L::LDR + k : k * L::LDR + r0;
      const int o1 = CONTIG ? r1 * L::LDR + k : k * L::LDR + r1;
      const double a0 = __dadd_rn((double)Ds[o0], __dmul_rn((double)Ys[o0], inv_mu));  // g_elem on D
      const double a1 = __dadd_rn((double)Ds[o1], __dmul_rn((double)Ys[o1], inv_mu));
#pragma unroll
      for (int j = 0; j < NT; ++j)
        dmma((TWO && (ks & 1)) ? acb[TWO ? j : 0] : acc[j], a0, a1, Us[(8 * j + g) * L::LDU + k]);
    }
    if (cur.chunk == nchunk - 1) {  // tile done: write A
      if (TWO) {
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) acc[j][q4] += acb[TWO ? j : 0][q4];
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int row = 16 * w + g + 8 * (q4 >> 1);
          const int r = 8 * j + 2 * t + (q4 & 1);
          if (r >= R) continue;
          if (CONTIG) {
            const int64_t kap = cur.tile * P1_MT + row;
            if (kap < m.J) m.A[r + (int64_t)R * kap] = acc[j][q4];
          } else if (cross) {
            const int64_t kap = cur.tile * P1_MT + row;
            if (kap < m.J) {
              const int64_t q = kap / inner;
              m.A[(kap - q * inner) + inner * ((int64_t)r + (int64_t)R * q)] = acc[j][q4];
            }
          } else {
            const int64_t p = cur.pb * P1_MT + row;
            if (p < inner) m.A[p + inner * ((int64_t)r + (int64_t)R * cur.q)] = acc[j][q4];
          }
        }
      }
    }
    advance(cur);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int RP, bool CONTIG, bool CROSS, class EL>
void launch_p1(const ModeDev& m, const EL* D, const EL* Y, const Ctl* ctl, int grid, cudaStream_t st) {
  using L = P1Layout<RP, CONTIG, EL>;
  ensure_smem_attr<k_pass1<RP, CONTIG, CROSS, EL>>(L::bytes);
  k_pass1<RP, CONTIG, CROSS, EL><<<grid, P1_THREADS, L::bytes, st>>>(m, D, Y, ctl);
}

template <bool CONTIG, bool CROSS, class EL>
void launch_p1_rp(const ModeDev& m, const EL* D, const EL* Y, const Ctl* ctl, int grid, cudaStream_t st) {
  switch ((m.R + 7) / 8 * 8) {
    case 8: launch_p1<8, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
    case 16: launch_p1<16, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
    case 24: launch_p1<24, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
    case 32: launch_p1<32, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
    case 40: launch_p1<40, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
    case 48: launch_p1<48, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
    case 56: launch_p1<56, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
    default: launch_p1<64, CONTIG, CROSS>(m, D, Y, ctl, grid, st); break;
  }
}

inline int pass1_grid(const ModeDev& m, int sms) {
  return (int)imin64(p1_ntiles(m), P1_CTAS * sms);
}

template <class EL>
void launch_contract_A_mma(const ModeDev& m, const EL* D, const EL* Y, const Ctl* ctl, int sms, cudaStream_t st) {
  const int grid = pass1_grid(m, sms);
  if (m.inner == 1)
    launch_p1_rp<true, false>(m, D, Y, ctl, grid, st);
  else if (p1_cross(m.inner))
    launch_p1_rp<false, true>(m, D, Y, ctl, grid, st);
  else
    launch_p1_rp<false, false>(m, D, Y, ctl, grid, st);
}

}  // namespace pasd
