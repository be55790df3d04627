// pasd_pass1.cuh — pass 1 of a PASD iteration on the FP64 tensor cores:
//   A_n = U_n^T G_(n),  G_n = (T - E) + Y_n / mu          (proj/src/pasd.cpp:77,178-186)
// for one mode n, directly on the strided tensor (no unfolding copy,
// tensor.cpp:98-113).  As a GEMM: A (J x R) = G (J x I) * U (I x R), with
// kappa = unfolding column (J, large), K = I_n, N = R_n <= 64.
//
// CTA: 128 columns kappa x all R (RP = R padded to 8), 8 warps, warp w owns
// the m16 tile of kappa rows 16w..16w+15 and all RP/8 n-tiles (the A
// fragment is reused across them).  K runs over i in chunks of 16; the G
// chunk is formed elementwise from T, E, Y_n (prefetched into registers one
// chunk ahead, coalesced along the contiguous index) and double-buffered in
// shared memory; the U chunk arrives by cp.async.
#pragma once
#include "pasd_pass2.cuh"

namespace pasd {

constexpr int P1_MT = 128;  // kappa columns per CTA
constexpr int P1_KC = 16;   // i rows per chunk
constexpr int P1_THREADS = 256;
constexpr int P1_EPT = P1_MT * P1_KC / P1_THREADS;  // elements per thread per chunk (8)

template <int RP>
__global__ void __launch_bounds__(P1_THREADS, 2) k_contract_A_mma(ModeDev m, const double* __restrict__ T,
                                                              const double* __restrict__ E0,
                                                              const double* __restrict__ E1,
                                                              const double* __restrict__ Y, const Ctl* ctl) {
  if (ctl->done) return;
  constexpr int NT = RP / 8, LDG = P1_MT + 4, LDU = RP + 4;
  extern __shared__ double p1sm[];
  double(*Gs)[P1_KC][LDG] = reinterpret_cast<double(*)[P1_KC][LDG]>(p1sm);
  double(*Us)[P1_KC][LDU] = reinterpret_cast<double(*)[P1_KC][LDU]>(p1sm + 2 * P1_KC * LDG);
  const double* __restrict__ E = ctl->ecur ? E1 : E0;
  const double inv_mu = __ddiv_rn(1.0, ctl->mu);  // pasd.cpp:170
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int64_t k0 = (int64_t)blockIdx.x * P1_MT;
  const int64_t I = m.I, inner = m.inner;
  const int R = m.R;
  const bool contig_i = inner == 1;  // mode 1: i is the contiguous index
  // per-thread staging elements: (kk_j, ii_j) and base offsets
  int kk[P1_EPT], ii[P1_EPT];
  int64_t base[P1_EPT];
  bool colok[P1_EPT];
#pragma unroll
  for (int j = 0; j < P1_EPT; ++j) {
    const int e = tid + P1_THREADS * j;
    if (contig_i) { ii[j] = e % P1_KC; kk[j] = e / P1_KC; }
    else { kk[j] = e % P1_MT; ii[j] = e / P1_MT; }
    const int64_t kap = k0 + kk[j];
    colok[j] = kap < m.J;
    const int64_t q = colok[j] ? kap / inner : 0;
    const int64_t p = colok[j] ? kap - q * inner : 0;
    base[j] = p + inner * ((int64_t)ii[j] + I * q);  // + inner * i0 per chunk
  }
  double tv[P1_EPT], ev[P1_EPT], yv[P1_EPT];
  auto load_chunk = [&](int64_t i0) {
#pragma unroll
    for (int j = 0; j < P1_EPT; ++j) {
      const bool ok = colok[j] && i0 + ii[j] < I;
      const int64_t off = base[j] + inner * i0;
      tv[j] = ok ? T[off] : 0.0;
      ev[j] = ok ? E[off] : 0.0;
      yv[j] = ok ? Y[off] : 0.0;
    }
  };
  auto store_chunk = [&](int buf, int64_t i0) {
#pragma unroll
    for (int j = 0; j < P1_EPT; ++j) Gs[buf][ii[j]][kk[j]] = g_elem(tv[j], ev[j], yv[j], inv_mu);
    for (int idx = tid; idx < P1_KC * RP; idx += P1_THREADS) {
      const int i = idx % P1_KC, r = idx / P1_KC;
      const bool ok = r < R && i0 + i < I;
      cp_async8(&Us[buf][i][r], ok ? m.U + m.ioff + (i0 + i) + m.Ifull * r : m.U, ok);
    }
  };
  double acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
  const int nchunks = (int)((I + P1_KC - 1) / P1_KC);
  load_chunk(0);
  store_chunk(0, 0);
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    if (c + 1 < nchunks) load_chunk((int64_t)(c + 1) * P1_KC);  // in flight during the MMAs
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < P1_KC / 4; ++ks) {
      const int k = 4 * ks + t;
      const double a0 = Gs[buf][k][16 * w + g], a1 = Gs[buf][k][16 * w + g + 8];
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[j], a0, a1, Us[buf][k][8 * j + g]);
    }
    if (c + 1 < nchunks) store_chunk(buf ^ 1, (int64_t)(c + 1) * P1_KC);
  }
  // epilogue: C rows kappa = 16w + g (+8), cols r = 8j + 2t (+1)
#pragma unroll
  for (int j = 0; j < NT; ++j) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t kap = k0 + 16 * w + g + 8 * (q >> 1);
      const int r = 8 * j + 2 * t + (q & 1);
      if (kap < m.J && r < R) m.A[a_offset(m, kap, r)] = acc[j][q];
    }
  }
}

template <int RP>
constexpr size_t p1_smem_bytes() {
  return sizeof(double) * 2 * P1_KC * ((P1_MT + 4) + (RP + 4));
}

template <int RP>
void launch_p1(const ModeDev& m, const double* T, const double* E0, const double* E1, const double* Y, const Ctl* ctl,
               cudaStream_t st) {
  static bool attr = false;  // idempotent attribute set (benign race)
  if (!attr) {
    cudaFuncSetAttribute(k_contract_A_mma<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p1_smem_bytes<RP>());
    attr = true;
  }
  const unsigned grid = (unsigned)((m.J + P1_MT - 1) / P1_MT);
  k_contract_A_mma<RP><<<grid, P1_THREADS, p1_smem_bytes<RP>(), st>>>(m, T, E0, E1, Y, ctl);
}

inline void launch_contract_A_mma(const ModeDev& m, const double* T, const double* E0, const double* E1,
                                  const double* Y, const Ctl* ctl, cudaStream_t st) {
  switch ((m.R + 7) / 8 * 8) {
    case 8: launch_p1<8>(m, T, E0, E1, Y, ctl, st); break;
    case 16: launch_p1<16>(m, T, E0, E1, Y, ctl, st); break;
    case 24: launch_p1<24>(m, T, E0, E1, Y, ctl, st); break;
    case 32: launch_p1<32>(m, T, E0, E1, Y, ctl, st); break;
    case 40: launch_p1<40>(m, T, E0, E1, Y, ctl, st); break;
    case 48: launch_p1<48>(m, T, E0, E1, Y, ctl, st); break;
    case 56: launch_p1<56>(m, T, E0, E1, Y, ctl, st); break;
    default: launch_p1<64>(m, T, E0, E1, Y, ctl, st); break;
  }
}

}  // namespace pasd
