// pasd_gram.cuh — Gram_n = A_n A_n^T (R_n x R_n) on the FP64 tensor cores.
// Replaces the dgesdd of the R x J matrix A_n inside svt (linops.cpp:83): the
// SVT only needs eig(A A^T) (see pasd_small.cuh).  Persistent CTAs stream
// 64-column chunks of A_n into shared memory (cp.async, double-buffered) and
// accumulate a private partial Gram with DMMA; k_gram_reduce sums the
// per-CTA partials in a fixed order.
#pragma once
#include "pasd_pass2.cuh"
#include "pasd_small.cuh"

namespace pasd {

constexpr int GM_KC = 64;  // kappa per chunk
constexpr int GM_THREADS = 256;

template <int RP>
struct GramLayout {
  static constexpr int RM = (RP + 15) / 16 * 16;
  static constexpr int LD = RM + 4;
  static constexpr int MT = RM / 16, NT = RP / 8;
  static constexpr size_t bytes = sizeof(double) * 2 * GM_KC * LD;
};

// Partial Gram of the chunks cta, cta + ncta, ... of mode m into
// m.Gpart[cta] (R x R).  RP >= round_up(R, 8).
template <int RP>
__device__ void gram_partial(const ModeDev& m, int cta, int ncta, double* gsm) {
  using L = GramLayout<RP>;
  constexpr int TILES = L::MT * L::NT;
  constexpr int TPW = (TILES + 7) / 8;  // tiles per warp
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int R = m.R;
  const int64_t nchunks = (m.J + GM_KC - 1) / GM_KC;
  // zero padding columns (r >= R) of both buffers once
  for (int idx = tid; idx < 2 * GM_KC * (L::LD - R); idx += GM_THREADS) {
    const int row = idx / (L::LD - R), c = R + idx % (L::LD - R);
    gsm[row * L::LD + c] = 0.0;
  }
  auto issue = [&](int64_t ch, int buf) {
    if (ch >= nchunks) return;
    double* dst = gsm + buf * GM_KC * L::LD;
    const int64_t k0 = ch * GM_KC;
    for (int idx = tid; idx < GM_KC * R; idx += GM_THREADS) {
      int kk, r;
      if (m.inner == 1) { r = idx % R; kk = idx / R; }   // A[r + R kappa]: r contiguous
      else { kk = idx % GM_KC; r = idx / GM_KC; }          // kappa (p) contiguous
      const int64_t kap = k0 + kk;
      const bool ok = kap < m.J;
      cp_async8(dst + kk * L::LD + r, ok ? m.A + a_offset(m, kap, r) : m.A, ok);
    }
  };
  double acc[TPW][4];
#pragma unroll
  for (int j = 0; j < TPW; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
  int64_t ch = cta;
  issue(ch, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  int buf = 0;
  for (; ch < nchunks; ch += ncta, buf ^= 1) {
    issue(ch + ncta, buf ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const double* As = gsm + buf * GM_KC * L::LD;
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int tile = w + 8 * j;
      if (tile < TILES) {
        const int m0 = 16 * (tile / L::NT), n0 = 8 * (tile % L::NT);
#pragma unroll 4
        for (int ks = 0; ks < GM_KC / 4; ++ks) {
          const double* row = As + (4 * ks + t) * L::LD;
          dmma(acc[j], row[m0 + g], row[m0 + g + 8], row[n0 + g]);
        }
      }
    }
    __syncthreads();  // buffer `buf` is refilled two chunks later
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  double* out = m.Gpart + (int64_t)cta * R * R;
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tile = w + 8 * j;
    if (tile < TILES) {
      const int m0 = 16 * (tile / L::NT), n0 = 8 * (tile % L::NT);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = m0 + g + 8 * (q >> 1), c = n0 + 2 * t + (q & 1);
        if (r < R && c < R) out[r * R + c] = acc[j][q];
      }
    }
  }
}

template <int RP>
__global__ void __launch_bounds__(GM_THREADS) k_gram_mma(ModeDev m, const Ctl* ctl) {
  if (ctl->done) return;
  extern __shared__ double gsm[];
  gram_partial<RP>(m, blockIdx.x, gridDim.x, gsm);
}

// All modes' Gram matrices and their SVTs in one launch (unsharded solves):
// CTAs [base_n, base_n + nkc_g) form mode n's partials; the last of them to
// finish (atomic ticket) sums the partials in index order (deterministic) and
// runs the SVT of mode n in the same CTA.  Replaces k_gram_mma + k_gram_reduce
// per mode and k_svt (7 launches at order 3).
template <int RP>
__global__ void __launch_bounds__(GM_THREADS) k_gram_svt(const ModePack* __restrict__ mp, Ctl* ctl, int* tickets) {
  if (ctl->done) return;
  extern __shared__ double gsm[];
  __shared__ int last;
  int n = 0, base = 0;
  while (n + 1 < mp->order && (int)blockIdx.x >= base + mp->m[n].nkc_g) base += mp->m[n++].nkc_g;
  const ModeDev& m = mp->m[n];
  gram_partial<RP>(m, blockIdx.x - base, m.nkc_g, gsm);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&tickets[n], 1) == m.nkc_g - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) tickets[n] = 0;  // ready for the next replay
  const int RR = m.R * m.R;
  for (int idx = threadIdx.x; idx < RR; idx += blockDim.x) {
    double a = 0.0;
    for (int kc = 0; kc < m.nkc_g; ++kc) a += __ldcg(m.Gpart + (int64_t)kc * RR + idx);
    m.Gram[idx] = a;
  }
  __syncthreads();
  svt_mode(m, n, ctl, gsm);
}

template <int RP>
void launch_gram_svt_rp(const ModePack* mp, Ctl* ctl, int* tickets, int grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gram_svt<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_gram_svt<RP><<<grid, GM_THREADS, smem, st>>>(mp, ctl, tickets);
}

// smem of k_gram_svt<rp>: the larger of the chunk ring and the SVT workspace
inline size_t gram_svt_smem(int rp, int maxR) {
  const size_t ring = sizeof(double) * 2 * GM_KC * ((rp + 15) / 16 * 16 + 4);
  const size_t ws = small_ws_bytes(maxR);
  return ring > ws ? ring : ws;
}

inline void launch_gram_svt(int rp, const ModePack* mp, Ctl* ctl, int* tickets, int grid, size_t smem,
                            cudaStream_t st) {
  switch (rp) {
    case 8: launch_gram_svt_rp<8>(mp, ctl, tickets, grid, smem, st); break;
    case 16: launch_gram_svt_rp<16>(mp, ctl, tickets, grid, smem, st); break;
    case 24: launch_gram_svt_rp<24>(mp, ctl, tickets, grid, smem, st); break;
    case 32: launch_gram_svt_rp<32>(mp, ctl, tickets, grid, smem, st); break;
    case 40: launch_gram_svt_rp<40>(mp, ctl, tickets, grid, smem, st); break;
    case 48: launch_gram_svt_rp<48>(mp, ctl, tickets, grid, smem, st); break;
    case 56: launch_gram_svt_rp<56>(mp, ctl, tickets, grid, smem, st); break;
    default: launch_gram_svt_rp<64>(mp, ctl, tickets, grid, smem, st); break;
  }
}

template <int RP>
void launch_gram_rp(const ModeDev& m, const Ctl* ctl, cudaStream_t st) {
  using L = GramLayout<RP>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gram_mma<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes);
    attr = true;
  }
  k_gram_mma<RP><<<m.nkc_g, GM_THREADS, L::bytes, st>>>(m, ctl);
}

inline void launch_gram_mma(const ModeDev& m, const Ctl* ctl, cudaStream_t st) {
  switch ((m.R + 7) / 8 * 8) {
    case 8: launch_gram_rp<8>(m, ctl, st); break;
    case 16: launch_gram_rp<16>(m, ctl, st); break;
    case 24: launch_gram_rp<24>(m, ctl, st); break;
    case 32: launch_gram_rp<32>(m, ctl, st); break;
    case 40: launch_gram_rp<40>(m, ctl, st); break;
    case 48: launch_gram_rp<48>(m, ctl, st); break;
    case 56: launch_gram_rp<56>(m, ctl, st); break;
    default: launch_gram_rp<64>(m, ctl, st); break;
  }
}

}  // namespace pasd
