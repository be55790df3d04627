// pasd_gram.cuh — Gram_n = A_n A_n^T (R_n x R_n) on the FP64 tensor cores.
// Replaces the dgesdd of the R x J matrix A_n inside svt (linops.cpp:83): the
// SVT only needs eig(A A^T) (see pasd_small.cuh).  Persistent CTAs stream
// 64-column chunks of A_n into shared memory (cp.async, double-buffered) and
// accumulate a private partial Gram with DMMA; k_gram_reduce sums the
// per-CTA partials in a fixed order.
#pragma once
#include "pasd_pass2.cuh"

namespace pasd {

constexpr int GM_KC = 64;  // kappa per chunk
constexpr int GM_THREADS = 256;

template <int RP>
struct GramLayout {
  static constexpr int RM = (RP + 15) / 16 * 16;  // rows covered by the m16 tiles
  static constexpr int MT = RM / 16, NT = RP / 8;
  // Gram is symmetric: only the tiles that meet the upper triangle r <= c
  // (n0 + 8 > m0, i.e. nt >= 2 mt) are formed; the reductions mirror the rest.
  static constexpr int upper_tiles() {
    int u = 0;
    for (int mt = 0; mt < MT; ++mt) u += NT > 2 * mt ? NT - 2 * mt : 0;
    return u;
  }
  static constexpr int UT = upper_tiles();
  // mode 1 (inner == 1): chunk as [kappa][r] (A_1 columns are contiguous in r);
  // other modes: [r][kappa] (64 contiguous kappa per r).  Both pitches are
  // 4 mod 16 doubles, so the fragment reads are conflict-free.
  static constexpr int LDR = RM + 4, LDK = GM_KC + 4;
  static constexpr int BUF = GM_KC * LDR > RM * LDK ? GM_KC * LDR : RM * LDK;
  static constexpr size_t bytes = sizeof(double) * 2 * BUF;
};

// Partial Gram of the chunks cta, cta + ncta, ... of mode m into
// m.Gpart[cta] (R x R).  RP >= round_up(R, 8).  Chunks of the strided modes
// never cross an outer index, so every staged row is one contiguous run.
template <int RP, bool CONTIG>
__device__ void gram_partial(const ModeDev& m, int cta, int ncta, double* gsm) {
  using L = GramLayout<RP>;
  constexpr int TILES = L::UT;
  constexpr int TPW = (TILES + 7) / 8;  // tiles per warp
  // upper tile index -> (m0, n0)
  auto tile_mn = [](int tile, int& m0, int& n0) {
    int mt = 0;
    while (tile >= L::NT - 2 * mt) {
      tile -= L::NT - 2 * mt;
      ++mt;
    }
    m0 = 16 * mt;
    n0 = 8 * (2 * mt + tile);
  };
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int R = m.R;
  const int64_t inner = m.inner;
  const int64_t pblocks = CONTIG ? 1 : (inner + GM_KC - 1) / GM_KC;
  const int64_t nchunks = CONTIG ? (m.J + GM_KC - 1) / GM_KC : pblocks * m.outer;
  auto at = [&](int kk, int r) { return CONTIG ? kk * L::LDR + r : r * L::LDK + kk; };
  // zero both buffers once: padding (r >= R) is never written by the copies
  for (int idx = tid; idx < 2 * L::BUF; idx += GM_THREADS) gsm[idx] = 0.0;
  __syncthreads();
  const bool al = CONTIG ? (R % 2 == 0) : (inner % 2 == 0);
  auto issue = [&](int64_t ch, int buf) {
    if (ch >= nchunks) return;
    const unsigned sb = smem_u32(gsm + buf * L::BUF);
    if (CONTIG) {
      // warp w -> columns kk = w + 8 j; lane -> r pair (16 B) or r = lane, lane + 32
      const int64_t k0 = ch * GM_KC;
#pragma unroll
      for (int j = 0; j < GM_KC / 8; ++j) {
        const int kk = w + 8 * j;
        const bool cok = k0 + kk < m.J;
        const double* col = m.A + (int64_t)R * (k0 + kk);
        if (al) {
          const int r = 2 * lane;
          if (r < R) cp16s(sb + 8u * at(kk, r), cok ? col + r : m.A, cok ? 16 : 0);
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            if (r < R) cp8s(sb + 8u * at(kk, r), cok ? col + r : m.A, cok ? 8 : 0);
          }
        }
      }
    } else {
      // thread -> 16-byte piece c of the 64-kappa run, rows r = tid / 32 + 8 j
      const int64_t q = ch / pblocks, p0 = (ch % pblocks) * GM_KC;
      const int np = (int)imin64(GM_KC, inner - p0);
      const double* base = m.A + p0 + inner * (int64_t)R * q;
      if (al) {
        const int c = lane, v = np - 2 * c, nb = v >= 2 ? 16 : (v == 1 ? 8 : 0);
#pragma unroll
        for (int j = 0; j < L::RM / 8; ++j) {
          const int r = w + 8 * j;
          if (r < R) cp16s(sb + 8u * at(2 * c, r), nb ? base + 2 * c + inner * r : m.A, nb);
        }
      } else {
#pragma unroll
        for (int j = 0; j < L::RM / 8; ++j) {
          const int r = w + 8 * j;
          if (r < R) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = lane + 32 * h;
              const bool ok = c < np;
              cp8s(sb + 8u * at(c, r), ok ? base + c + inner * r : m.A, ok ? 8 : 0);
            }
          }
        }
      }
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
    const double* As = gsm + buf * L::BUF;
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int tile = w + 8 * j;
      if (tile < TILES) {
        int m0, n0;
        tile_mn(tile, m0, n0);
#pragma unroll 4
        for (int ks = 0; ks < GM_KC / 4; ++ks) {
          const int kk = 4 * ks + t;
          dmma(acc[j], As[at(kk, m0 + g)], As[at(kk, m0 + g + 8)], As[at(kk, n0 + g)]);
        }
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's issue
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  double* out = m.Gpart + (int64_t)cta * R * R;
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tile = w + 8 * j;
    if (tile < TILES) {
      int m0, n0;
      tile_mn(tile, m0, n0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = m0 + g + 8 * (q >> 1), c = n0 + 2 * t + (q & 1);
        if (r < R && c < R) out[r * R + c] = acc[j][q];
      }
    }
  }
}

template <int RP>
__device__ __forceinline__ void gram_partial_any(const ModeDev& m, int cta, int ncta, double* gsm) {
  if (m.inner == 1)
    gram_partial<RP, true>(m, cta, ncta, gsm);
  else
    gram_partial<RP, false>(m, cta, ncta, gsm);
}

template <int RP>
__global__ void __launch_bounds__(GM_THREADS) k_gram_mma(ModeDev m, const Ctl* ctl) {
  if (ctl->done) return;
  extern __shared__ double gsm[];
  gram_partial_any<RP>(m, blockIdx.x, gridDim.x, gsm);
}

// All modes' Gram partials in one launch (unsharded solves): CTAs
// [base_n, base_n + nkc_g) form mode n's partials.  k_gram_reduce_all then
// sums them (one warp per entry, all modes in one launch) and k_svt runs the
// per-mode SVTs.  (A ticketed variant that reduced and ran the SVT in each
// mode's last CTA was slower at R >= 40: the single-CTA reduction of 148
// partials is latency bound.)
template <int RP>
__global__ void __launch_bounds__(GM_THREADS) k_gram_all(const ModePack* __restrict__ mp, const Ctl* ctl) {
  if (ctl->done) return;
  extern __shared__ double gsm[];
  int n = 0, base = 0;
  while (n + 1 < mp->order && (int)blockIdx.x >= base + mp->m[n].nkc_g) base += mp->m[n++].nkc_g;
  gram_partial_any<RP>(mp->m[n], blockIdx.x - base, mp->m[n].nkc_g, gsm);
}

// Gram_n = sum of the partials for every mode: one warp per entry, lanes take
// partials l, l+32, ..., then a fixed xor-shuffle tree (same order as
// k_gram_reduce, so sharded and unsharded solves agree bit for bit).
__global__ void k_gram_reduce_all(const ModePack* __restrict__ mp, const Ctl* ctl) {
  if (ctl->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t total = 0;
  for (int n = 0; n < mp->order; ++n) total += (int64_t)mp->m[n].R * mp->m[n].R;
  for (int64_t e = wid; e < total; e += nw) {
    int n = 0;
    int64_t idx = e;
    while (idx >= (int64_t)mp->m[n].R * mp->m[n].R) idx -= (int64_t)mp->m[n].R * mp->m[n++].R;
    const ModeDev& m = mp->m[n];
    const int64_t RR = (int64_t)m.R * m.R;
    const int64_t r = idx / m.R, c = idx - r * m.R;
    const int64_t src = r <= c ? idx : c * m.R + r;  // partials hold the upper triangle
    double a = 0.0;
    for (int kc = lane; kc < m.nkc_g; kc += 32) a += m.Gpart[kc * RR + src];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) m.Gram[idx] = a;
  }
}

template <int RP>
void launch_gram_all_rp(const ModePack* mp, const Ctl* ctl, int grid, cudaStream_t st) {
  ensure_smem_attr<k_gram_all<RP>>(GramLayout<RP>::bytes);
  k_gram_all<RP><<<grid, GM_THREADS, GramLayout<RP>::bytes, st>>>(mp, ctl);
}

inline void launch_gram_all(int rp, const ModePack* mp, const Ctl* ctl, int grid, cudaStream_t st) {
  switch (rp) {
    case 8: launch_gram_all_rp<8>(mp, ctl, grid, st); break;
    case 16: launch_gram_all_rp<16>(mp, ctl, grid, st); break;
    case 24: launch_gram_all_rp<24>(mp, ctl, grid, st); break;
    case 32: launch_gram_all_rp<32>(mp, ctl, grid, st); break;
    case 40: launch_gram_all_rp<40>(mp, ctl, grid, st); break;
    case 48: launch_gram_all_rp<48>(mp, ctl, grid, st); break;
    case 56: launch_gram_all_rp<56>(mp, ctl, grid, st); break;
    default: launch_gram_all_rp<64>(mp, ctl, grid, st); break;
  }
}

template <int RP>
void launch_gram_rp(const ModeDev& m, const Ctl* ctl, cudaStream_t st) {
  using L = GramLayout<RP>;
  ensure_smem_attr<k_gram_mma<RP>>(L::bytes);
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
