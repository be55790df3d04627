// pasd_synth.cuh — the reference's synthetic instance generator on the device
// (the step before the hot path), included by pasd_solver.cu.
//
//   gen_lowrank_tucker  proj/src/synth.cpp:71-89   core N(0,1) (R_1 x ... x R_N),
//                                                   factor n = Haar Q of an I_n x R_n
//                                                   N(0,1) matrix, sign-fixed by diag(R)
//                                                   (synth.cpp:40-53); T = core x_1 U_1 ... x_N U_N
//   corrupt_sparse      proj/src/synth.cpp:91-121  round(rho S) positions by partial
//                                                   Fisher-Yates, sorted, U[lo,hi] added
//                                                   (or written) in index order
//   RngStream           proj/include/tenrec/rng.hpp:17-79 (splitmix64-derived
//                                                   mt19937_64 streams, Box-Muller)
//
// Every random draw is the reference's: the streams are sequential by
// definition, so they run on the host (one mt19937_64 per purpose: core and
// factor Gaussians -- at most R^N + sum I_n R_n draws -- the round(rho S)
// Fisher-Yates indices and the noise values).  The tensor work runs on the
// device: the N mode products (1e11 flops at 1000^3, R = 50), the non-negative
// rescale, and placing the noise in sorted-index order WITHOUT sorting (a
// bitmap of the selected positions and its prefix popcount give every
// position its rank).  The partial Fisher-Yates keeps only displaced pool
// entries (open addressing), so it needs O(rho S) memory, not the reference's
// S-entry pool.
//
// Extensions for BASELINE configs[2..3] (documented in DESIGN.md; the oracle
// restates the same recipe): factor_kind 1 = |N(0,1)| factors, columns
// l2-normalised, |core|, T scaled by 1/max (C4); corrupt_mode 2 = per frame
// (last mode) `cells` aligned block x block cells of the mode-1 x mode-2 plane
// replaced by U[lo,hi] (C4 foreground, purposes 64/65).
//
// Parity: support and noise values are identical to the oracle's (exact
// integer / RNG work); L0 differs from the oracle's LAPACK / OpenBLAS
// arithmetic by rounding only (tests/test_gpu_synth.py).
#pragma once

#include <random>

namespace {

// ---------------------------------------------------------------- rng.hpp
constexpr uint64_t sx_splitmix64(uint64_t x) {  // rng.hpp:17-22
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
constexpr uint64_t sx_derive_seed(uint64_t seed, uint64_t stream, uint64_t purpose) {  // rng.hpp:24-26
  return sx_splitmix64(sx_splitmix64(sx_splitmix64(seed) ^ stream) ^ (purpose * 0x2545f4914f6cdd1dULL));
}
namespace sx_purpose {  // rng.hpp:28-35 (+ the C4 foreground tags)
constexpr uint64_t core = 1, support = 2, noise = 3, factor = 16, block_support = 64, block_noise = 65;
}

class SxRng {  // RngStream, rng.hpp:37-79
 public:
  SxRng(uint64_t seed, uint64_t stream, uint64_t purpose) : eng_(sx_derive_seed(seed, stream, purpose)) {}
  uint64_t next_u64() { return eng_(); }
  double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  uint64_t below(uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
      x = next_u64();
    } while (x >= limit);
    return x % n;
  }
  double gaussian() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    const double u1 = static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53;
    const double u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }

 private:
  std::mt19937_64 eng_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// Haar factor (synth.cpp:40-53): Householder QR of the Gaussian matrix, Q formed
// explicitly, columns negated where diag(R) < 0 (which makes Q unique).
// kind 1 (C4): |N(0,1)| entries, columns l2-normalised.
std::vector<double> sx_factor(int64_t rows, int64_t cols, SxRng& rng, int kind) {
  std::vector<double> a((size_t)(rows * cols));
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) a[i + rows * j] = rng.gaussian();
  if (kind == 1) {
    for (int64_t j = 0; j < cols; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < rows; ++i) {
        a[i + rows * j] = std::fabs(a[i + rows * j]);
        s += a[i + rows * j] * a[i + rows * j];
      }
      s = std::sqrt(s);
      for (int64_t i = 0; i < rows; ++i) a[i + rows * j] /= s;
    }
    return a;
  }
  // Householder: a := H_{cols-1} ... H_0 a = R (upper), reflectors v_k (v_k[k] = 1) kept below the diagonal.
  std::vector<double> beta((size_t)cols), rdiag((size_t)cols);
  for (int64_t k = 0; k < cols; ++k) {
    double* x = &a[k + rows * k];
    const int64_t m = rows - k;
    double sig = 0.0;
    for (int64_t i = 1; i < m; ++i) sig += x[i] * x[i];
    const double x0 = x[0];
    if (sig == 0.0) {  // already upper triangular in this column
      beta[k] = 0.0;
      rdiag[k] = x0;
      continue;
    }
    const double nrm = std::sqrt(x0 * x0 + sig);
    const double alpha = x0 <= 0.0 ? nrm : -nrm;  // R(k,k) = alpha, opposite sign to x0
    const double v0 = x0 - alpha;
    for (int64_t i = 1; i < m; ++i) x[i] /= v0;
    beta[k] = -v0 / alpha;  // H = I - beta v v^T with v = (1, x[1:] / v0)
    rdiag[k] = alpha;
    for (int64_t j = k + 1; j < cols; ++j) {
      double* c = &a[k + rows * j];
      double d = c[0];
      for (int64_t i = 1; i < m; ++i) d += x[i] * c[i];
      d *= beta[k];
      c[0] -= d;
      for (int64_t i = 1; i < m; ++i) c[i] -= d * x[i];
    }
  }
  // Q = H_0 H_1 ... H_{cols-1} applied to the first cols columns of the identity.
  std::vector<double> q((size_t)(rows * cols), 0.0);
  for (int64_t j = 0; j < cols; ++j) q[j + rows * j] = 1.0;
  for (int64_t k = cols - 1; k >= 0; --k) {
    if (beta[k] == 0.0) continue;
    const double* v = &a[k + rows * k];
    const int64_t m = rows - k;
    for (int64_t j = 0; j < cols; ++j) {
      double* c = &q[k + rows * j];
      double d = c[0];
      for (int64_t i = 1; i < m; ++i) d += v[i] * c[i];
      d *= beta[k];
      c[0] -= d;
      for (int64_t i = 1; i < m; ++i) c[i] -= d * v[i];
    }
  }
  for (int64_t j = 0; j < cols; ++j)
    if (rdiag[j] < 0.0)
      for (int64_t i = 0; i < rows; ++i) q[i + rows * j] = -q[i + rows * j];
  return q;
}

// Partial Fisher-Yates of synth.cpp:101-110 over [0, total): the first `count`
// entries of the shuffled pool, in draw order.  Only displaced entries are
// stored (open addressing on the position), so memory is O(count).
std::vector<int64_t> sx_partial_fisher_yates(int64_t total, int64_t count, SxRng& rng) {
  std::vector<int64_t> out((size_t)count);
  size_t cap = 16;
  while (cap < (size_t)count * 2 + 16) cap <<= 1;
  std::vector<int64_t> key(cap, -1), val(cap, 0);
  const size_t mask = cap - 1;
  auto slot = [&](int64_t p) {
    size_t h = (size_t)sx_splitmix64((uint64_t)p) & mask;
    while (key[h] != -1 && key[h] != p) h = (h + 1) & mask;
    return h;
  };
  for (int64_t i = 0; i < count; ++i) {
    const int64_t j = i + (int64_t)rng.below((uint64_t)(total - i));
    const size_t si = slot(i);
    const int64_t vi = key[si] == i ? val[si] : i;  // pool[i]
    const size_t sj = slot(j);
    const int64_t vj = key[sj] == j ? val[sj] : j;  // pool[j]
    out[(size_t)i] = vj;                              // swap: pool[i] = pool[j] (final)
    key[sj] = j;                                      // pool[j] = old pool[i]
    val[sj] = vi;
  }
  return out;
}

// out(p, i, q) = sum_r Q(i, r) in(p, r, q): the mode-n product of tensor.cpp:162-172.
__global__ void k_mode_product(const double* __restrict__ in, const double* __restrict__ Q, int64_t inner, int R,
                               int64_t I, int64_t outer, double* __restrict__ out) {
  const int64_t total = inner * I * outer;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rest = idx / inner;
    const int64_t p = idx - rest * inner;
    const int64_t q = rest / I;
    const int64_t i = rest - q * I;
    const double* src = in + p + inner * (int64_t)R * q;
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc = fma(Q[i + I * r], src[inner * r], acc);
    out[idx] = acc;
  }
}

__global__ void k_abs_inplace(double* x, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = fabs(x[i]);
}

// maxima of a non-negative buffer (the kind-1 instance)
__global__ void k_max_part(const double* __restrict__ x, int64_t n, double* part) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, x[i]);
  m = block_reduce(m, MaxOp(), red);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

__global__ void k_div_inplace(double* x, int64_t n, double d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __ddiv_rn(x[i], d);
}

__global__ void k_mark(const int64_t* __restrict__ pos, int64_t count, unsigned* __restrict__ bits) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos[k];
    atomicOr(&bits[p >> 5], 1u << (p & 31));
  }
}

// Exclusive prefix popcount of the bitmap words, in three passes over blocks of
// kScanBlock words.
constexpr int kScanBlock = 1024;
struct AddI64 {
  __device__ int64_t operator()(int64_t a, int64_t b) const { return a + b; }
  __device__ static int64_t identity() { return 0; }
};
__global__ void k_scan_block_sums(const unsigned* __restrict__ bits, int64_t nwords, int64_t* __restrict__ bsum) {
  __shared__ int64_t red[32];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock;
  int64_t s = 0;
  for (int t = threadIdx.x; t < kScanBlock; t += blockDim.x)
    if (base + t < nwords) s += __popc(bits[base + t]);
  s = block_reduce(s, AddI64(), red);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}
__global__ void k_scan_sums_serial(int64_t* bsum, int64_t nblocks) {  // one thread: nblocks <= ~3e4
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t acc = 0;
    for (int64_t b = 0; b < nblocks; ++b) {
      const int64_t v = bsum[b];
      bsum[b] = acc;
      acc += v;
    }
  }
}
__global__ void k_scan_words(const unsigned* __restrict__ bits, int64_t nwords, const int64_t* __restrict__ bsum,
                             int64_t* __restrict__ wpre) {
  // one block of kScanBlock threads per block of words: Hillis-Steele in shared memory
  __shared__ int64_t sh[kScanBlock];
  const int64_t w = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const int64_t c = w < nwords ? __popc(bits[w]) : 0;
  sh[threadIdx.x] = c;
  __syncthreads();
  for (int off = 1; off < kScanBlock; off <<= 1) {
    const int64_t add = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
    __syncthreads();
    sh[threadIdx.x] += add;
    __syncthreads();
  }
  if (w < nwords) wpre[w] = bsum[blockIdx.x] + sh[threadIdx.x] - c;
}
// out[p] (+)= noise[rank(p)] for every selected p (rank = its position in sorted order).
__global__ void k_scatter_noise(const int64_t* __restrict__ pos, int64_t count, const unsigned* __restrict__ bits,
                                const int64_t* __restrict__ wpre, const double* __restrict__ noise, int replace,
                                double* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos[k];
    const unsigned word = bits[p >> 5];
    const int64_t rank = wpre[p >> 5] + __popc(word & ((1u << (p & 31)) - 1u));
    const double v = noise[rank];
    out[p] = replace ? v : __dadd_rn(out[p], v);  // synth.cpp:114-117
  }
}
__global__ void k_scatter_pairs(const int64_t* __restrict__ pos, const double* __restrict__ v, int64_t count,
                                double* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x)
    out[pos[k]] = v[k];
}

constexpr int kSynthBlocks = 2368;

template <class T>
T* talloc(TmpDev& t, int64_t n) {
  return t.alloc<T>((size_t)std::max<int64_t>(n, 1));
}

void synth_instance(const pasd_synth_spec* sp, double* t_out, int t_is_device, double* l0_out, int l0_is_device,
                    int64_t* support_out, int64_t* count_out) {
  if (!sp || !sp->dims || !sp->ranks) fail(PASD_ERR_ARGUMENT, "pasd_b200: null synth spec");
  const int N = sp->order;
  if (N < 1) fail(PASD_ERR_ARGUMENT, "tensor order must be at least 1");
  std::vector<int64_t> dims(sp->dims, sp->dims + N), ranks(sp->ranks, sp->ranks + N);
  const int64_t S = dims_product(dims);
  // SynthSpec::validate (synth.cpp:12-37)
  for (int n = 0; n < N; ++n) {
    if (ranks[n] < 1)
      fail(PASD_ERR_ARGUMENT, "SynthSpec: rank of mode " + std::to_string(n + 1) + " must be positive");
    if (ranks[n] > dims[n])
      fail(PASD_ERR_ARGUMENT, "SynthSpec: rank " + std::to_string(ranks[n]) + " exceeds dimension " +
                                  std::to_string(dims[n]) + " in mode " + std::to_string(n + 1));
    int64_t other = 1;
    for (int m = 0; m < N; ++m)
      if (m != n) other *= ranks[m];
    if (ranks[n] > other)
      fail(PASD_ERR_ARGUMENT, "SynthSpec: rank " + std::to_string(ranks[n]) + " in mode " + std::to_string(n + 1) +
                                  " is unattainable (product of other ranks is " + std::to_string(other) + ")");
  }
  if (!(sp->corruption >= 0.0 && sp->corruption <= 1.0))
    fail(PASD_ERR_ARGUMENT, "SynthSpec: corruption fraction must lie in [0, 1]");
  if (!t_out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null output");
  CK(cudaSetDevice(sp->device));
  TmpDev tmp;
  // core (synth.cpp:74-78)
  std::vector<int64_t> cur = ranks;
  const int64_t core_size = dims_product(cur);
  std::vector<double> core((size_t)core_size);
  {
    SxRng rng(sp->seed, 0, sx_purpose::core);
    for (double& x : core) x = rng.gaussian();
    if (sp->factor_kind == 1)
      for (double& x : core) x = std::fabs(x);
  }
  // the largest intermediate of the product chain (the last product writes the output)
  int64_t maxsz = core_size;
  {
    std::vector<int64_t> d = ranks;
    for (int n = 0; n + 1 < N; ++n) {
      d[n] = dims[n];
      maxsz = std::max(maxsz, dims_product(d));
    }
  }
  double* bufA = t_is_device ? nullptr : talloc<double>(tmp, S);
  double* out_dev = t_is_device ? t_out : bufA;  // the final product lands here
  double* bufB = talloc<double>(tmp, maxsz);
  double* bufC = talloc<double>(tmp, maxsz);
  CK(cudaMemcpy(bufB, core.data(), sizeof(double) * core_size, cudaMemcpyHostToDevice));
  double* src = bufB;
  // mode products (synth.cpp:80-85): T = T x_n U_n
  for (int n = 0; n < N; ++n) {
    SxRng frng(sp->seed, 0, sx_purpose::factor + (uint64_t)n + 1);
    const std::vector<double> q = sx_factor(dims[n], ranks[n], frng, sp->factor_kind);
    double* dq = talloc<double>(tmp, dims[n] * ranks[n]);
    CK(cudaMemcpy(dq, q.data(), sizeof(double) * q.size(), cudaMemcpyHostToDevice));
    int64_t inner = 1, outer = 1;
    for (int l = 0; l < n; ++l) inner *= cur[l];
    for (int l = n + 1; l < N; ++l) outer *= cur[l];
    double* dst = (n == N - 1) ? out_dev : (src == bufB ? bufC : bufB);
    k_mode_product<<<kSynthBlocks, 256>>>(src, dq, inner, (int)ranks[n], dims[n], outer, dst);
    CK(cudaGetLastError());
    cur[n] = dims[n];
    src = dst;
  }
  if (sp->factor_kind == 1) {  // C4: scale into [0, 1] by the maximum
    double* part = talloc<double>(tmp, kSynthBlocks);
    k_max_part<<<kSynthBlocks, 256>>>(out_dev, S, part);
    std::vector<double> hp(kSynthBlocks);
    CK(cudaMemcpy(hp.data(), part, sizeof(double) * kSynthBlocks, cudaMemcpyDeviceToHost));
    double mx = 0.0;
    for (double v : hp) mx = std::max(mx, v);
    if (mx > 0.0) k_div_inplace<<<kSynthBlocks, 256>>>(out_dev, S, mx);
  }
  if (l0_out)
    CK(cudaMemcpy(l0_out, out_dev, sizeof(double) * S, l0_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
  int64_t count = 0;
  if (sp->corrupt_mode == 0 || sp->corrupt_mode == 1) {
    // corrupt_sparse (synth.cpp:91-121)
    count = (int64_t)std::llround(sp->corruption * (double)S);
    if (count > 0) {
      SxRng srng(sp->seed, 0, sx_purpose::support);
      const std::vector<int64_t> pos = sx_partial_fisher_yates(S, count, srng);
      std::vector<double> noise((size_t)count);
      SxRng nrng(sp->seed, 0, sx_purpose::noise);
      for (double& v : noise) v = nrng.uniform(sp->lo, sp->hi);
      int64_t* dpos = talloc<int64_t>(tmp, count);
      double* dnoise = talloc<double>(tmp, count);
      CK(cudaMemcpy(dpos, pos.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dnoise, noise.data(), sizeof(double) * count, cudaMemcpyHostToDevice));
      const int64_t nwords = (S + 31) / 32, nblk = (nwords + kScanBlock - 1) / kScanBlock;
      unsigned* bits = talloc<unsigned>(tmp, nwords);
      int64_t* bsum = talloc<int64_t>(tmp, nblk);
      int64_t* wpre = talloc<int64_t>(tmp, nwords);
      CK(cudaMemset(bits, 0, sizeof(unsigned) * nwords));
      k_mark<<<kSynthBlocks, 256>>>(dpos, count, bits);
      k_scan_block_sums<<<(unsigned)nblk, 256>>>(bits, nwords, bsum);
      k_scan_sums_serial<<<1, 1>>>(bsum, nblk);
      k_scan_words<<<(unsigned)nblk, kScanBlock>>>(bits, nwords, bsum, wpre);
      k_scatter_noise<<<kSynthBlocks, 256>>>(dpos, count, bits, wpre, dnoise, sp->corrupt_mode == 1, out_dev);
      CK(cudaGetLastError());
      if (support_out) {  // sorted support (synth.cpp:111): the bitmap in index order
        std::vector<unsigned> hb((size_t)nwords);
        CK(cudaMemcpy(hb.data(), bits, sizeof(unsigned) * nwords, cudaMemcpyDeviceToHost));
        int64_t k = 0;
        for (int64_t w = 0; w < nwords; ++w)
          for (unsigned b = hb[w]; b; b &= b - 1) support_out[k++] = w * 32 + __builtin_ctz(b);
      }
    }
  } else if (sp->corrupt_mode == 2) {
    // C4 foreground: per frame `cells` of the aligned block x block cells, U[lo, hi]
    if (N != 3) fail(PASD_ERR_ARGUMENT, "corrupt_blocks: order-3 tensors only");
    const int64_t block = sp->block, i1 = dims[0], i2 = dims[1], i3 = dims[2];
    if (block < 1) fail(PASD_ERR_ARGUMENT, "corrupt_blocks: block must be positive");
    const int64_t c1 = i1 / block, c2 = i2 / block, ncell = c1 * c2;
    if (sp->cells > ncell || sp->cells < 0) fail(PASD_ERR_ARGUMENT, "corrupt_blocks: too many cells");
    SxRng srng(sp->seed, 0, sx_purpose::block_support);
    SxRng nrng(sp->seed, 0, sx_purpose::block_noise);
    std::vector<int64_t> pos, pool((size_t)ncell);
    std::vector<double> val;
    pos.reserve((size_t)(i3 * sp->cells * block * block));
    val.reserve(pos.capacity());
    for (int64_t k = 0; k < i3; ++k) {
      for (int64_t c = 0; c < ncell; ++c) pool[(size_t)c] = c;
      for (int64_t i = 0; i < sp->cells; ++i) {
        const int64_t j = i + (int64_t)srng.below((uint64_t)(ncell - i));
        std::swap(pool[(size_t)i], pool[(size_t)j]);
      }
      std::vector<int64_t> chosen(pool.begin(), pool.begin() + sp->cells);
      std::sort(chosen.begin(), chosen.end());
      for (int64_t cidx : chosen) {
        const int64_t b1 = cidx % c1, b2 = cidx / c1;
        for (int64_t jj = 0; jj < block; ++jj)
          for (int64_t ii = 0; ii < block; ++ii) {
            pos.push_back((b1 * block + ii) + i1 * ((b2 * block + jj) + i2 * k));
            val.push_back(nrng.uniform(sp->lo, sp->hi));
          }
      }
    }
    count = (int64_t)pos.size();
    if (count) {
      int64_t* dpos = talloc<int64_t>(tmp, count);
      double* dval = talloc<double>(tmp, count);
      CK(cudaMemcpy(dpos, pos.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dval, val.data(), sizeof(double) * count, cudaMemcpyHostToDevice));
      k_scatter_pairs<<<kSynthBlocks, 256>>>(dpos, dval, count, out_dev);
      CK(cudaGetLastError());
      if (support_out) {
        std::vector<int64_t> sorted = pos;
        std::sort(sorted.begin(), sorted.end());
        std::memcpy(support_out, sorted.data(), sizeof(int64_t) * count);
      }
    }
  } else {
    fail(PASD_ERR_ARGUMENT, "pasd_b200: unknown corrupt_mode " + std::to_string(sp->corrupt_mode));
  }
  if (!t_is_device) CK(cudaMemcpy(t_out, out_dev, sizeof(double) * S, cudaMemcpyDeviceToHost));
  CK(cudaDeviceSynchronize());
  if (count_out) *count_out = count;
}

}  // namespace

extern "C" {

int pasd_b200_synth(const pasd_synth_spec* spec, double* t_out, int t_is_device, double* l0_out, int l0_is_device,
                    int64_t* support_out, int64_t* count_out, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    synth_instance(spec, t_out, t_is_device, l0_out, l0_is_device, support_out, count_out);
  });
}

int pasd_b200_synth_factor(int64_t rows, int64_t cols, uint64_t seed, int32_t mode, int32_t kind, double* out,
                           char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (rows < 1 || cols < 1 || cols > rows || !out) fail(PASD_ERR_ARGUMENT, "pasd_b200: bad factor shape");
    SxRng rng(seed, 0, sx_purpose::factor + (uint64_t)mode);
    const std::vector<double> q = sx_factor(rows, cols, rng, kind);
    std::memcpy(out, q.data(), sizeof(double) * q.size());
  });
}

int pasd_b200_synth_support(int64_t total, double rho, uint64_t seed, int64_t* pos_out, int64_t* count_out,
                            char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!(rho >= 0.0 && rho <= 1.0)) fail(PASD_ERR_ARGUMENT, "corrupt_sparse: rho must lie in [0, 1]");
    if (total < 1) fail(PASD_ERR_ARGUMENT, "pasd_b200: total must be positive");
    const int64_t count = (int64_t)std::llround(rho * (double)total);
    if (count_out) *count_out = count;
    if (!pos_out || count == 0) return;
    SxRng rng(seed, 0, sx_purpose::support);
    const std::vector<int64_t> pos = sx_partial_fisher_yates(total, count, rng);
    std::memcpy(pos_out, pos.data(), sizeof(int64_t) * count);
  });
}

}  // extern "C"
