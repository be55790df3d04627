// pasd_pass2.cuh — fused pass 2 of a PASD iteration for order-3 tensors on
// the FP64 tensor cores (DMMA, mma.sync.m16n8k4.f64).
//
// One kernel replaces, per iteration (reference: proj/src/pasd.cpp:189-228 and
// the next iteration's procrustes product, linops.cpp:98):
//   Z_n = fold_n(U_n V_n) = UM_n x_n A_n          (refold; V_n = M_n A_n)
//   h   = sum_n (T - Z_n) + Y_n/mu ; E = soft(h/N, 1/(mu N))
//   Y_n += mu ((T - Z_n) - E) ; resid_n = max |.| ; NaN flag
//   Wt_n = G_n^{next} A_n^T with G_n^{next} = (T - E) + Y_n/mu_next, and ||G_n^{next}||^2
// HBM traffic: T, Y_1..3 read once, E, Y_1..3 written once; A_n slices come
// through L2: by default (PASD_P2_BULK) as one
// cp.async.bulk copy per slice from the tiled, padded copies k_retile writes
// (released per slice by shared-memory counters, completed on mbarriers).
//
// Work decomposition.  A persistent CTA walks "pencils": a 16 (i1) x 8 (i3)
// patch swept over all i2 in steps of 8.  Per step the brick is
// 16 x 8 x 8 = 1024 elements.  The A_2 slice of the pencil (R2 x 16 x 8,
// indexed by (i1, i3)) stays resident in shared memory for the whole sweep;
// A_1 (R1 x 8 x 8, by (i2, i3)) and A_3 (R3 x 16 x 8, by (i1, i2)) are loaded
// per step.  Warp w (of 8) owns the (16 i1 x 8 i2) tile at i3 = w for Z_1 and
// Z_2 (identical accumulator layouts), and the (16 i1 x 8 i3) tile at i2 = w
// for Z_3 (exchanged through shared memory).  Wt_1 uses the warp's own G_1
// values directly as the DMMA A operand; Wt_2 / Wt_3 read G_2 / G_3 from
// shared memory.  Wt_1 / Wt_3 rows are fixed along a pencil (register
// accumulation, one partial per pencil, or per pencil segment when the solver
// splits the i2 sweep, Pass2Args::nseg); Wt_2 rows change per step and go to a
// per-CTA partial (its two K-halves exchanged by a warp-pair barrier, or kept as
// two partials when they fit in L2, Pass2Args::nw2).  All reductions are in a
// fixed order (deterministic).
#pragma once
#include <type_traits>

#include <cuda.h>  // CUtensorMap (TMA descriptors, encoded on the host through the driver entry point)

#include "pasd_kernels.cuh"

namespace pasd {

#ifndef PASD_P2_PAIRBAR
#define PASD_P2_PAIRBAR 1  // Wt_2 K-half exchange synchronised per warp pair (named barrier)
#endif
#ifndef PASD_P2_PROBE
#define PASD_P2_PROBE 0  // timing probes only (wrong results): 1 = skip the Wt DMMAs, 2 = skip the Z DMMAs,
                         // 3 = skip both, 4 = skip the elementwise arithmetic (loads and stores stay),
                         // 5 = Z products with the pencil-constant operands loaded once (register reuse bound),
                         // 6 = no element stores (E, D, Y_n), 7 = no element loads (T, Y_n)
#endif
#ifndef PASD_P2_EPF
#define PASD_P2_EPF 0  // T / Y_n element bricks staged into shared memory with cp.async a step ahead
#endif
#ifndef PASD_P2_WS
#define PASD_P2_WS 1  // warps 0-3 run the Wt_2 products over the full K while warps 4-7 issue the next staging
#endif
#ifndef PASD_P2_TIL
#define PASD_P2_TIL 1  // TMA variant (TIO) loads only: the T, Y_n bricks of the next step arrive by TMA (requested
                       // right after the elementwise phase), E / D / Y_n leave by plain stores, G_2 / G_3 go
                       // through the padded exchange buffers (0: loads and stores by TMA, six bricks;
                       // 2: as 1, but E and Y_n also leave by TMA from the load bricks, in place; D by plain stores)
#endif
#ifndef PASD_P2_BULK
#define PASD_P2_BULK 1  // A_1 / A_2 / A_3 slices and the UM_2 rows arrive as single cp.async.bulk copies from
                        // pre-tiled, pre-padded copies of A_n (k_retile, one launch before pass 2) instead of
                        // ~190 warp-LDGSTS per step; buffers are released per slice (shared-memory counters),
                        // barrier D and the warp-specialised staging phase go away
#endif
#ifndef PASD_P2_ELD
#define PASD_P2_ELD 0  // (bulk variant) where a step's T / Y_n element loads are issued: 0 = at the step's top (in
                       // flight during the Z products), 1 = before the previous step's Wt_2 products,
                       // 2 = right after the previous step's elementwise phase
#endif
#ifndef PASD_P2_ZPIPE
#define PASD_P2_ZPIPE 0  // Z products software-pipelined by hand: the nine operand loads of k-step s + 1 are issued
                         // (volatile ld.shared, so ptxas keeps the order) before the DMMAs of k-step s.  ncu's
                         // per-instruction samples showed the unpipelined loop waiting ~120 cycles per k-step on
                         // its own operand loads: all 8 warps issue their loads in the same burst
#endif
#ifndef PASD_P2_SOFTSEL
#define PASD_P2_SOFTSEL 0  // elementwise phase without branches (soft threshold as selects, unguarded residual
                           // reductions: 399 -> 264 instructions, the four elements' FP64 chains interleaved).
                           // Parity-green; measured slower: C5 38.1 vs 37.4, C3 2.135 vs 2.109 ms per launch
#endif
#ifndef PASD_P2_L2HINT
#define PASD_P2_L2HINT 1  // bulk copies of the tiled slices carry an L2 evict_last policy
#endif
#ifndef PASD_P2_EHINT
#define PASD_P2_EHINT 0  // (bulk variant, float64 storage) the element streams T, Y_n, E, D carry an L2 evict_first
                         // policy.  Measured worse at C5: DRAM reads 46.6 -> 50.5 GB, 37.1 -> 37.9 ms per launch
#endif
#ifndef PASD_P2_HALF
#define PASD_P2_HALF 0  // padded ranks 8 mod 16 (RP 40, 56): the last m-tile of the Wt_2 / Wt_3 products has only
                        // padding in its upper 8 rows -> one DMMA.8x8x4 per k-step instead of two; the m-tiles are
                        // assigned so that each scheduler hosts exactly one of the four light (m-tile, K-half) items.
                        // Parity-green; no gain (predicated upper half: C5 36.7 vs 36.8, C3 2.12 vs 2.08 ms per
                        // launch; as separate m8n8k4 loops: 38.3 ms, 250 registers)
#endif
#ifndef PASD_P2_TIMING
#define PASD_P2_TIMING 0  // probe build: per-phase clock64() sums of warp 0 (pasd_b200_debug_p2_phases)
#endif
#ifndef PASD_P2_TWARP
#define PASD_P2_TWARP 0  // the warp whose lane 0 records the phase clocks
#endif
#if PASD_P2_TIMING
__device__ unsigned long long g_p2_phase[12];
#define P2T(k)                                   \
  do {                                           \
    if (tid == 32 * PASD_P2_TWARP) {             \
      const long long now_ = clock64();          \
      ph_acc[k] += (unsigned long long)(now_ - ph_t); \
      ph_t = now_;                               \
    }                                            \
  } while (0)
#else
#define P2T(k) do {} while (0)
#endif
#ifndef PASD_P2_BW
#define PASD_P2_BW 12  // i1-block band width of the pencil order
#endif
#ifndef PASD_P2_DW2
#define PASD_P2_DW2 0  // (bulk variant) the Wt_2 products of a step are deferred into the next step's
                       // elementwise phase (one instruction stream: the DMMAs fill the phase that had none);
                       // G_2 exchange buffer doubled, K-half partials through their own exchange buffer
#endif
// Bulk-staged slices (PASD_P2_BULK): plain element I/O only.
template <bool TIO>
constexpr bool pass2_bulk() {
  return !TIO && PASD_P2_BULK && !PASD_P2_EPF;
}
template <bool TIO>
constexpr bool pass2_dw2() {
  return pass2_bulk<TIO>() && PASD_P2_DW2;
}
constexpr int P2_B1 = 16, P2_B2 = 8, P2_B3 = 8;
constexpr int P2_THREADS = 256;
constexpr int P2_BRICK = P2_B1 * P2_B2 * P2_B3;  // 1024

struct Pass2Args {
  ModeDev m[3];
  const double* T;
  double* E0;
  double* E1;
  double* D;   // T - E_new (pass 1's tensor operand)
  double* Y[3];
  double* W1p;     // [npencils][16][R1]
  double* W3p;     // [npencils][8][R3]
  double* W2part;  // [grid][I2][R2]
  double* gpart;   // [grid][3]
  double* resid_part;  // [grid][PASD_MAX_ORDER]
  int* bad_part;       // [grid]
  int n1b, n3b, npencils;
  int nseg;  // i2 segments per pencil (Wt_1 / Wt_3 partials: npencils x nseg)
  int nw2;  // Wt_2 partial slices in W2part (fused: 2 per CTA, one per K-half; m8: 1 per CTA)
  int b1;  // i1 extent of a pencil (16 for k_pass2_fused, 8 for k_pass2_m8)
  // unsharded solves: the last CTA runs the iteration's finish (mu schedule,
  // history, stop rule) -- one launch fewer per iteration
  int* finish_ticket;  // nullptr: k_finish runs separately
  double* history;
  // PASD_P2_BULK: tiled copies of A_n / UM_2 in the shared-memory slice layouts of k_pass2_fused (k_retile)
  double* At1;  // [ib3][i2 block][64 columns (l2 + 8 l3)][RP + 4]
  double* At2;  // [ib3][ib1][RP][132]  (column 16 l3 + l1)
  double* At3;  // [ib1][i2 block][RP][132]  (column 16 l2 + l1)
  double* U2t;  // [i2 block][8][RP + 4]
  int n2b;      // i2 blocks of 8
};

// TMA descriptors of the element streams of k_pass2_fused<RP, true>: 3-D
// float64 maps with a 16 x 8 x 8 box and 128-byte swizzle.  "A" maps are
// (I1, I2, I3); the "B" map of Y_3 is (I1, I3, I2), so its brick lands in
// shared memory as [l2][l3][l1] and the Wt_3 operand reads are conflict-free.
struct P2Tmaps {
  CUtensorMap t, y1, y2, y3b;  // loads
  CUtensorMap y3a;             // Y_3 in the A layout (PASD_P2_TIL)
  CUtensorMap e0, e1, d;       // stores (E double buffer: the kernel writes E[ecur ^ 1])
};

__host__ __device__ inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// m16n8k4 as two m8n8k4 (the same two DMMA.8x8x4), the rows 8-15 half under a warp-uniform predicate.
__device__ __forceinline__ void dmma_split(double (&c)[4], double a0, double a1, double b0, bool upper) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %7, 0;\n\t"
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%4}, {%6}, {%0,%1};\n\t"
      "@p mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%2,%3}, {%5}, {%6}, {%2,%3};\n\t}"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0), "r"((unsigned)upper));
}

// Asynchronous global->shared copy of one double (LDGSTS); src_bytes = 0
// zero-fills the destination (out-of-range / padding entries).
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int nbytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int nbytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(nbytes) : "memory");
}

// Stage `rows` rows of 16 consecutive doubles (row j: src + j*step_r, with
// the i1 extent clipped to `nvalid`) into dst[j*ld .. j*ld+15].  16-byte
// copies when the source rows are 16-byte aligned, else 8-byte copies.
__device__ __forceinline__ void stage_rows16(double* dst, int ld, const double* src, int64_t row_stride, int rows,
                                             int nvalid, bool aligned16, const double* dummy) {
  const int tid = threadIdx.x;
  if (aligned16) {
    const int c = tid & 7;  // 16-byte chunk within the row
    const int v = nvalid - 2 * c;
    const int nb = v >= 2 ? 16 : (v == 1 ? 8 : 0);
    for (int j = tid >> 3; j < rows; j += P2_THREADS / 8)
      cp_async16(dst + j * ld + 2 * c, nb ? src + row_stride * j + 2 * c : dummy, nb);
  } else {
    const int c = tid & 15;
    const bool ok = c < nvalid;
    for (int j = tid >> 4; j < rows; j += P2_THREADS / 16)
      cp_async8(dst + j * ld + c, ok ? src + row_stride * j + c : dummy, ok);
  }
}

// Same copies addressed by a 32-bit shared-window address (no per-copy
// generic->shared conversion in the unrolled staging loops).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16s(unsigned s, const void* gmem, int nbytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp8s(unsigned s, const void* gmem, int nbytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(nbytes) : "memory");
}

// Same copies with an all-or-nothing zero fill: the ignore-src predicate form
// (LDGSTS.ZFILL with a predicate) needs no per-copy src-size arithmetic.
// `gmem` must still be a valid address when !valid (it is not read).
__device__ __forceinline__ void cp16z(unsigned s, const void* gmem, bool valid) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\t"
      "cp.async.cg.shared.global [%0], [%1], 16, p;\n\t}" ::"r"(s),
      "l"(gmem), "r"((unsigned)valid)
      : "memory");
}
__device__ __forceinline__ void cp8z(unsigned s, const void* gmem, bool valid) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\t"
      "cp.async.ca.shared.global [%0], [%1], 8, p;\n\t}" ::"r"(s),
      "l"(gmem), "r"((unsigned)valid)
      : "memory");
}

// Shared-memory load the compiler may not reorder against the DMMAs (both volatile asm).
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Brick element index e = i1 + 16 * (i2 + 8 * i3) (local coordinates).
__device__ __forceinline__ int bidx(int l1, int l2, int l3) { return l1 + P2_B1 * (l2 + P2_B2 * l3); }
// Padded exchange layouts (strides in doubles), conflict-free for their
// write and read patterns within a half-warp (g, t in 0..3):
//   Z3: written (l1=g, l3=2t), read (l1=g, l2=2t)        -> strides 22 / 182
//   G2: written (l1=g, l2=2t), read (l1=t+c, l2=g)        -> strides 20 / 160
//   G3: written (l1=g, l2=2t), read (l1=t+c, l3=g)        -> strides 22 / 180
__device__ __forceinline__ int zx(int l1, int l2, int l3) { return l1 + 22 * l2 + 182 * l3; }
__device__ __forceinline__ int g2x(int l1, int l2, int l3) { return l1 + 20 * l2 + 160 * l3; }
__device__ __forceinline__ int g3x(int l1, int l2, int l3) { return l1 + 22 * l2 + 180 * l3; }
__device__ __forceinline__ bool mt_dummy_guard(int w, int MT) { return (w & 3) < MT; }
// Staged element brick (PASD_P2_EPF): row (l2, l3) holds 16 consecutive i1 as eight
// 16-byte chunks, chunk c stored at c ^ (l2 & 6), so the elementwise reads
// (l1 = g (+8), l2 = 2t (+1)) of a half-warp hit 16 distinct bank pairs.
__device__ __forceinline__ int ex(int l1, int l2, int l3) {
  return 16 * (l2 + 8 * l3) + 2 * ((l1 >> 1) ^ (l2 & 6)) + (l1 & 1);
}

// Shared-memory footprint (bytes) of k_pass2_fused<RP, TIO>.
template <int RP, bool TIO>
struct P2Layout {
  // The Wt_2 / Wt_3 products read the A_2 / A_3 slices as 16-row M tiles
  // covering RM rows; rows >= RP of the last tile run past the slice into the
  // next buffer.  Those rows only feed output rows r >= RP, which are never
  // stored, so the slices hold RP rows (rows R..RP-1 zero: the Z products use
  // them along K).
  static constexpr int RM = (RP + 15) / 16 * 16;
  // A1s is column-major: [column c = l2 + 8 l3][r], pitch LD1 = RP + 4 (4 or 12
  // mod 16: the Z_1 reads (c = g, r = t) are conflict-free, the Wt_1 reads
  // (c = 2t, r = g) 2-way), so each column's R1 contiguous values of A_1
  // stage as 16-byte copies.  Other pitches keep the fragment reads
  // (rows t x cols g, rows g x cols t) on distinct banks per half-warp.
  // (Double-buffering A_1 to stage it a whole step ahead measured slower:
  // 49.7 vs 43.2 ms per C5 launch.)
  static constexpr int LD1 = RP + 4, LD2 = 128 + 4, LD3 = 128 + 4, LDU = RP + 4;
  static constexpr int oA1 = 0;
  static constexpr int oA2 = oA1 + 64 * LD1;
  static constexpr int oA3 = oA2 + RP * LD2;
  static constexpr int oU1 = oA3 + RP * LD3;
  static constexpr int oU2 = oU1 + 16 * LDU;
  static constexpr int oU3 = oU2 + 8 * LDU;
  static constexpr int oZ3 = oU3 + 8 * LDU;
  // plain I/O: G_2 / G_3 exchange buffers.  TMA I/O (TIO): six 16 x 8 x 8
  // bricks (T->E, Y_1, Y_2, Y_3 [B layout], D, D [B layout]) read by the
  // Wt_2 / Wt_3 products directly (G = D + Y/mu formed in the fragment load).
  static constexpr int oG2 = oZ3 + 8 * 182;
  static constexpr bool TIL = TIO && PASD_P2_TIL;  // TMA loads only: four bricks (T, Y_1..3) + the exchange buffers
  static constexpr bool DW2 = pass2_dw2<TIO>();  // two G_2 buffers (step parity) + the Wt_2 K-half exchange
  static constexpr int oG3 = oG2 + (TIO && !TIL ? 0 : 8 * 160) * (DW2 ? 2 : 1);
  static constexpr int oX2 = oG3 + (TIO && !TIL ? 0 : 8 * 180);
  static constexpr int oRed = oX2 + (DW2 ? 512 : 0);
  static constexpr int oBrick = oRed + 64;              // + runtime 1024-byte alignment
  // plain I/O with PASD_P2_EPF: the next step's T, Y_1..3 bricks (4 x 1024, swizzled rows)
  static constexpr bool EPF =
      !TIO && PASD_P2_EPF && sizeof(double) * (size_t)(oBrick + 4 * P2_BRICK) <= 227u * 1024u;
  static constexpr int total = oBrick + (TIO ? (TIL ? 4 : 6) * P2_BRICK + 128 : (EPF ? 4 * P2_BRICK : 0));
  static constexpr size_t bytes = sizeof(double) * (size_t)total;
  static_assert((RM - RP) * LD3 <= total - oU1, "M-tile overrun must stay inside shared memory");
  static_assert(128 * RP <= oA3 + RP * LD3, "end-of-pencil scratch must fit in A1s..A3s");
};

// The layout as a kernel with element type EL sees it: the element-brick staging
// (PASD_P2_EPF) copies 16-byte pairs of float64 and is off for float storage.
template <int RP, bool TIO, class EL>
struct P2LayoutE : P2Layout<RP, TIO> {
  static constexpr bool EPF = P2Layout<RP, TIO>::EPF && sizeof(EL) == 8;
};

// Element (l1, l2, l3) of a 16 x 8 x 8 brick in the TMA SWIZZLE_128B layout:
// 128-byte rows of 16 doubles, 16-byte chunks XOR-ed with (row mod 8).
// Layout A: row = l2 + 8 l3; layout B: row = l3 + 8 l2.
__device__ __forceinline__ int swz_row(int l1, int row) { return row * 16 + (((l1 >> 1) ^ (row & 7)) << 1) + (l1 & 1); }
__device__ __forceinline__ int swzA(int l1, int l2, int l3) { return swz_row(l1, l2 + 8 * l3); }
__device__ __forceinline__ int swzB(int l1, int l2, int l3) { return swz_row(l1, l3 + 8 * l2); }

__device__ __forceinline__ void tma_load3(double* dst, const CUtensorMap* map, uint64_t* mbar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      :
      : "r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(reinterpret_cast<uint64_t>(map)),
        "r"(static_cast<unsigned>(__cvta_generic_to_shared(mbar))), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, const double* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
               :
               : "l"(reinterpret_cast<uint64_t>(map)), "r"(static_cast<unsigned>(__cvta_generic_to_shared(src))),
                 "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(mbar)))
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(mbar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(mbar))),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, no tensor map): `bytes` a multiple of 16,
// both addresses 16-byte aligned; completion is signalled on `mbar` (complete_tx).
__device__ __forceinline__ void bulk_load(double* dst, const double* src, unsigned bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(src), "r"(bytes),
                 "r"(static_cast<unsigned>(__cvta_generic_to_shared(mbar)))
               : "memory");
}
// ... with an L2 cache policy (createpolicy): the tiled A slices are re-read by every pencil of a band, the
// element streams pass through L2 once
__device__ __forceinline__ void bulk_load_hint(double* dst, const double* src, unsigned bytes, uint64_t* mbar,
                                               uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      :
      : "r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(src), "r"(bytes),
        "r"(static_cast<unsigned>(__cvta_generic_to_shared(mbar))), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Predicated float64 load / store with an L2 cache policy (no branch: the predicate is part of the instruction).
__device__ __forceinline__ double ldg_hint(const double* p, bool ok, uint64_t policy) {
  double v = 0.0;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
      "@p ld.global.L2::cache_hint.f64 %0, [%1], %3;\n\t}"
      : "+d"(v)
      : "l"(p), "r"((unsigned)ok), "l"(policy));
  return v;
}
__device__ __forceinline__ void stg_hint(double* p, double v, bool ok, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
      "@p st.global.L2::cache_hint.f64 [%0], %1, %3;\n\t}" ::"l"(p),
      "d"(v), "r"((unsigned)ok), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mbar_init_n(uint64_t* mbar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(mbar))),
               "r"(count)
               : "memory");
}
// Warp-specialised Wt_2 / staging phase: measured at C5 (RP 56) 41.1 -> 38.9 ms per
// launch; at RP <= 40 (C3) the split Wt_2 partials it gives up were worth more.
template <int RP, bool TIO>
__host__ __device__ constexpr bool pass2_ws() {
  return (!TIO || PASD_P2_TIL) && PASD_P2_WS && RP >= 48 && !pass2_bulk<TIO>();
}

// RP = common padded rank (multiple of 8, >= every R_n); rows r >= R_n of each
// mode's operands are zero, so padding changes no result.
// EL = storage type of the element streams T, E, D, Y_n (double; float in the
// fp32 mode, PASD_FLAG_FP32): loaded into fp64 registers, every operation below
// in fp64, rounded to EL on store.
template <int RP, bool TIO, class EL = double>
__global__ void __launch_bounds__(P2_THREADS, 1) k_pass2_fused(const Pass2Args a, const Ctl* ctl,
                                                                const __grid_constant__ P2Tmaps tm) {
  static_assert(!TIO || sizeof(EL) == 8, "TMA element bricks are float64");
  if (ctl->done) return;
  using L = P2LayoutE<RP, TIO, EL>;
  constexpr int KS = RP / 4;   // k-steps of the Z products
  constexpr int NT1 = RP / 8;  // n-tiles of the Wt_1 product
  constexpr int MT = L::RM / 16;
  constexpr bool WS = pass2_ws<RP, TIO>();  // warp-specialised Wt_2 / staging phase
  constexpr bool TIL = L::TIL;              // TMA loads only (see PASD_P2_TIL)
  constexpr bool TILS = TIL && PASD_P2_TIL == 2;  // ... and TMA stores of E, Y_n from the same bricks
  constexpr bool BS = pass2_bulk<TIO>();          // slices by cp.async.bulk from the tiled copies (PASD_P2_BULK)
  constexpr unsigned kBytesA1 = 64u * L::LD1 * 8u, kBytesA2 = (unsigned)RP * L::LD2 * 8u,
                     kBytesA3 = (unsigned)RP * L::LD3 * 8u, kBytesU2 = 8u * L::LDU * 8u;
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
  double* G2s = sm + L::oG2;
  double* G3s = sm + L::oG3;
  double* X2s = sm + L::oX2;
  constexpr bool DW2 = L::DW2;
  double* red = sm + L::oRed;
  // TIO bricks: [0] T -> E, [1] Y_1, [2] Y_2, [3] Y_3 (layout B), [4] D, [5] D (layout B)
  double* brk = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sm + L::oBrick) + 1023) & ~uintptr_t(1023));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 56);
  unsigned mph = 0;  // mbarrier phase parity of the next element-brick load
  // BS: "step slices landed" (3 arrivals: A_3, A_1, UM_2 copies), "pencil slice landed" (A_2), and the
  // per-slice release counters (8 warps each; the last one to arrive issues the next step's copy)
  uint64_t* full_s = reinterpret_cast<uint64_t*>(red + 57);
  uint64_t* full_p = reinterpret_cast<uint64_t*>(red + 58);
  int* rel3 = reinterpret_cast<int*>(red + 59);
  int* rel1 = rel3 + 1;
  unsigned phs = 0, php = 0;
  const uint64_t l2pol = (BS && PASD_P2_L2HINT) ? l2_policy_evict_last() : 0;
  constexpr bool EH = BS && PASD_P2_EHINT && sizeof(EL) == 8;  // element streams with an evict_first policy
  const uint64_t l2ef = EH ? l2_policy_evict_first() : 0;
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

  // Wt_2 partials: one per K-half (no exchange after the Wt_2 product) when the
  // solver sized them so (small I_2 R_2: they stay in L2), else one per CTA
  // with the two K-halves exchanged through shared memory.
  const bool w2s = a.nw2 == 2 * (int)gridDim.x;
  const int NW2 = w2s ? 2 : 1;
  double* W2c = a.W2part + (int64_t)blockIdx.x * NW2 * I2 * R2;  // per-CTA Wt_2 partial(s)
  for (int64_t idx = tid; idx < NW2 * I2 * R2; idx += P2_THREADS) W2c[idx] = 0.0;
  // m-tile and K-half of the Wt_2 (mt) / Wt_3 (mt3) products.  The two warps of a K-half pair are any two
  // warps; rotating the tiles puts the last m-tile of the four (product, K-half) items on four different
  // schedulers (warp w issues on scheduler w & 3).
  constexpr bool HALF = PASD_P2_HALF && (L::RM - RP == 8) && !(TIO && !TIL) && !WS;
  const int kh = w >> 2;
  const int mt = !HALF ? (w & 3) : ((w + kh + 2) & 3);
  const int mt3 = !HALF ? (w & 3) : ((w + kh) & 3);
  double* W2k = W2c + (w2s ? (int64_t)kh * I2 * R2 : 0);
  // zero padding rows once (never overwritten by the staging copies)
  for (int idx = tid; idx < (RP - R2) * 128; idx += P2_THREADS) A2s[(R2 + idx / 128) * L::LD2 + (idx & 127)] = 0.0;
  for (int idx = tid; idx < (RP - R3) * 128; idx += P2_THREADS) A3s[(R3 + idx / 128) * L::LD3 + (idx & 127)] = 0.0;
  for (int idx = tid; idx < L::oBrick - L::oU1; idx += P2_THREADS) U1s[idx] = 0.0;  // UM rows, exchange buffers
  if (BS) __syncthreads();  // (the zero fill above covers `red`)
  if (TIO && tid == 0) {
    mbar_init(mbar);
  }
  if (BS && tid == 0) {
    mbar_init_n(full_s, 3);
    mbar_init_n(full_p, 1);
    *rel3 = 0;
    *rel1 = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // TIO: the next brick's T, Y_1..3 (after the previous stores have read the bricks)
  auto load_bricks = [&](int64_t i1o_, int64_t i2o_, int64_t i3o_) {
    if (TIL) {  // all four in the A layout; their slots are free once the elementwise phase has read them
      if (tid == 0 && PASD_P2_PROBE != 7) {
        if (TILS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // ... and the stores have left
        mbar_expect(mbar, 4u * P2_BRICK * sizeof(double));
        const int c0 = (int)i1o_, c1 = (int)i2o_, c2 = (int)i3o_;
        tma_load3(brk, &tm.t, mbar, c0, c1, c2);
        tma_load3(brk + P2_BRICK, &tm.y1, mbar, c0, c1, c2);
        tma_load3(brk + 2 * P2_BRICK, &tm.y2, mbar, c0, c1, c2);
        tma_load3(brk + 3 * P2_BRICK, &tm.y3a, mbar, c0, c1, c2);
      }
    } else if (TIO && tid == 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_expect(mbar, 4u * P2_BRICK * sizeof(double));
      const int c0 = (int)i1o_, c1 = (int)i2o_, c2 = (int)i3o_;
      tma_load3(brk, &tm.t, mbar, c0, c1, c2);
      tma_load3(brk + P2_BRICK, &tm.y1, mbar, c0, c1, c2);
      tma_load3(brk + 2 * P2_BRICK, &tm.y2, mbar, c0, c1, c2);
      tma_load3(brk + 3 * P2_BRICK, &tm.y3b, mbar, c0, c2, c1);
    }
  };

  double worst[3] = {0.0, 0.0, 0.0};
  double gsq[3] = {0.0, 0.0, 0.0};
  int bad = 0;
  const int64_t S12 = I1 * I2;
#if PASD_P2_TIMING
  unsigned long long ph_acc[12] = {};
  long long ph_t = clock64();
#endif
  const int ksz = (max(R1, max(R2, R3)) + 3) / 4;  // Z k-steps that touch a nonzero rank row
  const bool al1 = (I1 % 2) == 0;  // 16-byte aligned rows of 16 consecutive i1

  // Work items: pencil x i2 segment (see the solver's choice of nseg).
  const int64_t seg_len = (((I2 + P2_B2 - 1) / P2_B2 + a.nseg - 1) / a.nseg) * P2_B2;
  for (int item = blockIdx.x; item < a.npencils * a.nseg; item += gridDim.x) {
    const int seg = item / a.npencils, lin = item - seg * a.npencils;
    const int64_t i2b = seg * seg_len, i2e = imin64(I2, i2b + seg_len);
    // Banded pencil order: the ~gridDim pencils processed concurrently form a
    // ~12 x 12 patch of (i1-block, i3-block), so the A_3 slices (shared along
    // i3) and A_1 slices (shared along i1) they stage each step are L2 hits.
    int ib1, ib3;
    {
      const int BW = PASD_P2_BW;
      const int band = lin / (BW * a.n3b), lin_in = lin - band * BW * a.n3b;
      const int bw = min(BW, a.n1b - band * BW);
      ib1 = band * BW + lin_in % bw;
      ib3 = lin_in / bw;
    }
    const int pen = ib1 + a.n1b * ib3 + a.npencils * seg;  // index of the Wt_1 / Wt_3 partials
    const int64_t i1o = (int64_t)ib1 * P2_B1, i3o = (int64_t)ib3 * P2_B3;
    const int nv1 = (int)imin64(16, I1 - i1o);
    if (i2b >= i2e) {  // empty i2 segment (the segment count does not divide the steps): zero partials, no staging
      for (int idx = tid; idx < 16 * R1; idx += P2_THREADS) a.W1p[(int64_t)pen * 16 * R1 + idx] = 0.0;
      for (int idx = tid; idx < 8 * R3; idx += P2_THREADS) a.W3p[(int64_t)pen * 8 * R3 + idx] = 0.0;
      continue;
    }
    const int nbc1 = (nv1 - 2 * (tid & 7)) >= 2 ? 16 : ((nv1 - 2 * (tid & 7)) == 1 ? 8 : 0);  // A_3 chunk bytes
    __syncthreads();  // previous pencil fully done with shared memory
    load_bricks(i1o, i2b, i3o);
    // BS: one bulk copy per slice from the tiled copies (issued by a single thread; the proxy fence orders
    // the generic-proxy accesses of the slice before the asynchronous write)
    auto bulk = [&](double* dst, const double* src, unsigned bytes, uint64_t* mb) {
      if (PASD_P2_L2HINT)
        bulk_load_hint(dst, src, bytes, mb, l2pol);
      else
        bulk_load(dst, src, bytes, mb);
    };
    auto issue_a3 = [&](int64_t i2o_) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(full_s, kBytesA3);
      bulk(A3s, a.At3 + ((int64_t)ib1 * a.n2b + i2o_ / P2_B2) * (RP * L::LD3), kBytesA3, full_s);
    };
    auto issue_a1 = [&](int64_t i2o_) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(full_s, kBytesA1);
      bulk(A1s, a.At1 + ((int64_t)ib3 * a.n2b + i2o_ / P2_B2) * (64 * L::LD1), kBytesA1, full_s);
    };
    auto issue_u2 = [&](int64_t i2o_) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(full_s, kBytesU2);
      bulk(U2s, a.U2t + (i2o_ / P2_B2) * (8 * L::LDU), kBytesU2, full_s);
    };
    // ---- pencil-resident: A_2 slice (I1, R2, I3 layout), UM_1 rows, UM_3 rows ----
    if constexpr (BS) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(full_p, kBytesA2);
        bulk_load(A2s, a.At2 + ((int64_t)ib3 * a.n1b + ib1) * (RP * L::LD2), kBytesA2, full_p);  // read once
        issue_a3(i2b);
        issue_a1(i2b);
        issue_u2(i2b);
      }
    } else {
      for (int l3 = 0; l3 < 8; ++l3) {
        const bool in3 = i3o + l3 < I3;
        stage_rows16(A2s + 16 * l3, L::LD2, m2.A + i1o + I1 * (int64_t)R2 * (i3o + l3), I1, R2, in3 ? nv1 : 0, al1, m2.A);
      }
    }
    for (int idx = tid; idx < 16 * R1; idx += P2_THREADS) {
      const int l1 = idx & 15, r = idx >> 4;
      const bool v = l1 < nv1;
      cp_async8(U1s + l1 * L::LDU + r, v ? m1.UM + m1.ioff + i1o + l1 + m1.Ifull * r : m1.UM, v);
    }
    for (int idx = tid; idx < 8 * R3; idx += P2_THREADS) {
      const int l3 = idx & 7, r = idx >> 3;
      const bool v = i3o + l3 < I3;
      cp_async8(U3s + l3 * L::LDU + r, v ? m3.UM + m3.ioff + i3o + l3 + m3.Ifull * r : m3.UM, v);
    }
    double w1acc[NT1][4];
#pragma unroll
    for (int j = 0; j < NT1; ++j) w1acc[j][0] = w1acc[j][1] = w1acc[j][2] = w1acc[j][3] = 0.0;
    double w3acc[4] = {0.0, 0.0, 0.0, 0.0};  // Wt_3^T m-tile (w & 3), K-half (w >> 2)

    // per-step staging (issued one step ahead, overlapping the Wt_2 products).
    // Per-thread source/destination bases are fixed along the pencil; a step
    // only advances them by 8 i2.
    const int n3v = (int)imin64(8, I3 - i3o);  // valid i3 of the pencil
    auto stage_a1 = [&](int64_t i2o, double* A1b, int wv, int nwv) {
      for (int l2w = wv; l2w < 8; l2w += nwv) {  // A_1 (R1, I2, I3 layout): warp -> columns (l2, l3 = k); lane -> r pair
        const bool c2ok = i2o + l2w < I2;
        const char* gp = reinterpret_cast<const char*>(m1.A + (int64_t)R1 * ((i2o + l2w) + I2 * i3o));
        const int64_t kst = 8 * (int64_t)R1 * I2;  // bytes to the next l3
        const unsigned sp = smem_u32(A1b + l2w * L::LD1);
        if ((R1 & 1) == 0) {
          if (lane < RP / 2) {
            const int r = 2 * lane;
            const bool rok = c2ok && r < R1;
            gp += 16 * lane;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const bool ok = rok && k < n3v;
              cp16z(sp + 8 * (k * 8 * L::LD1 + r), ok ? (const void*)gp : (const void*)m1.A, ok);
              gp += kst;
            }
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            if (r < RP) {
              const bool rok = c2ok && r < R1;
              const char* gq = gp + 8 * r;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const bool ok = rok && k < n3v;
                cp8s(sp + 8 * (k * 8 * L::LD1 + r), ok ? (const void*)gq : (const void*)m1.A, ok ? 8 : 0);
                gq += kst;
              }
            }
          }
        }
      }
    };
    // u = thread index within the NT issuing threads (NT = 256: the whole CTA,
    // 128: the staging warps of the warp-specialised Wt_2 phase)
    auto stage_a3u2 = [&](int64_t i2o, int u, auto NTc) {
      constexpr int NT = decltype(NTc)::value, RS = NT / 64;
      {  // A_3 (I1, I2, R3 layout): rows (r, l2) of 16 consecutive i1; thread ->
         // 16-byte chunk c, l2, rows r = r0 + RS k (padding rows stay zero)
        const int c = u & 7, l2 = (u >> 3) & 7, r0 = u >> 6;
        const bool ok2 = i2o + l2 < I2;
        const int nb = ok2 ? nbc1 : 0;
        const char* gp = reinterpret_cast<const char*>(nb ? m3.A + i1o + 2 * c + I1 * (i2o + l2) + S12 * (int64_t)r0 : m3.A);
        const int64_t gst = nb ? 8 * RS * S12 : 0;  // RS rows r
        const unsigned sp = smem_u32(A3s + r0 * L::LD3 + 16 * l2 + 2 * c);
        if (al1) {  // even I1: every 16-byte chunk is wholly inside or outside
#pragma unroll
          for (int k = 0; k < (RP + RS - 1) / RS; ++k) {
            if (r0 + RS * k < R3) cp16z(sp + 8 * RS * k * L::LD3, gp, nb != 0);
            gp += gst;
          }
        } else {
          const int n0 = nb >= 8 ? 8 : 0, n1 = nb >= 16 ? 8 : 0;
#pragma unroll
          for (int k = 0; k < (RP + RS - 1) / RS; ++k) {
            if (r0 + RS * k < R3) {
              cp8s(sp + 8 * RS * k * L::LD3, n0 ? (const void*)gp : (const void*)m3.A, n0);
              cp8s(sp + 8 * RS * k * L::LD3 + 8, n1 ? (const void*)(gp + 8) : (const void*)m3.A, n1);
            }
            gp += gst;
          }
        }
      }
      {  // UM_2 rows of the step: thread -> (l2, r = u / 8 + (NT / 8) k)
        const int l2 = u & 7;
        const bool v = i2o + l2 < I2;
        const double* src = m2.UM + m2.ioff + i2o + l2;
#pragma unroll
        for (int k = 0; k < (RP + NT / 8 - 1) / (NT / 8); ++k) {
          const int r = (u >> 3) + (NT / 8) * k;
          if (r < R2) cp8z(smem_u32(U2s + l2 * L::LDU + r), v ? (const void*)(src + m2.Ifull * r) : (const void*)m2.UM, v);
        }
      }
    };
    using All = std::integral_constant<int, P2_THREADS>;
    using Half = std::integral_constant<int, P2_THREADS / 2>;
    // this thread's 4 elements: (i1 = g, g+8) x (i2 = 2t, 2t+1) at i3 = w
    double tv[4], yv[3][4];
    bool inb[4];
    int64_t off[4];
    auto load_elems = [&](int64_t i2o) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t i1 = i1o + g + 8 * (q >> 1), i2 = i2o + 2 * t + (q & 1), i3 = i3o + w;
        inb[q] = i1 < I1 && i2 < I2 && i3 < I3;
        off[q] = i1 + I1 * i2 + S12 * i3;
        const bool ld = inb[q] && PASD_P2_PROBE != 7;
        if constexpr (EH) {
          tv[q] = ldg_hint(reinterpret_cast<const double*>(T) + off[q], ld, l2ef);
#pragma unroll
          for (int n = 0; n < 3; ++n) yv[n][q] = ldg_hint(reinterpret_cast<const double*>(Yp[n]) + off[q], ld, l2ef);
        } else {
          tv[q] = ld ? T[off[q]] : 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) yv[n][q] = ld ? (double)Yp[n][off[q]] : 0.0;
        }
      }
    };
    // PASD_P2_EPF: this thread's 8 copies of a step's T, Y_1..3 brick (stream ts,
    // row (l2, l3), 16-byte chunk c); issued right after the previous step's
    // elementwise phase, so they land during its Wt products and the next Z.
    double* El = sm + L::oBrick;
    auto stage_elems = [&](int64_t i2o, int u, auto NTc) {
      constexpr int NT = decltype(NTc)::value;
      const int c = u & 7;
      const bool cok = 2 * c < nv1;
#pragma unroll
      for (int k = 0; k < 4 * P2_BRICK / 2 / NT; ++k) {
        const int idx = u + NT * k;
        const int row = (idx >> 3) & 63, ts = idx >> 9;
        const int l2 = row & 7, l3 = row >> 3;
        const bool ok = cok && i2o + l2 < I2 && i3o + l3 < I3;
        const EL* base = ts == 0 ? T : Yp[ts - 1];
        const EL* src = ok ? base + i1o + 2 * c + I1 * (i2o + l2) + S12 * (i3o + l3) : base;
        const unsigned dst = smem_u32(El + ts * P2_BRICK + 16 * row + 2 * (c ^ (l2 & 6)));
        if (al1) {
          cp16z(dst, src, ok);
        } else {
          const bool ok1 = ok && 2 * c + 1 < nv1;
          cp8z(dst, src, ok);
          cp8z(dst + 8, ok1 ? (const void*)(src + 1) : (const void*)base, ok1);
        }
      }
    };
    if constexpr (!BS) {
      stage_a1(i2b, A1s, w, 8);
      stage_a3u2(i2b, tid, All{});
    }
    if (L::EPF) stage_elems(i2b, tid, All{});

    double d2old[4] = {0, 0, 0, 0};  // DW2: deferred Wt_2 product of the previous step
    double d2acc[4][4] = {};
    auto w2_quarter = [&](int qq, const double* G2b) {
      if (mt < MT && PASD_P2_PROBE != 1 && PASD_P2_PROBE != 3) {
        const double* rowa = A2s + (16 * mt + g) * L::LD2 + 64 * kh;
        const double* rowb = rowa + 8 * L::LD2;
#pragma unroll
        for (int ks = 4 * qq; ks < 4 * qq + 4; ++ks) {
          const int k = 64 * kh + 4 * ks + t;
          dmma(d2acc[ks & 3], rowa[4 * ks + t], rowb[4 * ks + t], G2b[g2x(k & 15, g, k >> 4)]);
        }
      }
    };
    // K-half sum in the order of the undeferred product, then (after a barrier) the partial update
    auto w2_sum = [&]() {
#pragma unroll
      for (int q = 0; q < 4; ++q) d2acc[0][q] += (d2acc[1][q] + d2acc[2][q]) + d2acc[3][q];
      if (!w2s && kh == 1 && mt < MT) {
#pragma unroll
        for (int q = 0; q < 4; ++q) X2s[(mt * 32 + lane) * 4 + q] = d2acc[0][q];
      }
    };
    auto w2_store = [&](int64_t i2base) {
      if (mt < MT && (w2s || kh == 0)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 16 * mt + g + 8 * (q >> 1);
          const int64_t i2 = i2base + 2 * t + (q & 1);
          const double v = w2s ? d2acc[0][q] : (d2acc[0][q] + X2s[(mt * 32 + lane) * 4 + q]);
          if (r < R2 && i2 < I2) W2k[i2 * R2 + r] = d2old[q] + v;
        }
      }
    };

    for (int64_t i2o = i2b; i2o < i2e; i2o += P2_B2) {
      const bool more = i2o + P2_B2 < i2e;
      const double* A1c = A1s;
      P2T(0);  // 0: pencil setup / loop top
      constexpr int ELD = BS ? PASD_P2_ELD : 0;
      if (!TIO && !L::EPF && (ELD == 0 || i2o == i2b)) load_elems(i2o);  // this step's T, Y: in flight while the staging lands and Z runs
                                             // (measured 2 ms faster at C5 than prefetching them a step ahead)
      cp_async_wait_all();
      if constexpr (BS) {
        mbar_wait(full_s, phs);  // this step's A_1, A_3, UM_2 slices
        phs ^= 1;
        if (i2o == i2b) {
          mbar_wait(full_p, php);  // the pencil's A_2 slice
          php ^= 1;
        }
      }
      P2T(1);  // 1: element-load issue + staging wait
      __syncthreads();  // step data staged; previous step's smem consumers done
      P2T(2);  // 2: barrier A
      // ---- Z products (6 independent accumulator chains) ----
      double z1[4] = {0, 0, 0, 0}, z2[4] = {0, 0, 0, 0}, z3[4] = {0, 0, 0, 0};
      {
        double y1[4] = {0, 0, 0, 0}, y2[4] = {0, 0, 0, 0}, y3[4] = {0, 0, 0, 0};
        // k-steps past max R_n only multiply zero padding: max R_n > RP - 8, so
        // ksz is KS - 1 or KS.  The first KS - 1 run as straight-line code (no
        // per-step branch, so the compiler can hoist the next step's operand
        // loads above this step's DMMAs), the last one behind a single test.
        auto zstep = [&](int ks) {
          const int k = 4 * ks + t;
          double(&c1)[4] = (ks & 1) ? y1 : z1;
          double(&c2)[4] = (ks & 1) ? y2 : z2;
          double(&c3)[4] = (ks & 1) ? y3 : z3;
          const int kc = PASD_P2_PROBE == 5 ? t : k;  // probe 5: pencil-constant operands loaded once
          dmma(c1, U1s[g * L::LDU + kc], U1s[(g + 8) * L::LDU + kc], A1c[(g + 8 * w) * L::LD1 + k]);
          dmma(c2, A2s[kc * L::LD2 + g + 16 * w], A2s[kc * L::LD2 + g + 8 + 16 * w], U2s[g * L::LDU + k]);
          dmma(c3, A3s[k * L::LD3 + g + 16 * w], A3s[k * L::LD3 + g + 8 + 16 * w], U3s[g * L::LDU + kc]);
        };
        if (PASD_P2_ZPIPE && PASD_P2_PROBE != 2 && PASD_P2_PROBE != 3 && PASD_P2_PROBE != 5) {
          // two operand sets; loads of k-step s + 1, then the DMMAs of k-step s
          const unsigned pu1 = smem_u32(U1s + g * L::LDU + t), pa1 = smem_u32(A1c + (g + 8 * w) * L::LD1 + t);
          const unsigned pa2 = smem_u32(A2s + t * L::LD2 + g + 16 * w), pu2 = smem_u32(U2s + g * L::LDU + t);
          const unsigned pa3 = smem_u32(A3s + t * L::LD3 + g + 16 * w), pu3 = smem_u32(U3s + g * L::LDU + t);
          double o[2][9];
          auto zload = [&](int ks, double(&d)[9]) {
            d[0] = lds_f64(pu1 + 32 * ks);
            d[1] = lds_f64(pu1 + 32 * ks + 64 * L::LDU);
            d[2] = lds_f64(pa1 + 32 * ks);
            d[3] = lds_f64(pa2 + 32 * ks * L::LD2);
            d[4] = lds_f64(pa2 + 32 * ks * L::LD2 + 64);
            d[5] = lds_f64(pu2 + 32 * ks);
            d[6] = lds_f64(pa3 + 32 * ks * L::LD3);
            d[7] = lds_f64(pa3 + 32 * ks * L::LD3 + 64);
            d[8] = lds_f64(pu3 + 32 * ks);
          };
          auto zmma = [&](int ks, const double(&d)[9]) {
            dmma((ks & 1) ? y1 : z1, d[0], d[1], d[2]);
            dmma((ks & 1) ? y2 : z2, d[3], d[4], d[5]);
            dmma((ks & 1) ? y3 : z3, d[6], d[7], d[8]);
          };
          const bool lastk = ksz == KS;  // the last k-step touches a nonzero rank row
          zload(0, o[0]);
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            if (ks + 1 < KS - 1) {
              zload(ks + 1, o[(ks + 1) & 1]);
            } else if (ks + 1 == KS - 1) {
              if (lastk) zload(ks + 1, o[(ks + 1) & 1]);
            }
            if (PASD_P2_ZPIPE == 2) __syncwarp();  // keeps ptxas from hoisting the loads of later k-steps above this point
            if (ks < KS - 1) {
              zmma(ks, o[ks & 1]);
            } else if (lastk) {
              zmma(ks, o[ks & 1]);
            }
          }
        } else if (PASD_P2_PROBE != 2 && PASD_P2_PROBE != 3) {
          if constexpr (RP >= 48) {
            // at RP >= 48 the hoisted loads push the kernel to 254 registers and the
            // Z phase measured slower (C5: 4.5 vs 4.25 k cycles per step), as did an
            // explicit two-stage operand pipeline in a rolled loop (5.2 k): keep one
            // test per k-step there, which pins each step's loads next to its DMMAs
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              if (ks >= ksz) break;
              zstep(ks);
            }
          } else {  // C3 / C4: 2.13 -> 2.10 / 2.08 -> 2.03 ms per launch
#pragma unroll
            for (int ks = 0; ks < KS - 1; ++ks) zstep(ks);
            if (ksz == KS) zstep(KS - 1);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          z1[q] += y1[q];
          z2[q] += y2[q];
          z3[q] += y3[q];
        }
      }
      Z3s[zx(g, w, 2 * t)] = z3[0];
      Z3s[zx(g, w, 2 * t + 1)] = z3[1];
      Z3s[zx(g + 8, w, 2 * t)] = z3[2];
      Z3s[zx(g + 8, w, 2 * t + 1)] = z3[3];
      P2T(3);  // 3: Z products
      __syncthreads();
      P2T(4);  // 4: barrier B
      if (BS && more && tid == 0) issue_u2(i2o + P2_B2);  // UM_2 rows are read by the Z products only
      // DW2: the previous step's Wt_2 products (m-tile mt, K-half kh) run inside this step's elementwise
      // phase, a quarter of the K range after each of the thread's four elements.  On a pencil's first
      // step they multiply stale G_2 values and the result is dropped.
      const int gpar = (int)((i2o - i2b) >> 3) & 1;  // this step's G_2 buffer; the previous step's is the other
      double* G2w = G2s + (DW2 ? gpar * (8 * 160) : 0);
      const double* G2r = G2s + (DW2 ? (gpar ^ 1) * (8 * 160) : 0);
      const bool w2prev = DW2 && i2o > i2b && mt < MT;
#pragma unroll
      for (int q = 0; q < 4; ++q) d2old[q] = d2acc[0][q] = d2acc[1][q] = d2acc[2][q] = d2acc[3][q] = 0.0;
      if (w2prev && (w2s || kh == 0)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 16 * mt + g + 8 * (q >> 1);
          const int64_t i2 = i2o - P2_B2 + 2 * t + (q & 1);
          if (r < R2) d2old[q] = W2k[i2 * R2 + r];
        }
      }
      // ---- elementwise (reference op order, no FMA contraction) ----
      double g1v[4];
      if constexpr (!TIO) {
        int64_t offc[4];
        bool inc[4];
        if (L::EPF) {  // this step's T, Y from the staged bricks
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int l1 = g + 8 * (q >> 1), l2 = 2 * t + (q & 1);
            const int64_t i1 = i1o + l1, i2 = i2o + l2, i3 = i3o + w;
            inb[q] = i1 < I1 && i2 < I2 && i3 < I3;
            off[q] = i1 + I1 * i2 + S12 * i3;
            const int e = ex(l1, l2, w);
            tv[q] = El[e];
#pragma unroll
            for (int n = 0; n < 3; ++n) yv[n][q] = El[(1 + n) * P2_BRICK + e];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int l1 = g + 8 * (q >> 1), l2 = 2 * t + (q & 1);
          const double zz[3] = {z1[q], z2[q], Z3s[zx(l1, l2, w)]};
          const double tt = tv[q];
          if (PASD_P2_PROBE == 4) {  // timing probe: loads / stores / exchange only
            if (inb[q]) {
              for (int n = 0; n < 3; ++n) Yp[n][off[q]] = (EL)(yv[n][q] + zz[n]);
              Enew[off[q]] = (EL)tt;
              Dp[off[q]] = (EL)tt;
            }
            g1v[q] = tt;
            G2w[g2x(l1, l2, w)] = yv[1][q];
            G3s[g3x(l1, l2, w)] = yv[2][q];
            if constexpr (DW2) w2_quarter(q, G2r);
            continue;
          }
          double zt[3], h = 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            zt[n] = __dsub_rn(tt, zz[n]);
            h = __dadd_rn(h, __dadd_rn(zt[n], __dmul_rn(yv[n][q], inv_mu)));  // pasd.cpp:202
          }
          const double e = PASD_P2_SOFTSEL ? soft_sel(__dmul_rn(h, inv_n), tau) : soft(__dmul_rn(h, inv_n), tau);  // pasd.cpp:208
          double gn[3];
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            const double r = __dsub_rn(zt[n], e);                       // pasd.cpp:220
            const double ynew = __dadd_rn(yv[n][q], __dmul_rn(mu, r));  // pasd.cpp:221
#if PASD_P2_SOFTSEL
            // entries outside the tensor have T = Y_n = Z_n = 0 (zero-filled loads, zero slice entries), so
            // r = 0 there: the residual / NaN reductions need no guard, and the only guarded statement
            // left is the store (one predicated STG, no branch: the four elements' chains interleave)
            const double ar = fabs(r);
            worst[n] = ar > worst[n] ? ar : worst[n];
            bad |= !isfinite(r);
            if (inb[q] && PASD_P2_PROBE != 6) Yp[n][off[q]] = (EL)ynew;
#else
            if (inb[q]) {
              const double ar = fabs(r);
              if (ar > worst[n]) worst[n] = ar;
              bad |= !isfinite(r);
              if (!EH && PASD_P2_PROBE != 6) Yp[n][off[q]] = (EL)ynew;
            }
            if constexpr (EH) stg_hint(reinterpret_cast<double*>(Yp[n]) + off[q], ynew, inb[q] && PASD_P2_PROBE != 6, l2ef);
#endif
            gn[n] = inb[q] ? g_elem(tt, e, ynew, inv_mu_next) : 0.0;  // next G_n
            gsq[n] = fma(gn[n], gn[n], gsq[n]);
          }
          if constexpr (EH) {
            stg_hint(reinterpret_cast<double*>(Enew) + off[q], e, inb[q] && PASD_P2_PROBE != 6, l2ef);
            stg_hint(reinterpret_cast<double*>(Dp) + off[q], __dsub_rn(tt, e), inb[q] && PASD_P2_PROBE != 6, l2ef);
          } else if (inb[q] && PASD_P2_PROBE != 6) {
            Enew[off[q]] = (EL)e;
            Dp[off[q]] = (EL)__dsub_rn(tt, e);  // next pass 1 reads D = T - E
          }
          g1v[q] = gn[0];
          G2w[g2x(l1, l2, w)] = gn[1];
          G3s[g3x(l1, l2, w)] = gn[2];
          offc[q] = off[q];
          inc[q] = inb[q];
          if constexpr (DW2) w2_quarter(q, G2r);
        }
        if constexpr (DW2) w2_sum();
        (void)offc;
        (void)inc;
      } else {
        // T, Y_n from the TMA bricks; E, D, Y_n written back in place.  Entries
        // outside the tensor arrive as zeros (TMA fill) with zero Z, so they
        // produce zeros everywhere and the stores clip them.
        if (!(TIL && PASD_P2_PROBE == 7)) mbar_wait(mbar, mph);
        mph ^= 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int l1 = g + 8 * (q >> 1), l2 = 2 * t + (q & 1);
          const int pa = swzA(l1, l2, w), pb = swzB(l1, l2, w);
          if constexpr (TIL) {
            // loads from the bricks, plain stores
            const int64_t i1 = i1o + l1, i2 = i2o + l2, i3 = i3o + w;
            const bool in = i1 < I1 && i2 < I2 && i3 < I3;
            const int64_t o = i1 + I1 * i2 + S12 * i3;
            const double zz[3] = {z1[q], z2[q], Z3s[zx(l1, l2, w)]};
            const double tt = brk[pa];
            const double yq[3] = {brk[P2_BRICK + pa], brk[2 * P2_BRICK + pa], brk[3 * P2_BRICK + pa]};
            double zt[3], h = 0.0;
#pragma unroll
            for (int n = 0; n < 3; ++n) {
              zt[n] = __dsub_rn(tt, zz[n]);
              h = __dadd_rn(h, __dadd_rn(zt[n], __dmul_rn(yq[n], inv_mu)));  // pasd.cpp:202
            }
            const double e = soft(__dmul_rn(h, inv_n), tau);  // pasd.cpp:208
            double gn[3];
#pragma unroll
            for (int n = 0; n < 3; ++n) {
              const double r = __dsub_rn(zt[n], e);                    // pasd.cpp:220
              const double ynew = __dadd_rn(yq[n], __dmul_rn(mu, r));  // pasd.cpp:221
              if (in) {
                const double ar = fabs(r);
                if (ar > worst[n]) worst[n] = ar;
                bad |= !isfinite(r);
                if (PASD_P2_PROBE != 6 && !TILS) Yp[n][o] = (EL)ynew;
              }
              gn[n] = in ? g_elem(tt, e, ynew, inv_mu_next) : 0.0;  // next G_n
              gsq[n] = fma(gn[n], gn[n], gsq[n]);
              if (TILS) brk[(1 + n) * P2_BRICK + pa] = ynew;  // (entries outside the tensor are clipped by the store)
            }
            if (TILS) brk[pa] = e;
            if (in && PASD_P2_PROBE != 6) {
              if (!TILS) Enew[o] = (EL)e;
              Dp[o] = (EL)__dsub_rn(tt, e);  // next pass 1 reads D = T - E
            }
            g1v[q] = gn[0];
            G2s[g2x(l1, l2, w)] = gn[1];
            G3s[g3x(l1, l2, w)] = gn[2];
            (void)pb;
            continue;
          }
          const double zz[3] = {z1[q], z2[q], Z3s[zx(l1, l2, w)]};
          const double tt = brk[pa];
          const double yq[3] = {brk[P2_BRICK + pa], brk[2 * P2_BRICK + pa], brk[3 * P2_BRICK + pb]};
          double zt[3], h = 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            zt[n] = __dsub_rn(tt, zz[n]);
            h = __dadd_rn(h, __dadd_rn(zt[n], __dmul_rn(yq[n], inv_mu)));  // pasd.cpp:202
          }
          const double e = soft(__dmul_rn(h, inv_n), tau);  // pasd.cpp:208
          const double dq = __dsub_rn(tt, e);              // D = T - E (next pass 1)
          double gn[3];
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            const double r = __dsub_rn(zt[n], e);                  // pasd.cpp:220
            const double ynew = __dadd_rn(yq[n], __dmul_rn(mu, r));  // pasd.cpp:221
            const double ar = fabs(r);
            if (ar > worst[n]) worst[n] = ar;
            bad |= !isfinite(r);
            gn[n] = __dadd_rn(dq, __dmul_rn(ynew, inv_mu_next));  // = g_elem(tt, e, ynew, inv_mu_next)
            gsq[n] = fma(gn[n], gn[n], gsq[n]);
            brk[(1 + n) * P2_BRICK + (n == 2 ? pb : pa)] = ynew;
          }
          brk[pa] = e;
          brk[4 * P2_BRICK + pa] = dq;
          brk[5 * P2_BRICK + pb] = dq;
          g1v[q] = gn[0];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // bricks -> TMA (async proxy)
      }
      P2T(5);  // 5: elementwise (incl. waiting for this step's element loads)
      __syncthreads();  // G exchange / bricks complete
      P2T(6);  // 6: barrier C
      if (w2prev) w2_store(i2o - P2_B2);
      if (L::EPF && !WS && more) stage_elems(i2o + P2_B2, tid, All{});  // the element bricks are consumed: next step's
      if (TIL && !TILS && more) load_bricks(i1o, i2o + P2_B2, i3o);  // the bricks are consumed: next step's T, Y_n
      if (TILS && tid == 0) {  // E, Y_1..3 of this brick leave from the bricks they arrived in
        const int c0 = (int)i1o, c1 = (int)i2o, c2 = (int)i3o;
        tma_store3(ctl->ecur ? &tm.e0 : &tm.e1, brk, c0, c1, c2);
        tma_store3(&tm.y1, brk + P2_BRICK, c0, c1, c2);
        tma_store3(&tm.y2, brk + 2 * P2_BRICK, c0, c1, c2);
        tma_store3(&tm.y3a, brk + 3 * P2_BRICK, c0, c1, c2);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (TIO && !TIL && tid == 0) {  // E, Y_1..3, D of this brick: TMA tensor stores
        const int c0 = (int)i1o, c1 = (int)i2o, c2 = (int)i3o;
        tma_store3(ctl->ecur ? &tm.e0 : &tm.e1, brk, c0, c1, c2);
        tma_store3(&tm.y1, brk + P2_BRICK, c0, c1, c2);
        tma_store3(&tm.y2, brk + 2 * P2_BRICK, c0, c1, c2);
        tma_store3(&tm.y3b, brk + 3 * P2_BRICK, c0, c2, c1);
        tma_store3(&tm.d, brk + 4 * P2_BRICK, c0, c1, c2);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      // ---- Wt_1 uses the warp's own G_1 as the A operand (A_1 slice as B) ----
      auto wt1 = [&]() {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
#pragma unroll
          for (int j = 0; j < NT1; ++j) dmma(w1acc[j], g1v[p], g1v[2 + p], A1c[(8 * w + 2 * t + p) * L::LD1 + 8 * j + g]);
        }
      };
      // BS: a warp is done with a slice -> count it; the last of the 8 issues the next step's copy
      auto release = [&](int* cnt, auto&& issue) {
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          const int old = atomicAdd(cnt, 1);
          if ((old & 7) == 7 && more) issue(i2o + P2_B2);
        }
      };
      if (ELD == 2 && more) load_elems(i2o + P2_B2);
      if (!BS && PASD_P2_PROBE != 1 && PASD_P2_PROBE != 3) wt1();
      // ---- Wt_3^T (m-tile mt, K-half kh), K = (i1, i2) ----
      if (mt3 < MT && PASD_P2_PROBE != 1 && PASD_P2_PROBE != 3) {
        double acc[3][4] = {};
        const double* rowa = A3s + (16 * mt3 + g) * L::LD3 + 64 * kh;
        const double* rowb = rowa + 8 * L::LD3;
        const double* gcol = G3s + 180 * g;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const int k = 64 * kh + 4 * ks + t;
          double(&c)[4] = (ks & 3) == 0 ? w3acc : acc[(ks & 3) - 1];
          double b3;
          if constexpr (TIO && !TIL) {  // G_3 at (i1 = k & 15, i2 = k >> 4, i3 = g) from the B-layout bricks
            const int pb = swzB(k & 15, k >> 4, g);
            b3 = __dadd_rn(brk[5 * P2_BRICK + pb], __dmul_rn(brk[3 * P2_BRICK + pb], inv_mu_next));
          } else {
            b3 = gcol[(k & 15) + 22 * (k >> 4)];
          }
          if constexpr (HALF)
            dmma_split(c, rowa[4 * ks + t], rowb[4 * ks + t], b3, mt3 != MT - 1);  // last m-tile: rows 8-15 are padding
          else
            dmma(c, rowa[4 * ks + t], rowb[4 * ks + t], b3);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) w3acc[q] += (acc[0][q] + acc[1][q]) + acc[2][q];
      }
      if constexpr (BS) {
        release(rel3, issue_a3);
        if (PASD_P2_PROBE != 1 && PASD_P2_PROBE != 3) wt1();
        release(rel1, issue_a1);
        if (ELD == 1 && more) load_elems(i2o + P2_B2);
      }
      // prefetch this step's Wt_2 partial rows (read-modify-write below)
      double w2old[4] = {0, 0, 0, 0};
      if (!DW2 && (WS ? (w < MT) : ((w2s || kh == 0) && mt < MT))) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 16 * mt + g + 8 * (q >> 1);
          const int64_t i2 = i2o + 2 * t + (q & 1);
          if (r < R2 && i2 < I2) w2old[q] = W2k[i2 * R2 + r];
        }
      }
      P2T(7);  // 7: Wt_1 + Wt_3 products, Wt_2 partial prefetch
      if constexpr (!BS) __syncthreads();  // A1s / A3s / U2s no longer needed this step
      P2T(8);  // 8: barrier D
      if (TILS && more) load_bricks(i1o, i2o + P2_B2, i3o);  // the stores have read the bricks by now
      if constexpr (DW2) {  // this step's Wt_2 products run in the next step's elementwise phase (or the drain)
        P2T(10);
        continue;
      }
      if constexpr (WS) {
        // Warp-specialised: warps 4-7 issue the next step's staging (LSU-bound,
        // ~1.8k cycles) while warps 0-3 run the Wt_2 products over the full K
        // (no K-half exchange); the next step's top barrier joins them.
        if (w >= 4) {
          if (more) {
            stage_a1(i2o + P2_B2, A1s, w - 4, 4);
            stage_a3u2(i2o + P2_B2, tid - P2_THREADS / 2, Half{});
            if (L::EPF) stage_elems(i2o + P2_B2, tid - P2_THREADS / 2, Half{});  // next step's T, Y
          }
        } else if (w < MT && PASD_P2_PROBE != 1 && PASD_P2_PROBE != 3) {
          double acc[4][4] = {};
          const double* rowa = A2s + (16 * w + g) * L::LD2;
          const double* rowb = rowa + 8 * L::LD2;
#pragma unroll
          for (int ks = 0; ks < 32; ++ks) {
            const int k = 4 * ks + t;
            dmma(acc[ks & 3], rowa[4 * ks + t], rowb[4 * ks + t], G2s[g2x(k & 15, g, k >> 4)]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = 16 * w + g + 8 * (q >> 1);
            const int64_t i2 = i2o + 2 * t + (q & 1);
            const double v = (acc[0][q] + acc[1][q]) + (acc[2][q] + acc[3][q]);
            if (r < R2 && i2 < I2) W2c[i2 * R2 + r] = w2old[q] + v;
          }
        }
        P2T(10);
        continue;
      }
      if (more && !BS) {
        stage_a1(i2o + P2_B2, A1s, w, 8);
        stage_a3u2(i2o + P2_B2, tid, All{});
      }
      P2T(9);  // 9: staging issue
      // ---- W-b: Wt_2^T (m-tile mt, K-half kh), K = (i1, i3) ----
      double acc2[4] = {0, 0, 0, 0};
      if (mt < MT && PASD_P2_PROBE != 1 && PASD_P2_PROBE != 3) {
        double acc[3][4] = {};
        const double* rowa = A2s + (16 * mt + g) * L::LD2 + 64 * kh;
        const double* rowb = rowa + 8 * L::LD2;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const int k = 64 * kh + 4 * ks + t;
          double(&c)[4] = (ks & 3) == 0 ? acc2 : acc[(ks & 3) - 1];
          double b2;
          if constexpr (TIO && !TIL) {  // G_2 at (i1 = k & 15, i2 = g, i3 = k >> 4) from the A-layout bricks
            const int pa = swzA(k & 15, g, k >> 4);
            b2 = __dadd_rn(brk[4 * P2_BRICK + pa], __dmul_rn(brk[2 * P2_BRICK + pa], inv_mu_next));
          } else {
            b2 = G2s[g2x(k & 15, g, k >> 4)];
          }
          if constexpr (HALF)
            dmma_split(c, rowa[4 * ks + t], rowb[4 * ks + t], b2, mt != MT - 1);
          else
            dmma(c, rowa[4 * ks + t], rowb[4 * ks + t], b2);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc2[q] += (acc[0][q] + acc[1][q]) + acc[2][q];
        if (!w2s && kh == 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q) Z3s[(mt * 32 + lane) * 4 + q] = acc2[q];  // exchange (Z3s free now)
        }
      }
      if ((TIO && !TIL) || (!w2s && !PASD_P2_PAIRBAR)) {
        __syncthreads();
      } else if (!w2s && mt < MT) {  // only the two K-half warps of m-tile mt exchange
        asm volatile("bar.sync %0, 64;" ::"r"(1 + mt) : "memory");
      }
      if (more && !TIL) load_bricks(i1o, i2o + P2_B2, i3o);  // the bricks are free: next step's T, Y (TIO)
      if (w2s && mt < MT) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 16 * mt + g + 8 * (q >> 1);
          const int64_t i2 = i2o + 2 * t + (q & 1);
          if (r < R2 && i2 < I2) W2k[i2 * R2 + r] = w2old[q] + acc2[q];
        }
      } else if (!w2s && kh == 0 && mt < MT) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 16 * mt + g + 8 * (q >> 1);
          const int64_t i2 = i2o + 2 * t + (q & 1);
          if (r < R2 && i2 < I2) W2c[i2 * R2 + r] = w2old[q] + (acc2[q] + Z3s[(mt * 32 + lane) * 4 + q]);
        }
      }
      P2T(10);  // 10: Wt_2 products + K-half exchange + partial update
    }
    if constexpr (DW2) {  // drain: the last step's Wt_2 products
      const int64_t i2l = i2b + ((i2e - i2b - 1) / P2_B2) * P2_B2;
      const double* G2r = G2s + ((int)((i2l - i2b) >> 3) & 1) * (8 * 160);
      __syncthreads();  // the last step's partial update has read X2s
#pragma unroll
      for (int q = 0; q < 4; ++q) d2old[q] = d2acc[0][q] = d2acc[1][q] = d2acc[2][q] = d2acc[3][q] = 0.0;
      if (mt < MT && (w2s || kh == 0)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 16 * mt + g + 8 * (q >> 1);
          const int64_t i2 = i2l + 2 * t + (q & 1);
          if (r < R2 && i2 < I2) d2old[q] = W2k[i2 * R2 + r];
        }
      }
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) w2_quarter(qq, G2r);
      w2_sum();
      __syncthreads();
      w2_store(i2l);
    }
    // combine the two K-halves of Wt_3 through shared memory
    __syncthreads();
    if (w >= 4 && mt3 < MT) {  // K-half 1 of m-tile mt3 (K-half 0 of m-tile w is warp w)
#pragma unroll
      for (int q = 0; q < 4; ++q) Z3s[(mt3 * 32 + lane) * 4 + q] = w3acc[q];
    }
    __syncthreads();
    if (w < 4 && w < MT) {
#pragma unroll
      for (int q = 0; q < 4; ++q) w3acc[q] += Z3s[(w * 32 + lane) * 4 + q];
    }
    // ---- end of pencil: Wt_1 (sum over the 8 warps' column sets) and Wt_3 ----
    __syncthreads();
    double* wred = A1s;  // 8 warps x 16 x RP doubles (fits below A3s)
#pragma unroll
    for (int j = 0; j < NT1; ++j) {
#pragma unroll
      for (int q = 0; q < 4; ++q) wred[(w * 16 + g + 8 * (q >> 1)) * RP + 8 * j + 2 * t + (q & 1)] = w1acc[j][q];
    }
    __syncthreads();
    double* w1out = a.W1p + (int64_t)pen * 16 * R1;
    for (int idx = tid; idx < 16 * R1; idx += P2_THREADS) {
      const int l1 = idx / R1, r = idx - l1 * R1;
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s += wred[(ww * 16 + l1) * RP + r];
      w1out[idx] = s;
    }
    if (w < 4 && w < MT) {
      double* w3out = a.W3p + (int64_t)pen * 8 * R3;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = 16 * w + g + 8 * (q >> 1);
        if (r < R3) w3out[(2 * t + (q & 1)) * R3 + r] = w3acc[q];
      }
    }
    __syncthreads();
    // restore the zero padding rows of A2s clobbered by the reduction scratch
    // (A1s itself is rewritten, padding included, by every step's staging)
    for (int idx = tid; idx < (RP - R2) * 128; idx += P2_THREADS) A2s[(R2 + idx / 128) * L::LD2 + (idx & 127)] = 0.0;
  }
#if PASD_P2_TIMING
  P2T(11);  // 11: pencil ends (reductions, restores)
  if (tid == 32 * PASD_P2_TWARP)
    for (int k = 0; k < 12; ++k) atomicAdd(&g_p2_phase[k], ph_acc[k]);
#endif
  if (TIO && (!TIL || TILS) && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // element stores done
  // ---- per-CTA residual / NaN / ||G||^2 partials ----
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

// PASD_P2_BULK: copy A_1..3 and UM_2 into the tiled, padded slice layouts k_pass2_fused<RP> stages with
// one cp.async.bulk each (entries outside the tensor / rank rows >= R_n / pad columns are zero, so every
// copy is full-size and unpredicated).  One CTA per tile; ~2.3x the bytes of A_n (1.2 GB at C5) per iteration.
template <int RP>
__global__ void __launch_bounds__(256) k_retile(const Pass2Args a, const Ctl* ctl, int boff) {
  if (ctl->done) return;
  using L = P2Layout<RP, false>;
  const ModeDev& m1 = a.m[0];
  const ModeDev& m2 = a.m[1];
  const ModeDev& m3 = a.m[2];
  const int R1 = m1.R, R2 = m2.R, R3 = m3.R;
  const int64_t I1 = m1.I, I2 = m2.I, I3 = m3.I, S12 = I1 * I2;
  const int nt3 = a.n1b * a.n2b, nt2 = a.n1b * a.n3b, nt1 = a.n3b * a.n2b;
  int b = blockIdx.x + boff;  // boff: first tile of this launch (the A tiles and the UM_2 tiles can go separately)
  const int tid = threadIdx.x;
  if (b < nt3) {  // A_3 (I1, I2, R3): tile (ib1, i2 block), [r][16 l2 + l1]
    const int64_t i1o = (int64_t)(b / a.n2b) * P2_B1, i2o = (int64_t)(b % a.n2b) * P2_B2;
    double* out = a.At3 + (int64_t)b * (RP * L::LD3);
    for (int idx = tid; idx < RP * L::LD3; idx += 256) {
      const int r = idx / L::LD3, c = idx - r * L::LD3;
      const int64_t i1 = i1o + (c & 15), i2 = i2o + (c >> 4);
      out[idx] = (c < 128 && r < R3 && i1 < I1 && i2 < I2) ? m3.A[i1 + I1 * i2 + S12 * r] : 0.0;
    }
    return;
  }
  b -= nt3;
  if (b < nt2) {  // A_2 (I1, R2, I3): tile (ib3, ib1), [r][16 l3 + l1]
    const int64_t i1o = (int64_t)(b % a.n1b) * P2_B1, i3o = (int64_t)(b / a.n1b) * P2_B3;
    double* out = a.At2 + (int64_t)b * (RP * L::LD2);
    for (int idx = tid; idx < RP * L::LD2; idx += 256) {
      const int r = idx / L::LD2, c = idx - r * L::LD2;
      const int64_t i1 = i1o + (c & 15), i3 = i3o + (c >> 4);
      out[idx] = (c < 128 && r < R2 && i1 < I1 && i3 < I3) ? m2.A[i1 + I1 * (r + (int64_t)R2 * i3)] : 0.0;
    }
    return;
  }
  b -= nt2;
  if (b < nt1) {  // A_1 (R1, I2, I3): tile (ib3, i2 block), [column l2 + 8 l3][r]
    const int64_t i2o = (int64_t)(b % a.n2b) * P2_B2, i3o = (int64_t)(b / a.n2b) * P2_B3;
    double* out = a.At1 + (int64_t)b * (64 * L::LD1);
    for (int idx = tid; idx < 64 * L::LD1; idx += 256) {
      const int c = idx / L::LD1, r = idx - c * L::LD1;
      const int64_t i2 = i2o + (c & 7), i3 = i3o + (c >> 3);
      out[idx] = (r < R1 && i2 < I2 && i3 < I3) ? m1.A[r + (int64_t)R1 * (i2 + I2 * i3)] : 0.0;
    }
    return;
  }
  b -= nt1;
  {  // UM_2 rows: tile (i2 block), [l2][r]
    const int64_t i2o = (int64_t)b * P2_B2;
    double* out = a.U2t + (int64_t)b * (8 * L::LDU);
    for (int idx = tid; idx < 8 * L::LDU; idx += 256) {
      const int l2 = idx / L::LDU, r = idx - l2 * L::LDU;
      out[idx] = (r < R2 && i2o + l2 < I2) ? m2.UM[m2.ioff + i2o + l2 + m2.Ifull * r] : 0.0;
    }
  }
}
// doubles of the tiled copies (At1, At2, At3, U2t) for padded rank rp
struct RetileSizes {
  size_t at1, at2, at3, u2t;
  int blocks;
};
inline RetileSizes retile_sizes(int rp, int n1b, int n2b, int n3b) {
  RetileSizes z;
  z.at1 = (size_t)n3b * n2b * 64 * (rp + 4);
  z.at2 = (size_t)n3b * n1b * rp * 132;
  z.at3 = (size_t)n1b * n2b * rp * 132;
  z.u2t = (size_t)n2b * 8 * (rp + 4);
  z.blocks = n1b * n2b + n1b * n3b + n3b * n2b + n2b;
  return z;
}
// part 0: all tiles; 1: the A_1..3 tiles (ready after pass 1); 2: the UM_2 tiles (ready after the SVT)
inline void retile_launch(int rp, const Pass2Args& a, const Ctl* ctl, cudaStream_t st, int part = 0) {
  const int all = retile_sizes(rp, a.n1b, a.n2b, a.n3b).blocks;
  const int boff = part == 2 ? all - a.n2b : 0;
  const int blocks = part == 0 ? all : (part == 1 ? all - a.n2b : a.n2b);
  switch (rp) {
    case 8: k_retile<8><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
    case 16: k_retile<16><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
    case 24: k_retile<24><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
    case 32: k_retile<32><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
    case 40: k_retile<40><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
    case 48: k_retile<48><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
    case 56: k_retile<56><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
    default: k_retile<64><<<blocks, 256, 0, st>>>(a, ctl, boff); break;
  }
}

template <int RP, bool TIO, class EL = double>
void launch_pass2(const Pass2Args& a, const Ctl* ctl, const P2Tmaps& tm, int grid, cudaStream_t st) {
  k_pass2_fused<RP, TIO, EL><<<grid, P2_THREADS, P2Layout<RP, TIO>::bytes, st>>>(a, ctl, tm);
}
// float storage (fp32 mode) at the padded ranks this kernel serves by default (RP >= 32)
template <int RP>
constexpr bool p2_has_f32() {
  return RP >= 32;
}
template <int RP>
void setup_pass2() {
  cudaFuncSetAttribute(k_pass2_fused<RP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)P2Layout<RP, false>::bytes);
  if constexpr (p2_has_f32<RP>())
    cudaFuncSetAttribute(k_pass2_fused<RP, false, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)P2Layout<RP, false>::bytes);
  if (P2Layout<RP, true>::bytes <= 227u * 1024u)
    cudaFuncSetAttribute(k_pass2_fused<RP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)P2Layout<RP, true>::bytes);
}

inline int pass2_rp(int R1, int R2, int R3) {
  int r = R1 > R2 ? R1 : R2;
  r = r > R3 ? r : R3;
  return (r + 7) / 8 * 8;
}
template <int RP>
size_t pass2_smem_rp(bool tio) {
  return tio ? P2Layout<RP, true>::bytes : P2Layout<RP, false>::bytes;
}
inline size_t pass2_smem(int rp, bool tio) {
  switch (rp) {
    case 8: return pass2_smem_rp<8>(tio);
    case 16: return pass2_smem_rp<16>(tio);
    case 24: return pass2_smem_rp<24>(tio);
    case 32: return pass2_smem_rp<32>(tio);
    case 40: return pass2_smem_rp<40>(tio);
    case 48: return pass2_smem_rp<48>(tio);
    case 56: return pass2_smem_rp<56>(tio);
    default: return pass2_smem_rp<64>(tio);
  }
}
inline void pass2_setup(int rp) {
  switch (rp) {
    case 8: setup_pass2<8>(); break;
    case 16: setup_pass2<16>(); break;
    case 24: setup_pass2<24>(); break;
    case 32: setup_pass2<32>(); break;
    case 40: setup_pass2<40>(); break;
    case 48: setup_pass2<48>(); break;
    case 56: setup_pass2<56>(); break;
    default: setup_pass2<64>(); break;
  }
}
template <int RP>
void pass2_launch_rp(bool tio, bool f32, const Pass2Args& a, const Ctl* ctl, const P2Tmaps& tm, int grid,
                     cudaStream_t st) {
  if constexpr (p2_has_f32<RP>()) {
    if (f32) {
      launch_pass2<RP, false, float>(a, ctl, tm, grid, st);
      return;
    }
  }
  if (tio)
    launch_pass2<RP, true>(a, ctl, tm, grid, st);
  else
    launch_pass2<RP, false>(a, ctl, tm, grid, st);
}
inline void pass2_launch(int rp, bool tio, const Pass2Args& a, const Ctl* ctl, const P2Tmaps& tm, int grid,
                         cudaStream_t st, bool f32 = false) {
  switch (rp) {
    case 8: pass2_launch_rp<8>(tio, f32, a, ctl, tm, grid, st); break;
    case 16: pass2_launch_rp<16>(tio, f32, a, ctl, tm, grid, st); break;
    case 24: pass2_launch_rp<24>(tio, f32, a, ctl, tm, grid, st); break;
    case 32: pass2_launch_rp<32>(tio, f32, a, ctl, tm, grid, st); break;
    case 40: pass2_launch_rp<40>(tio, f32, a, ctl, tm, grid, st); break;
    case 48: pass2_launch_rp<48>(tio, f32, a, ctl, tm, grid, st); break;
    case 56: pass2_launch_rp<56>(tio, f32, a, ctl, tm, grid, st); break;
    default: pass2_launch_rp<64>(tio, f32, a, ctl, tm, grid, st); break;
  }
}

// Reduce the pass-2 partials into Wt_n (I_n x R_n, column-major) and
// ctl->gnorm2[n], in a fixed order.  grid = (ceil(max I_n R_n / 256), 3).
// Wt_n = sum of the pass-2 partials, one warp per output entry: lane l sums
// partials l, l+32, ... in order, then a fixed xor-shuffle tree (deterministic;
// a per-thread serial sum was load-latency bound at small sizes).
__global__ void k_pass2_reduce(const Pass2Args a, int nblk, Ctl* ctl, double* g2out) {
  if (ctl->done) return;
  const int n = blockIdx.y;
  const ModeDev& m = a.m[n];
  const int R = m.R, lane = threadIdx.x & 31;
  const int64_t IR = m.Ifull * R;  // full rows; rows outside this rank's slab are 0
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t idx = wid; idx < IR; idx += nw) {
    const int64_t ifull = idx % m.Ifull;
    const int r = (int)(idx / m.Ifull);
    const int64_t i = ifull - m.ioff;
    double s = 0.0;
    if (i >= 0 && i < m.I) {
      if (n == 0) {
        const int ib = (int)(i / a.b1), l = (int)(i % a.b1);
        for (int k = lane; k < a.n3b * a.nseg; k += 32) {
          const int b3 = k % a.n3b, sg = k / a.n3b;
          s += a.W1p[((int64_t)(ib + a.n1b * b3 + a.npencils * sg) * a.b1 + l) * R + r];
        }
      } else if (n == 1) {
        for (int c = lane; c < a.nw2; c += 32) s += a.W2part[((int64_t)c * m.I + i) * R + r];
      } else {
        const int ib = (int)(i / P2_B3), l = (int)(i % P2_B3);
        for (int k = lane; k < a.n1b * a.nseg; k += 32) {
          const int b1 = k % a.n1b, sg = k / a.n1b;
          s += a.W3p[((int64_t)(b1 + a.n1b * ib + a.npencils * sg) * 8 + l) * R + r];
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) m.Wt[idx] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double s = 0.0;
    for (int c = lane; c < nblk; c += 32) s += a.gpart[c * 3 + n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) g2out[n] = s;
  }
}

}  // namespace pasd
