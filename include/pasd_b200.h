/*
 * pasd_b200.h — C-ABI of the B200-native PASD ADMM solver (tensor robust PCA,
 * arXiv 1712.09999).  Plain pointers and sizes only: no torch, no C++ types.
 *
 * This is the drop-in boundary for the reference solver entry point
 *   tenrec::pasd_recover(const DenseTensor&, const PasdConfig&,
 *                        const IterationObserver&)        (proj/include/tenrec/pasd.hpp:65-66)
 * with
 *   PasdConfig      -> pasd_options         (proj/include/tenrec/pasd.hpp:8-27)
 *   RecoveryResult  -> pasd_outputs         (proj/include/tenrec/recovery.hpp:20-34)
 *   Certificate     -> pasd_outputs.cert_*  (proj/include/tenrec/recovery.hpp:14-18)
 *   IterationView   -> pasd_iteration_view  (proj/include/tenrec/recovery.hpp:38-48)
 *   exceptions      -> PASD_ERR_* + errbuf  (proj/include/tenrec/errors.hpp:9-30)
 *
 * Tensors are dense float64 with the FIRST index varying fastest
 * (proj/include/tenrec/tensor.hpp:23-24).  Matrices are column-major.
 *
 * Every call owns its stream(s), device buffers and (multi-GPU) NCCL
 * communicator, so concurrent calls from several host threads are safe (the
 * reference harness calls the solver from a thread pool,
 * proj/src/bench.cpp:226-248).  The only global mutable state is the opt-in
 * solver reuse of pasd_b200_recover (PASD_FLAG_REUSE_SOLVER, mutex-guarded;
 * see there for the HBM it retains).
 */
#ifndef PASD_B200_H
#define PASD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PASD_B200_ABI_VERSION 2

/* Status codes.  The numeric values follow the reference CLI's exit-code
 * taxonomy (proj/tools/cli.hpp:9-14): argument 1, I/O 2, numerical 3.  State
 * errors (certificate misuse) are 4 and CUDA/NCCL failures 5. */
enum {
  PASD_OK = 0,
  PASD_ERR_ARGUMENT = 1,  /* tenrec::ArgumentError  */
  PASD_ERR_IO = 2,        /* tenrec::IoError        */
  PASD_ERR_NUMERICAL = 3, /* tenrec::NumericalError */
  PASD_ERR_STATE = 4,     /* tenrec::StateError     */
  PASD_ERR_CUDA = 5       /* device / NCCL failure (no reference analogue) */
};

/* pasd_options.flags */
enum {
  PASD_FLAG_NONE = 0,
  /* Skip the certificate even when converged (reference always computes it,
   * pasd.cpp:272-273; this only saves the final ||T||_1 pass). */
  PASD_FLAG_NO_CERTIFICATE = 1u << 0,
  /* Deterministic fixed-iteration mode: ignore eps, run exactly maxiter
   * iterations (BASELINE "fixed N iters" runs).  converged is reported 0. */
  PASD_FLAG_FIXED_ITERS = 1u << 1,
  /* pasd_b200_recover only: keep this call's solver (device buffers + the
   * captured iteration graph) for the next call with identical options, which
   * then skips allocation, graph capture and teardown.  Results do not depend
   * on it.  The kept solver holds its HBM -- about (N + 4) S doubles plus the
   * A_n (R_n J_n doubles each): ~64 GB at 1000^3, R = 50 -- until
   * pasd_b200_release_cache() or exit; a call with different options frees it
   * before allocating its own. */
  PASD_FLAG_REUSE_SOLVER = 1u << 2,
  /* Sharded solvers: after every pasd_b200_solver_run, all-reduce a 64-bit
   * hash of the replicated U_n and M_n and fail (PASD_ERR_NUMERICAL) if any
   * rank differs (SURVEY 8(e) debug check; also env PASD_CHECK_REPLICAS). */
  PASD_FLAG_CHECK_REPLICAS = 1u << 3,
  /* fp32 mode (BASELINE north_star's optional mode; no reference analogue):
   * the element tensors T, E, D = T - E and Y_n live in HBM as float32 (half
   * the footprint and stream bytes); every contraction and elementwise step
   * still computes in fp64 registers (DMMA) and rounds to float32 on store;
   * U_n, M_n, A_n and the small solves stay fp64.  Inputs and outputs at this
   * boundary stay float64.  Order-3 tensors.  Expected agreement with the
   * fp64 reference: L, E to ~1e-4 relative (north_star's fp32 bar). */
  PASD_FLAG_FP32 = 1u << 4
};

/* Mirror of tenrec::PasdConfig (pasd.hpp:8-27) plus placement. */
typedef struct pasd_options {
  int32_t order;                 /* N = number of modes                           */
  const int64_t* dims;           /* [N] I_1..I_N                                   */
  const int64_t* ranks;          /* [N] R_n  (PasdConfig::ranks)                   */
  const double* lambdas;         /* [N] lambda_n (PasdConfig::lambdas)             */
  const double* output_weights;  /* [N] alpha_n, NULL = lambdas (pasd.hpp:16,26)   */
  double mu0;                    /* default 1e-4  (pasd.hpp:11)                    */
  double mu_max;                 /* default 1e10  (pasd.hpp:12)                    */
  double rho;                    /* default 1.1   (pasd.hpp:13)                    */
  double eps;                    /* default 1e-5  (pasd.hpp:14)                    */
  int32_t maxiter;               /* default 1000  (pasd.hpp:15)                    */
  int32_t device;                /* CUDA ordinal                                   */
  uint32_t flags;                /* PASD_FLAG_*                                    */
  int32_t poll_every;            /* host polls the on-device stop flag every k
                                    iterations (0 = auto). Results never depend on
                                    it: iterations after the stop are no-ops.      */
} pasd_options;

/* Multi-GPU slab sharding along the LAST mode (one process per GPU).  A NULL
 * shard means the whole tensor on one device.  With `loopback` set (a group
 * from pasd_b200_loopback_create) the ranks instead share ONE device inside
 * one process, one host thread per rank: the same sharded code path, with the
 * all-reduces done by host rendezvous + a reduce kernel (no NCCL, iterations
 * launched eagerly).  That is a test vehicle for nranks > 1, not a speed-up. */
typedef struct pasd_shard {
  int32_t rank;                  /* this process's rank                            */
  int32_t nranks;                /* world size                                     */
  const void* nccl_unique_id;    /* 128-byte ncclUniqueId from rank 0 (NULL if nranks==1) */
  int64_t slab_begin;            /* first last-mode index owned by this rank       */
  int64_t slab_end;              /* one past the last                              */
  void* loopback;                /* loopback group, or NULL for NCCL               */
} pasd_shard;

/* Loopback group of nranks (1..8) solvers sharing one device.  Destroy it after
 * every solver that uses it. */
int pasd_b200_loopback_create(int32_t nranks, void** group_out, char* errbuf, size_t errlen);
void pasd_b200_loopback_destroy(void* group);

/* Debug: with env PASD_B200_GUARD=1 every device buffer gets 64 KB canary
 * bands checked when it is freed.  Returns the number of overwritten bands;
 * `checked` = buffers verified so far, `live` = buffers not yet freed. */
int64_t pasd_b200_guard_report(int64_t* checked, int64_t* live);

/* Snapshot handed to the observer after each completed iteration
 * (tenrec::IterationView, recovery.hpp:38-48).  Pointers are host copies valid
 * only during the callback (pasd.cpp:241-242). */
typedef struct pasd_iteration_view {
  int32_t iter;                  /* 1-based count of completed iterations          */
  double mu_used;
  double mu_next;
  const double* residual_inf;    /* [N]                                            */
  const double* e;               /* S                                              */
  const double* const* z;        /* [N] x S                                        */
  const double* const* y;        /* [N] x S                                        */
  const double* const* u;        /* [N] x (I_n x R_n) column-major                 */
  const double* const* v;        /* [N] x (R_n x J_n) column-major, J_n = S / I_n  */
} pasd_iteration_view;

typedef void (*pasd_observer_fn)(const pasd_iteration_view* view, void* user);

/* Mirror of tenrec::RecoveryResult (recovery.hpp:20-34).  Every tensor pointer
 * is a caller-allocated HOST buffer of S doubles or NULL (= not wanted). */
typedef struct pasd_outputs {
  double* x;                     /* combined low-rank estimate                     */
  double* e;                     /* sparse estimate                                */
  double* const* z;              /* [N] per-mode Z_n, or NULL                      */
  double* const* y;              /* [N] final multipliers, or NULL                 */
  double* const* y_hat;          /* [N] auxiliary multipliers, or NULL             */
  double* residual_history;      /* capacity maxiter, or NULL                      */
  double* final_residuals;       /* [N], or NULL                                   */
  int32_t iters;
  int32_t converged;
  double objective;
  int32_t has_certificate;
  double cert_epsilon_hat;
  double cert_c;
  double cert_bound;
} pasd_outputs;

/* ---- one-call drop-in --------------------------------------------------- */

/* Full solve from a HOST tensor: H2D of t, the device-resident ADMM loop, the
 * finalisation and D2H of the requested outputs.  Returns PASD_OK or an error
 * code; errbuf receives the reference's exception message text.  With
 * PASD_FLAG_REUSE_SOLVER the solver is kept for the next identical call. */
int pasd_b200_recover(const double* t, const pasd_options* opt, pasd_outputs* out,
                      pasd_observer_fn observer, void* user, char* errbuf, size_t errlen);

/* Free the solver kept by pasd_b200_recover under PASD_FLAG_REUSE_SOLVER
 * (device memory returns to the allocator).  Safe to call at any time. */
void pasd_b200_release_cache(void);

/* SNN / HoRPCA full-SVT ADMM baseline (tenrec::snn_recover,
 * proj/src/baselines.cpp:37-143) on the device.  Options: order, dims,
 * lambdas, output_weights, mu0, mu_max, rho, eps, maxiter, device, flags
 * (PASD_FLAG_FIXED_ITERS honoured); ranks are ignored (SnnConfig has none).
 * Validation and error messages follow SnnConfig::validate
 * (baselines.cpp:12-29).  Outputs: x, e, z[N], y[N], iters, converged,
 * residual_history, final_residuals, objective; y_hat and the certificate are
 * not produced (snn_recover leaves them empty).  Observer views carry u = v =
 * NULL.  Limit of this build: every I_n <= 112 and <= prod of the others. */
int pasd_b200_snn_recover(const double* t, const pasd_options* opt, pasd_outputs* out,
                          pasd_observer_fn observer, void* user, char* errbuf, size_t errlen);


/* ---- device-resident solver handle (benchmarks, multi-GPU) -------------- */

typedef struct pasd_solver pasd_solver;

int pasd_b200_solver_create(const pasd_options* opt, const pasd_shard* shard, pasd_solver** out,
                            char* errbuf, size_t errlen);
/* Upload the (local slab of the) observed tensor.  `t_is_device` != 0 means t
 * is a device pointer on the solver's device (device-to-device copy). */
int pasd_b200_solver_load(pasd_solver* s, const double* t, int t_is_device, char* errbuf,
                          size_t errlen);
/* Reset the iterate to the initial state (E=0, Y=0, U=eye, V=0, mu=mu0). */
int pasd_b200_solver_reset(pasd_solver* s, char* errbuf, size_t errlen);
/* Run up to `iters` further iterations (stops early on convergence). */
int pasd_b200_solver_run(pasd_solver* s, int32_t iters, int32_t* iters_done, int32_t* converged,
                         char* errbuf, size_t errlen);
/* Finalise (Y-hat, objective, X, certificate) and copy requested outputs to
 * host buffers (local slab only for a sharded solver). */
int pasd_b200_solver_finalize(pasd_solver* s, pasd_outputs* out, char* errbuf, size_t errlen);
/* Replace the iterate (tenrec::PasdState, pasd.hpp:33-41) from HOST buffers:
 * e (S), y[N] (S each), u[N] (I_n x R_n), v[N] (R_n x J_n, unfolding layout),
 * the penalty mu of the next iteration and the completed-iteration count.
 * Used for single-step parity: the next pasd_b200_solver_run(s, 1, ...) then
 * performs exactly the reference iteration from that state (pasd.cpp:168-244). */
int pasd_b200_solver_set_state(pasd_solver* s, const double* e, const double* const* y, const double* const* u,
                               const double* const* v, double mu, int32_t iter, char* errbuf, size_t errlen);
/* Device pointers of the local slab of E and of Y_n (diagnostics / zero-copy). */
/* Device pointer of the current E (float64; float32 storage in the fp32 mode). */
const double* pasd_b200_solver_device_e(const pasd_solver* s);
/* The CUDA stream (cudaStream_t) the solver launches on. */
void* pasd_b200_solver_stream(const pasd_solver* s);
/* Kernel classes of one iteration, in launch order. */
enum {
  PASD_K_POLAR = 0,      /* Procrustes small solve (one CTA per mode)        */
  PASD_K_CONTRACT_A = 1, /* A_n = U_n^T G_(n)                                */
  PASD_K_GRAM = 2,       /* Gram_n partials                                  */
  PASD_K_SVT = 3,        /* SVT small solve (one CTA per mode)               */
  PASD_K_UPDATE = 4,     /* refold + E shrink + Y ascent + residuals         */
  PASD_K_FINISH = 5,     /* mu schedule / stop rule                          */
  PASD_K_CONTRACT_W = 6, /* Wt_n = G_(n)^{next} A_n^T                        */
  PASD_NUM_KERNEL_CLASSES = 7
};
/* Profiling run: `iters` further iterations launched eagerly (no graph) with
 * CUDA events around every kernel on the solver's stream.  Fills, per kernel
 * class, the summed device time in ms, the launch count, and the algorithmic
 * bytes / flops of one launch of that class summed over modes.
 * The iterate advances exactly as pasd_b200_solver_run would advance it. */
int pasd_b200_solver_profile(pasd_solver* s, int32_t iters, double* kernel_ms, int64_t* kernel_launches,
                             double* kernel_bytes, double* kernel_flops, char* errbuf, size_t errlen);
/* Ranks of the current iterate (diagnostics, e.g. to check that a run has
 * reached the full-rank phase): svt_keep[n] = number of singular values of
 * A_n kept by the last SVT (rank of V_n, linops.cpp:84-86), polar_rank[n] =
 * numerical rank of W_n in the last Procrustes step (0 when it was degenerate
 * and U_n was kept, pasd.cpp:70-74).  N entries each. */
int pasd_b200_solver_ranks(pasd_solver* s, int32_t* svt_keep, int32_t* polar_rank, char* errbuf, size_t errlen);
/* Number of kernel launches issued by the last pasd_b200_solver_run call. */
int64_t pasd_b200_solver_launches(const pasd_solver* s);
void pasd_b200_solver_destroy(pasd_solver* s);

/* ---- reference-shaped helpers (pasd.hpp:51-58, tensor.hpp:86-91) -------- */

/* lambda_n = sqrt(max(I_n, prod_{j!=n} I_j)) / N  (pasd.cpp:51-60). */
int pasd_b200_default_lambdas(int32_t order, const int64_t* dims, double* lambdas_out,
                              char* errbuf, size_t errlen);
/* R = floor(1.2 r) in integer arithmetic (pasd.cpp:62-66). */
int pasd_b200_default_rank_bound(int64_t target_rank, int64_t* out, char* errbuf, size_t errlen);
/* PasdConfig::validate (pasd.cpp:12-49): same checks, same messages. */
int pasd_b200_validate(const pasd_options* opt, char* errbuf, size_t errlen);

/* Device implementations of the reference linops (linops.hpp:15-46), built
 * from the same kernels the solver uses (k_gram + k_svt, k_contract_W +
 * k_polar).  Host buffers in, host buffers out; column-major.
 *   svt:        rows <= 64 (the R side of the Gram eigenproblem).  tau == 0
 *               returns m unchanged (linops.cpp:80-81).  *kept = #sigma > tau.
 *   procrustes: U = polar(g v^T) for g (I x P), v (R x P), R <= 64.  Returns
 *               *degenerate = 1 and leaves u_out untouched when
 *               ||g v^T||_F <= 1e-14 max(1, ||g||_F ||v||_F) (linops.cpp:99-101).
 *               u_prev (I x R, may be NULL = identity) seeds the deterministic
 *               completion of numerically null directions. */
int pasd_b200_svt(const double* m, int64_t rows, int64_t cols, double tau, double* out, int32_t* kept,
                  int32_t device, char* errbuf, size_t errlen);
int pasd_b200_procrustes(const double* g, int64_t i_rows, int64_t p_cols, const double* v, int64_t r_rows,
                         const double* u_prev, double* u_out, int32_t* degenerate, int32_t* rank, int32_t device,
                         char* errbuf, size_t errlen);

/* ---- spec-shaped single-step API (pasd.hpp:43-58, 68-70) ----------------
 * The reference's PasdState pieces as host buffers: t, e, y (S doubles each,
 * first index fastest), u (I_n x R_n) and v (R_n x J_n, J_n = S / I_n,
 * unfolding column order), all column-major; mode is 1-based like the
 * reference (out of range -> ArgumentError "mode m out of range 1..N",
 * tensor.cpp:133-137).  Device kernels compute every step; results go to
 * caller-allocated host buffers.
 *
 * pasd_g_matrix (pasd.cpp:82-97): g_out (I_n x J_n) = unfold_n((T - E) + Y / mu),
 * the reference's operation order (bit-exact). */
int pasd_b200_g_matrix(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y,
                       double mu, int32_t mode, double* g_out, int32_t device, char* errbuf, size_t errlen);
/* update_u (pasd.cpp:99-103 -> update_u_from, pasd.cpp:70-74): u_out (I_n x R_n)
 * = polar(G_n V_n^T), or u_prev when the product is numerically zero
 * (linops.cpp:99-101; *degenerate = 1). */
int pasd_b200_update_u(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y,
                       double mu, int32_t mode, int64_t rank, const double* u_prev, const double* v, double* u_out,
                       int32_t* degenerate, int32_t device, char* errbuf, size_t errlen);
/* update_v (pasd.cpp:105-109 -> update_v_from, pasd.cpp:76-78): v_out (R_n x J_n)
 * = svt(U_n^T G_n, lambda / mu); *kept = number of singular values kept. */
int pasd_b200_update_v(int32_t order, const int64_t* dims, const double* t, const double* e, const double* y,
                       double mu, int32_t mode, int64_t rank, const double* u, double lambda, double* v_out,
                       int32_t* kept, int32_t device, char* errbuf, size_t errlen);
/* update_e (pasd.cpp:111-130): e_out = soft(mean_n((T - fold_n(U_n V_n)) + Y_n / mu),
 * 1 / (mu N)); u[N], v[N], y[N], ranks[N]. */
int pasd_b200_update_e(int32_t order, const int64_t* dims, const int64_t* ranks, const double* t,
                       const double* const* u, const double* const* v, const double* const* y, double mu,
                       double* e_out, int32_t device, char* errbuf, size_t errlen);
/* suboptimality_certificate (pasd.hpp:68-70, pasd.cpp:277-309) of a finished
 * run: PASD_ERR_STATE "certificate requires a converged result" unless
 * converged, "certificate requires the final multipliers" when y / y_hat
 * (N host tensors each) are missing.  opt supplies dims, lambdas, mu0, rho,
 * eps (and the device). */
int pasd_b200_certificate(const double* t, const pasd_options* opt, int32_t iters, int32_t converged,
                          const double* const* y, const double* const* y_hat, double* epsilon_hat, double* c,
                          double* bound, char* errbuf, size_t errlen);

/* nuclear_norm(unfold(t, mode)) (linops.cpp:74-76; certify's objective check,
 * cli.cpp:504-511) on the device, for unfoldings of numerical rank <= 64 (the
 * low-rank estimates Z_n and Tucker truths it is used on): range finder +
 * Jacobi.  ArgumentError when the rank exceeds 64. */
int pasd_b200_nuclear_norm_unfold(const double* t, int32_t order, const int64_t* dims, int32_t mode, double* out,
                                  int32_t device, char* errbuf, size_t errlen);

/* ---- synthetic instances: the reference generator (synth.cpp:71-121) ------
 * T = core x_1 U_1 ... x_N U_N (+ sparse corruption) with the reference's
 * random streams (rng.hpp:17-79: splitmix64-derived mt19937_64 per purpose,
 * Box-Muller Gaussians, 53-bit uniforms): core and factor draws, the Haar
 * factors (Householder QR, diag(R) sign fix, synth.cpp:40-53), the partial
 * Fisher-Yates support of round(rho S) entries and the noise values drawn in
 * sorted-index order (synth.cpp:91-121).  The draws run on the host (they
 * are sequential by definition), the mode products and the scatter on the
 * device.  The reference's verify_tucker_rank SVD check (synth.cpp:55-67) is
 * not run. */
typedef struct pasd_synth_spec {
  int32_t order;
  const int64_t* dims;     /* [N] I_n                                             */
  const int64_t* ranks;    /* [N] Tucker ranks r_n (SynthSpec::ranks)             */
  uint64_t seed;           /* SynthSpec::seed (cli.cpp:164 default 0)             */
  int32_t factor_kind;     /* 0 Haar (reference); 1 |N(0,1)| columns l2-normalised,
                              |core|, T / max(T) (BASELINE configs[3] extension)  */
  int32_t corrupt_mode;    /* 0 add U[lo,hi] (reference: lo=-1, hi=1); 1 replace by
                              U[lo,hi] (reference: 0, 255); 2 per last-mode frame,
                              `cells` aligned block x block cells of the mode-1 x
                              mode-2 plane replaced by U[lo,hi] (configs[3])      */
  double corruption;       /* rho in [0, 1] (modes 0, 1)                          */
  double lo, hi;
  int64_t block, cells;    /* mode 2 only                                         */
  int32_t device;
} pasd_synth_spec;
/* t_out: S doubles (device pointer on spec->device if t_is_device, else host);
 * l0_out: the uncorrupted tensor (optional, same convention); support_out:
 * the sorted corrupted positions (optional host buffer of *count_out entries,
 * at most S); count_out: number of corrupted entries. */
int pasd_b200_synth(const pasd_synth_spec* spec, double* t_out, int t_is_device, double* l0_out, int l0_is_device,
                    int64_t* support_out, int64_t* count_out, char* errbuf, size_t errlen);
/* Host-only pieces of the generator (no device needed), for tests: the Haar /
 * kind-1 factor of mode `mode` (1-based, purpose factor + mode) and the
 * unsorted partial Fisher-Yates support of corrupt_sparse. */
int pasd_b200_synth_factor(int64_t rows, int64_t cols, uint64_t seed, int32_t mode, int32_t kind, double* out,
                           char* errbuf, size_t errlen);
int pasd_b200_synth_support(int64_t total, double rho, uint64_t seed, int64_t* pos_out, int64_t* count_out,
                            char* errbuf, size_t errlen);

/* 128-byte NCCL unique id for pasd_shard.nccl_unique_id (rank 0 creates it and
 * broadcasts it to the other ranks with the host launcher's own channel). */
int pasd_b200_nccl_unique_id(void* out128, char* errbuf, size_t errlen);

/* Library / build identification. */
int pasd_b200_abi_version(void);
const char* pasd_b200_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* PASD_B200_H */
