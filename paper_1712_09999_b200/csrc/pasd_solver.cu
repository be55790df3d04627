// pasd_solver.cu — host driver and C-ABI of the B200-native PASD solver.
//
// Drop-in for tenrec::pasd_recover (proj/include/tenrec/pasd.hpp:65-66,
// proj/src/pasd.cpp:132-275): same options (PasdConfig, pasd.hpp:8-27), same
// validation messages (pasd.cpp:12-49), same outputs (RecoveryResult,
// recovery.hpp:20-34) and the same error taxonomy (errors.hpp:9-30), mapped to
// status codes + message text at the C boundary (include/pasd_b200.h).
//
// The ADMM loop is device resident: one iteration is a fixed sequence of
// kernels that read mu / iteration / stop flag from device memory, captured
// once into a CUDA graph and replayed; the host only polls the stop flag every
// `poll_every` iterations.  Iterations launched after the stop are no-ops, so
// results never depend on the polling period.  No CPU fallback exists: every
// per-iteration step is a kernel in pasd_kernels.cuh / pasd_small.cuh.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pasd_b200.h"
#include "pasd_common.cuh"
#include "pasd_kernels.cuh"
#include "pasd_small.cuh"
#include "pasd_pass2.cuh"
#include "pasd_pass1.cuh"
#include "pasd_gram.cuh"
#include "pasd_pass2m8.cuh"
#include "pasd_pass2ts.cuh"
#include "pasd_comm.cuh"

using namespace pasd;

namespace {
// SMs left to NCCL while pass 1 of modes 1 and 2 overlaps the A_3 all-reduce
constexpr int kNcclSms = 16;

struct PasdError : std::runtime_error {
  int code;
  PasdError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw PasdError(code, msg); }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(PASD_ERR_CUDA, std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)
void nk(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(PASD_ERR_CUDA, std::string("nccl: ") + what + ": " + ncclGetErrorString(r));
}
#define NK(x) nk((x), #x)

int guarded_call(char* err, size_t errlen, const std::function<void()>& f);

// NCCL backend of the sharded iteration's collectives (pasd_comm.cuh).
class NcclComm final : public Comm {
 public:
  NcclComm(int nranks, int rank, const ncclUniqueId& id) { NK(ncclCommInitRank(&c_, nranks, id, rank)); }
  ~NcclComm() override {
    if (c_) ncclCommDestroy(c_);
  }
  void group_start() override { NK(ncclGroupStart()); }
  void group_end() override { NK(ncclGroupEnd()); }
  void allreduce(const double* send, double* recv, size_t count, RedOp op, cudaStream_t st) override {
    NK(ncclAllReduce(send, recv, count, ncclDouble, op == RedOp::Sum ? ncclSum : ncclMax, c_, st));
  }
  bool capturable() const override { return true; }
  const char* kind() const override { return "nccl"; }

 private:
  ncclComm_t c_ = nullptr;
};

// Loopback backend: all ranks of a group in this process on one device, one
// host thread per rank (pasd_comm.cuh).  Grouped calls are queued and run as
// one rendezvous at group_end.
class LoopbackComm final : public Comm {
 public:
  LoopbackComm(LoopbackGroup* g, int rank) : g_(g), rank_(rank) {}
  void group_start() override { in_group_ = true; }
  void group_end() override {
    in_group_ = false;
    flush();
  }
  void allreduce(const double* send, double* recv, size_t count, RedOp op, cudaStream_t st) override {
    ops_.push_back({send, recv, count, op, st});
    if (!in_group_) flush();
  }
  bool capturable() const override { return false; }
  const char* kind() const override { return "loopback"; }

 private:
  void flush() {
    std::vector<LoopbackGroup::Op> ops;
    ops.swap(ops_);
    for (const auto& o : ops) CK(cudaStreamSynchronize(o.st));  // this rank's partials are complete
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->posted[rank_] = ops;
    }
    if (!g_->barrier()) fail(PASD_ERR_CUDA, "pasd_b200: loopback group broken (another rank failed or timed out)");
    for (int q = 0; q < g_->nranks; ++q) {
      const auto& oq = g_->posted[q];
      bool same = oq.size() == ops.size();
      for (size_t k = 0; same && k < ops.size(); ++k) same = oq[k].count == ops[k].count && oq[k].op == ops[k].op;
      if (!same) {
        g_->abort();
        fail(PASD_ERR_CUDA, "pasd_b200: loopback ranks issued mismatched collectives");
      }
    }
    for (size_t k = 0; k < ops.size(); ++k) {
      LoopbackSrc src{};
      for (int q = 0; q < g_->nranks; ++q) src.p[q] = g_->posted[q][k].send;
      const int64_t cnt = (int64_t)ops[k].count;
      const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((cnt + 255) / 256, 1184));
      k_loopback_reduce<<<blocks, 256, 0, ops[k].st>>>(src, g_->nranks, ops[k].recv, cnt,
                                                       ops[k].op == RedOp::Max ? 1 : 0);
      CK(cudaGetLastError());
    }
    for (const auto& o : ops) CK(cudaStreamSynchronize(o.st));
    // every rank has read every send buffer before any rank overwrites one
    if (!g_->barrier()) fail(PASD_ERR_CUDA, "pasd_b200: loopback group broken (another rank failed or timed out)");
  }
  LoopbackGroup* g_;
  int rank_;
  bool in_group_ = false;
  std::vector<LoopbackGroup::Op> ops_;
};

void set_err(char* err, size_t len, const std::string& m) {
  if (err && len) std::snprintf(err, len, "%s", m.c_str());
}

struct Dims {
  std::vector<int64_t> d;
  int64_t total = 0;
};

// dims_product (tensor.cpp:9-23)
int64_t dims_product(const std::vector<int64_t>& dims) {
  if (dims.empty()) fail(PASD_ERR_ARGUMENT, "tensor order must be at least 1");
  int64_t prod = 1;
  for (size_t n = 0; n < dims.size(); ++n) {
    const int64_t d = dims[n];
    if (d < 1)
      fail(PASD_ERR_ARGUMENT, "dimension " + std::to_string(n + 1) + " must be positive, got " + std::to_string(d));
    if (prod > std::numeric_limits<int64_t>::max() / d) fail(PASD_ERR_ARGUMENT, "dimension product overflows");
    prod *= d;
  }
  return prod;
}

// PasdConfig::validate (pasd.cpp:12-49), same checks and messages, plus the
// kernel limits of this build (rank <= 64, order <= 8).
void validate_options(const pasd_options* o) {
  if (!o) fail(PASD_ERR_ARGUMENT, "config: null options");
  if (o->order < 1 || !o->dims) fail(PASD_ERR_ARGUMENT, "tensor order must be at least 1");
  const size_t n_modes = (size_t)o->order;
  std::vector<int64_t> dims(o->dims, o->dims + n_modes);
  dims_product(dims);
  if (!o->lambdas) fail(PASD_ERR_ARGUMENT, "config: expected " + std::to_string(n_modes) + " lambdas, got 0");
  for (size_t n = 0; n < n_modes; ++n)
    if (!(o->lambdas[n] > 0.0) || !std::isfinite(o->lambdas[n]))
      fail(PASD_ERR_ARGUMENT, "config: lambda of mode " + std::to_string(n + 1) + " must be positive");
  if (!o->ranks) fail(PASD_ERR_ARGUMENT, "config: expected " + std::to_string(n_modes) + " ranks, got 0");
  for (size_t n = 0; n < n_modes; ++n) {
    if (o->ranks[n] < 1) fail(PASD_ERR_ARGUMENT, "config: rank of mode " + std::to_string(n + 1) + " must be positive");
    if (o->ranks[n] > dims[n])
      fail(PASD_ERR_ARGUMENT, "config: rank " + std::to_string(o->ranks[n]) + " exceeds dimension " +
                                  std::to_string(dims[n]) + " in mode " + std::to_string(n + 1));
  }
  if (!(o->mu0 > 0.0) || !std::isfinite(o->mu0)) fail(PASD_ERR_ARGUMENT, "config: mu0 must be positive");
  if (!(o->mu_max >= o->mu0)) fail(PASD_ERR_ARGUMENT, "config: mu_max must be at least mu0");
  if (!(o->rho > 1.0) || !std::isfinite(o->rho)) fail(PASD_ERR_ARGUMENT, "config: rho must exceed 1");
  if (!(o->eps > 0.0)) fail(PASD_ERR_ARGUMENT, "config: eps must be positive");
  if (o->maxiter < 1) fail(PASD_ERR_ARGUMENT, "config: maxiter must be positive");
  if (o->output_weights) {
    for (size_t n = 0; n < n_modes; ++n)
      if (!(o->output_weights[n] > 0.0) || !std::isfinite(o->output_weights[n]))
        fail(PASD_ERR_ARGUMENT, "config: output weight of mode " + std::to_string(n + 1) + " must be positive");
  }
  // Limits of this build (no reference analogue).
  if (o->order > PASD_MAX_ORDER)
    fail(PASD_ERR_ARGUMENT, "pasd_b200: order " + std::to_string(o->order) + " exceeds the supported maximum " +
                                std::to_string(PASD_MAX_ORDER));
  for (size_t n = 0; n < n_modes; ++n)
    if (o->ranks[n] > PASD_MAX_RANK)
      fail(PASD_ERR_ARGUMENT, "pasd_b200: rank " + std::to_string(o->ranks[n]) + " of mode " + std::to_string(n + 1) +
                                  " exceeds the supported maximum " + std::to_string(PASD_MAX_RANK));
}

// Guard-band allocations (env PASD_B200_GUARD=1).  compute-sanitizer is closed
// on this GPU pool, so out-of-bounds global writes are caught by 64 KB canary
// bands (0xFF bytes, i.e. NaN doubles, so a stray READ of a band poisons the
// result the parity checks compare) on both sides of every device buffer,
// verified when the buffer is freed; pasd_b200_guard_report() returns the
// counts.  Off by default (no cost).
constexpr size_t kGuardBytes = 1 << 16;
struct GuardState {
  std::mutex mu;
  std::vector<std::pair<char*, size_t>> live;  // (user pointer, bytes)
  long long checked = 0, violations = 0;
};
GuardState& guard_state() {
  static GuardState g;
  return g;
}
bool guard_on() {
  static const bool on = [] {
    const char* e = std::getenv("PASD_B200_GUARD");
    return e && e[0] == '1';
  }();
  return on;
}

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  const size_t bytes = count * sizeof(T);
  if (!guard_on()) {
    CK(cudaMalloc(&p, bytes));
    return static_cast<T*>(p);
  }
  CK(cudaMalloc(&p, bytes + 2 * kGuardBytes));
  char* raw = static_cast<char*>(p);
  CK(cudaMemset(raw, 0xFF, kGuardBytes));
  CK(cudaMemset(raw + kGuardBytes + bytes, 0xFF, kGuardBytes));
  CK(cudaDeviceSynchronize());
  GuardState& g = guard_state();
  std::lock_guard<std::mutex> lk(g.mu);
  g.live.emplace_back(raw + kGuardBytes, bytes);
  return reinterpret_cast<T*>(raw + kGuardBytes);
}

// cudaFree for dalloc'd buffers; in guard mode verifies both bands first.
void dfree(void* p) {
  if (!p) return;
  if (!guard_on()) {
    cudaFree(p);
    return;
  }
  GuardState& g = guard_state();
  size_t bytes = 0;
  {
    std::lock_guard<std::mutex> lk(g.mu);
    for (size_t k = 0; k < g.live.size(); ++k)
      if (g.live[k].first == p) {
        bytes = g.live[k].second;
        g.live.erase(g.live.begin() + (long)k);
        break;
      }
  }
  char* raw = static_cast<char*>(p) - kGuardBytes;
  std::vector<unsigned char> band(kGuardBytes);
  cudaDeviceSynchronize();
  int bad = 0;
  for (int side = 0; side < 2; ++side) {
    cudaMemcpy(band.data(), side ? raw + kGuardBytes + bytes : raw, kGuardBytes, cudaMemcpyDeviceToHost);
    for (unsigned char c : band)
      if (c != 0xFF) {
        bad = 1;
        break;
      }
  }
  {
    std::lock_guard<std::mutex> lk(g.mu);
    ++g.checked;
    g.violations += bad;
  }
  if (bad) std::fprintf(stderr, "pasd_b200: guard band overwritten around a %zu-byte buffer\n", bytes);
  cudaFree(raw);
}

int rpt_for(int R) { return R <= 8 ? 2 : R <= 16 ? 4 : R <= 32 ? 8 : 16; }

// The small solves' dynamic shared-memory cap is a per-(kernel, device)
// attribute shared by every solver in the process: set it once per device to
// the largest workspace this build supports (R = PASD_MAX_RANK), so a solver
// created later with a smaller rank can never lower it under an earlier one.
void ensure_small_smem_attr() {
  static std::mutex mu;
  static std::vector<char> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if ((int)done.size() <= dev) done.resize(dev + 1, 0);
  if (done[dev]) return;
  const int bytes = (int)small_ws_bytes(PASD_MAX_RANK);
  CK(cudaFuncSetAttribute(k_svt, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_polar, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[dev] = 1;
}

}  // namespace

// ============================================================================
struct pasd_solver {
  // configuration
  int N = 0;
  std::vector<int64_t> dims;
  int64_t S = 0;
  std::vector<int64_t> ranks;
  std::vector<double> lambdas, alphas;
  double mu0 = 1e-4, mu_max = 1e10, rho = 1.1, eps = 1e-5;
  int maxiter = 1000;
  uint32_t flags = 0;
  int poll_every = 8;
  int device = 0;
  // device state
  cudaStream_t stream = nullptr;
  double* T = nullptr;
  double* E[2] = {nullptr, nullptr};
  double* D = nullptr;  // T - E (pass 1 operand, written by the update pass)
  std::vector<double*> Y;
  std::vector<ModeDev> modes;
  std::vector<void*> owned;
  ModePack* d_pack = nullptr;
  ModePack h_pack{};
  Ctl* d_ctl = nullptr;
  Ctl* h_ctl = nullptr;  // pinned mirror
  double* d_hist = nullptr;
  double* d_resid_part = nullptr;
  int* d_bad_part = nullptr;
  int nblk_update = 0;
  int sms = 148;
  size_t small_smem = 0;
  // all-modes Gram launches (unsharded)
  int gram_rp = 0, gram_grid = 0, gram_red_grid = 0;
  // fused order-3 pass 2 (pasd_pass2.cuh)
  bool fused = false;
  bool use_m8 = false;
  bool p2_bulk = false;  // k_pass2_fused stages its slices from the tiled copies (PASD_P2_BULK)
  bool p2_ts = false;    // two-team kernel k_pass2_ts (pasd_pass2ts.cuh) instead of k_pass2_fused
  int p2_rp = 0;
  Pass2Args p2{};
  int p2_grid = 0;
  size_t p2_smem = 0;
  bool p2_tio = false;  // element streams through TMA (k_pass2_fused<RP, true>)
  // PASD_FLAG_FP32: T, E, D, Y_n stored as float32 (the double* members then
  // point at float storage); small state and all arithmetic stay fp64
  bool f32 = false;
  size_t esz = sizeof(double);
  double* ebuf = nullptr;  // fp32 mode: S float64 scratch for conversions on the way out
  P2Tmaps p2_tmaps{};
  double* p2_resid = nullptr;
  int* p2_bad = nullptr;
  double* zbuf = nullptr;  // S scratch (finalisation / observer)
  double* xbuf = nullptr;  // S scratch
  double* d_stats = nullptr;
  int* d_flag = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaGraph_t graph = nullptr;
  // poll_every iterations captured back to back in one graph (one launch per
  // polling period; opt-in PASD_GRAPH_UNROLL=1: measured slower on the device
  // at C1 / C2, 0.101 -> 0.123 / 0.428 -> 0.441 ms per iteration, for ~2% less
  // host time end to end)
  cudaGraphExec_t graph_exec_k = nullptr;
  cudaGraph_t graph_k = nullptr;
  int graph_k_iters = 0;
  int64_t launches_last_run = 0;
  int launches_per_iter = 0;
  bool loaded = false;
  // slab sharding along the last mode (one process per GPU)
  bool sharded = false;
  int rank = 0, nranks = 1;
  int64_t slab_b = 0, slab_e = 0;
  std::vector<int64_t> gdims;  // global dims (dims = local slab dims)
  std::unique_ptr<Comm> comm;     // NCCL (one GPU per rank) or loopback (ranks share one GPU)
  LoopbackGroup* loop_group = nullptr;
  bool check_replicas = false;    // PASD_FLAG_CHECK_REPLICAS: cross-rank hash of U_n / M_n per run
  cudaStream_t side = nullptr;  // A_3 all-reduce, overlapped with pass 1 of modes 1 and 2
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // finalisation: D2H of E on its own stream, overlapping the X materialisation
  cudaStream_t xfer = nullptr;
  cudaEvent_t ev_xfork = nullptr, ev_xjoin = nullptr;
  // unsharded graph: pass 1 of the N modes as concurrent branches (small tensors
  // otherwise leave most SMs idle in each mode's single wave of tiles)
  cudaStream_t p1s[PASD_MAX_ORDER] = {};
  cudaEvent_t ev_p1fork = nullptr, ev_p1join[PASD_MAX_ORDER] = {};
  double* A3_partial = nullptr;
  std::vector<double*> gram_partial, wt_partial;
  double* g2_partial = nullptr;
  double* red_local = nullptr;
  double* red = nullptr;

  ~pasd_solver() {
    comm.reset();
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (ev_xfork) cudaEventDestroy(ev_xfork);
    if (ev_xjoin) cudaEventDestroy(ev_xjoin);
    if (xfer) cudaStreamDestroy(xfer);
    if (ev_p1fork) cudaEventDestroy(ev_p1fork);
    for (int n = 0; n < PASD_MAX_ORDER; ++n) {
      if (ev_p1join[n]) cudaEventDestroy(ev_p1join[n]);
      if (p1s[n]) cudaStreamDestroy(p1s[n]);
    }
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (graph_exec_k) cudaGraphExecDestroy(graph_exec_k);
    if (graph_k) cudaGraphDestroy(graph_k);
    if (graph) cudaGraphDestroy(graph);
    for (void* p : owned) dfree(p);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (stream) cudaStreamDestroy(stream);
  }

  template <class T>
  T* alloc(size_t count) {
    T* p = dalloc<T>(count);
    owned.push_back(p);
    return p;
  }
};

namespace {

double* ctl_gnorm2(pasd_solver* s) {  // device address of ctl->gnorm2[0]
  return reinterpret_cast<double*>(reinterpret_cast<char*>(s->d_ctl) + offsetof(Ctl, gnorm2));
}

template <class EL>
EL* as_el(double* p) {
  return reinterpret_cast<EL*>(p);
}
// pass 1 of one mode on the solver's element storage (float64, or float32 in the fp32 mode)
void launch_p1_any(pasd_solver* s, const ModeDev& m, double* Y, int sms, cudaStream_t st) {
  if (s->f32)
    launch_contract_A_mma(m, as_el<float>(s->D), as_el<float>(Y), s->d_ctl, sms, st);
  else
    launch_contract_A_mma(m, (const double*)s->D, (const double*)Y, s->d_ctl, sms, st);
}

// Launches one iteration.  `mark(cls, begin)` (optional) is called around
// every kernel; the profiler records CUDA events there.
template <class Mark>
void launch_iteration_marked(pasd_solver* s, cudaStream_t st, Mark&& mark, bool concurrent = false) {
  const int N = s->N;
  int launches = 0;
  bool retiled_a = false;  // the A tiles of the bulk-staged pass 2 were written on a branch
  if (!s->sharded && concurrent) {
    // Graph capture, unsharded: the Procrustes step (U_n) and pass 1 (A_n from D,
    // Y_n, U_n) are per mode, so each mode is one branch and the branches share
    // the SMs (small tensors leave most SMs idle in any single mode's kernels).
    CK(cudaEventRecord(s->ev_p1fork, st));
    for (int n = 0; n < N; ++n) {
      cudaStream_t bs = s->p1s[n];
      const ModeDev& m = s->modes[n];
      CK(cudaStreamWaitEvent(bs, s->ev_p1fork, 0));
      k_polar<<<kSmallCluster, kSmallThreads, s->small_smem, bs>>>(s->d_pack, s->d_ctl, n);
      launch_p1_any(s, m, s->Y[n], s->sms, bs);
      CK(cudaEventRecord(s->ev_p1join[n], bs));
      launches += 2;
    }
    for (int n = 0; n < N; ++n) CK(cudaStreamWaitEvent(st, s->ev_p1join[n], 0));
    if (s->fused && s->p2_bulk && !s->use_m8) {
      // the A tiles of pass 2 only need pass 1: retiled on a branch next to the Gram products and the SVTs
      // (HBM-bound copy next to tensor-bound / latency-bound kernels); the UM_2 tiles follow the SVT
      CK(cudaEventRecord(s->ev_p1fork, st));
      CK(cudaStreamWaitEvent(s->p1s[0], s->ev_p1fork, 0));
      retile_launch(s->p2_rp, s->p2, s->d_ctl, s->p1s[0], 1);
      CK(cudaEventRecord(s->ev_p1join[0], s->p1s[0]));
      ++launches;
      retiled_a = true;
    }
    // all modes' Gram partials, reductions and SVTs in three launches (per-mode
    // Gram / SVT branches measured slower: more, smaller launches)
    launch_gram_all(s->gram_rp, s->d_pack, s->d_ctl, s->gram_grid, st);
    k_gram_reduce_all<<<s->gram_red_grid, 256, 0, st>>>(s->d_pack, s->d_ctl);
    k_svt<<<N * kSmallCluster, kSmallThreads, s->small_smem, st>>>(s->d_pack, s->d_ctl);
    launches += 3;
    if (retiled_a) CK(cudaStreamWaitEvent(st, s->ev_p1join[0], 0));
  } else {
    mark(PASD_K_POLAR, true);
    k_polar<<<N * kSmallCluster, kSmallThreads, s->small_smem, st>>>(s->d_pack, s->d_ctl);
    mark(PASD_K_POLAR, false);
    ++launches;
    if (!s->sharded) {
      for (int n = 0; n < N; ++n) {
        mark(PASD_K_CONTRACT_A, true);
        launch_p1_any(s, s->modes[n], s->Y[n], s->sms, st);
        mark(PASD_K_CONTRACT_A, false);
        ++launches;
      }
    } else {
      // Mode 3 first: its slab partial A_3 (the one large exchange, R_3 I_1 I_2 doubles) is
      // all-reduced on the side stream while pass 1 of modes 1 and 2 runs on SMs left free
      // for NCCL's kernel; the main stream joins before the Gram products.
      ModeDev m3 = s->modes[N - 1];
      m3.A = s->A3_partial;
      mark(PASD_K_CONTRACT_A, true);
      launch_p1_any(s, m3, s->Y[N - 1], s->sms, st);
      mark(PASD_K_CONTRACT_A, false);
      ++launches;
      CK(cudaEventRecord(s->ev_fork, st));
      CK(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
      s->comm->allreduce(s->A3_partial, s->modes[N - 1].A, (size_t)m3.J * m3.R, RedOp::Sum, s->side);
      CK(cudaEventRecord(s->ev_join, s->side));
      const int sms_p1 = std::max(1, s->sms - kNcclSms);
      for (int n = 0; n < N - 1; ++n) {
        mark(PASD_K_CONTRACT_A, true);
        launch_p1_any(s, s->modes[n], s->Y[n], sms_p1, st);
        mark(PASD_K_CONTRACT_A, false);
        ++launches;
      }
      CK(cudaStreamWaitEvent(st, s->ev_join, 0));
    }
    if (!s->sharded) {
      // all modes' Gram partials, then all reductions (pasd_gram.cuh), then the SVTs
      mark(PASD_K_GRAM, true);
      launch_gram_all(s->gram_rp, s->d_pack, s->d_ctl, s->gram_grid, st);
      k_gram_reduce_all<<<s->gram_red_grid, 256, 0, st>>>(s->d_pack, s->d_ctl);
      mark(PASD_K_GRAM, false);
      mark(PASD_K_SVT, true);
      k_svt<<<N * kSmallCluster, kSmallThreads, s->small_smem, st>>>(s->d_pack, s->d_ctl);
      mark(PASD_K_SVT, false);
      launches += 3;
    } else {
      for (int n = 0; n < N; ++n) {
        const ModeDev& m = s->modes[n];
        mark(PASD_K_GRAM, true);
        launch_gram_mma(m, s->d_ctl, st);
        const bool part = n < N - 1;  // Gram_1, Gram_2 are partial over the slab
        k_gram_reduce<<<8, 256, 0, st>>>(m, part ? s->gram_partial[n] : m.Gram, s->d_ctl);
        mark(PASD_K_GRAM, false);
        launches += 2;
      }
      s->comm->group_start();
      for (int n = 0; n < N - 1; ++n) {
        const ModeDev& m = s->modes[n];
        s->comm->allreduce(s->gram_partial[n], m.Gram, (size_t)m.R * m.R, RedOp::Sum, st);
      }
      s->comm->group_end();
      mark(PASD_K_SVT, true);
      k_svt<<<N * kSmallCluster, kSmallThreads, s->small_smem, st>>>(s->d_pack, s->d_ctl);
      mark(PASD_K_SVT, false);
      ++launches;
    }
  }  // per-mode branches / sequential launches
  if (s->fused) {
    mark(PASD_K_UPDATE, true);
    if (s->use_m8)
      m8_launch(s->p2_rp, s->p2, s->d_ctl, s->p2_grid, st, s->f32);
    else {
      if (s->p2_bulk) {
        retile_launch(s->p2_rp, s->p2, s->d_ctl, st, retiled_a ? 2 : 0);
        ++launches;
      }
      if (s->p2_ts)
        ts_launch(s->p2_rp, s->f32, s->p2, s->d_ctl, s->p2_grid, st);
      else
        pass2_launch(s->p2_rp, s->p2_tio, s->p2, s->d_ctl, s->p2_tmaps, s->p2_grid, st, s->f32);
    }
    mark(PASD_K_UPDATE, false);
    ++launches;
    int64_t maxir = 1;
    for (const ModeDev& m : s->modes) maxir = std::max<int64_t>(maxir, m.Ifull * m.R);
    mark(PASD_K_CONTRACT_W, true);
    k_pass2_reduce<<<dim3((unsigned)std::min<int64_t>((maxir + 7) / 8, 8 * s->sms), 3), 256, 0, st>>>(
        s->p2, s->p2_grid, s->d_ctl, s->sharded ? s->g2_partial : ctl_gnorm2(s));
    mark(PASD_K_CONTRACT_W, false);
    ++launches;
    if (s->sharded) {
      k_resid_local<<<1, kThreads, 0, st>>>(s->d_ctl, s->p2_resid, s->p2_bad, s->p2_grid, s->red_local);
      ++launches;
      s->comm->group_start();
      for (int n = 0; n < N; ++n) {
        const ModeDev& m = s->modes[n];
        s->comm->allreduce(s->wt_partial[n], m.Wt, (size_t)m.Ifull * m.R, RedOp::Sum, st);
      }
      s->comm->allreduce(s->g2_partial, ctl_gnorm2(s), (size_t)N, RedOp::Sum, st);
      s->comm->allreduce(s->red_local, s->red, (size_t)N + 1, RedOp::Max, st);
      s->comm->group_end();
    }
    if (s->sharded) {
      mark(PASD_K_FINISH, true);
      k_finish<<<1, kThreads, 0, st>>>(s->d_ctl, s->p2_resid, s->p2_bad, s->p2_grid, s->d_hist, s->red);
      mark(PASD_K_FINISH, false);
      ++launches;
    }
  } else {
    mark(PASD_K_UPDATE, true);
    k_update<<<s->nblk_update, kThreads, 0, st>>>(s->d_pack, s->T, s->E[0], s->E[1], s->D, s->d_resid_part,
                                                  s->d_bad_part, s->S, s->d_ctl);
    mark(PASD_K_UPDATE, false);
    ++launches;
    mark(PASD_K_FINISH, true);
    k_finish<<<1, kThreads, 0, st>>>(s->d_ctl, s->d_resid_part, s->d_bad_part, s->nblk_update, s->d_hist, nullptr);
    mark(PASD_K_FINISH, false);
    ++launches;
    for (int n = 0; n < N; ++n) {
      const ModeDev& m = s->modes[n];
      const dim3 grid(m.nkc_w, m.nib_w);
      mark(PASD_K_CONTRACT_W, true);
      switch (rpt_for(m.R)) {
        case 2: k_contract_W<2><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
        case 4: k_contract_W<4><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
        case 8: k_contract_W<8><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
        default: k_contract_W<16><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
      }
      mark(PASD_K_CONTRACT_W, false);
      ++launches;
    }
    mark(PASD_K_CONTRACT_W, true);
    k_wreduce_generic<<<dim3(64, N), 256, 0, st>>>(s->d_pack, s->d_ctl);
    mark(PASD_K_CONTRACT_W, false);
    ++launches;
  }
  s->launches_per_iter = launches;
  CK(cudaGetLastError());
}

void launch_iteration(pasd_solver* s, cudaStream_t st) {
  static const bool seq = std::getenv("PASD_P1_SEQUENTIAL") != nullptr;  // A/B switch
  launch_iteration_marked(s, st, [](int, bool) {}, !seq);
}

// Algorithmic bytes / flops of one launch of each kernel class summed over
// modes: the data the kernel's function must touch once.
void kernel_work(const pasd_solver* s, double* bytes, double* flops) {
  const double S = (double)s->S, N = (double)s->N;
  const double es = (double)s->esz;  // bytes per element-tensor entry (8, or 4 in the fp32 mode)
  for (int k = 0; k < PASD_NUM_KERNEL_CLASSES; ++k) bytes[k] = flops[k] = 0.0;
  for (const ModeDev& m : s->modes) {
    const double RJ = (double)m.R * (double)m.J, R = m.R;
    bytes[PASD_K_CONTRACT_A] += es * 2.0 * S + 8.0 * RJ;     // D = T - E, Y_n in; A_n out
    flops[PASD_K_CONTRACT_A] += 2.0 * R * S;
    bytes[PASD_K_GRAM] += 8.0 * RJ;                         // A_n in
    flops[PASD_K_GRAM] += 2.0 * R * RJ;
    bytes[PASD_K_UPDATE] += 8.0 * RJ;                       // A_n in
    flops[PASD_K_UPDATE] += 2.0 * R * S;
    bytes[PASD_K_CONTRACT_W] += es * 3.0 * S + 8.0 * RJ;    // T, E, Y_n, A_n in
    flops[PASD_K_CONTRACT_W] += 2.0 * R * S;
    bytes[PASD_K_POLAR] += 8.0 * 4.0 * (double)m.I * R;
    bytes[PASD_K_SVT] += 8.0 * 2.0 * (double)m.I * R;
  }
  bytes[PASD_K_UPDATE] += es * (2.0 * N + 3.0) * S;          // T, Y_1..N in; E, D, Y_1..N out
  if (s->fused) {  // pass 2 also forms Wt_n = G^{next} A_n^T (A_n already counted)
    for (const ModeDev& m : s->modes) {
      flops[PASD_K_UPDATE] += 2.0 * (double)m.R * S;
      bytes[PASD_K_CONTRACT_W] = 0.0;
      flops[PASD_K_CONTRACT_W] = 0.0;
    }
  }
}

__global__ void k_init_state(ModePack* mp, Ctl* ctl, double mu0, double rho, double mu_max, double eps, int maxiter,
                             int fixed) {
  const int N = mp->order;
  for (int n = 0; n < N; ++n) {
    ModeDev& m = mp->m[n];
    const int64_t IR = m.Ifull * m.R;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < IR; idx += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = idx % m.Ifull, r = idx / m.Ifull;
      m.U[idx] = (i == r) ? 1.0 : 0.0;  // Matrix::Identity(rows, rank) (pasd.cpp:152)
      m.UM[idx] = 0.0;
    }
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)m.R * m.R;
         idx += (int64_t)gridDim.x * blockDim.x) {
      m.M[idx] = 0.0;  // V = 0 (pasd.cpp:153) <=> M = 0
      const double id = (idx % (m.R + 1) == 0) ? 1.0 : 0.0;
      m.P[idx] = id;   // warm starts of the eigen-solvers
      m.Qp[idx] = id;
    }
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < m.Ifull * m.R;
         idx += (int64_t)gridDim.x * blockDim.x)
      m.Wt[idx] = 0.0;  // Wt = G V^T = 0 for V = 0: first Procrustes is degenerate
    const int64_t wp = (int64_t)m.nkc_w * m.I * m.R;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < wp; idx += (int64_t)gridDim.x * blockDim.x)
      m.Wpart[idx] = 0.0;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)m.nkc_w * m.nib_w;
         idx += (int64_t)gridDim.x * blockDim.x)
      m.gpart[idx] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->mu = mu0;
    ctl->mu_used_last = mu0;
    ctl->rho = rho;
    ctl->mu_max = mu_max;
    ctl->eps = eps;
    ctl->iter = 0;
    ctl->maxiter = maxiter;
    ctl->done = 0;
    ctl->converged = 0;
    ctl->nan_flag = 0;
    ctl->ecur = 0;
    ctl->fixed_iters = fixed;
    ctl->order = N;
    for (int n = 0; n < PASD_MAX_ORDER; ++n) {
      ctl->resid[n] = CUDART_INF;
      ctl->gnorm2[n] = 0.0;
      ctl->vnorm2[n] = 0.0;
      ctl->nuclear[n] = 0.0;
      ctl->keep[n] = 0;
      ctl->degenerate[n] = 0;
      ctl->polar_rank[n] = 0;
    }
  }
}

// copy_d = false when a new tensor is loaded next (load_tensor forms D = T - E itself)
void reset_state(pasd_solver* s, bool copy_d = true) {
  CK(cudaMemsetAsync(s->E[0], 0, s->S * s->esz, s->stream));
  CK(cudaMemsetAsync(s->E[1], 0, s->S * s->esz, s->stream));
  for (int n = 0; n < s->N; ++n) CK(cudaMemsetAsync(s->Y[n], 0, s->S * s->esz, s->stream));
  if (copy_d)
    CK(cudaMemcpyAsync(s->D, s->T, s->S * s->esz, cudaMemcpyDeviceToDevice, s->stream));  // D = T - 0
  k_init_state<<<64, 256, 0, s->stream>>>(s->d_pack, s->d_ctl, s->mu0, s->rho, s->mu_max, s->eps, s->maxiter,
                                          (s->flags & PASD_FLAG_FIXED_ITERS) ? 1 : 0);
  CK(cudaGetLastError());
}

// 3-D float64 tensor map with a 16 x 8 x 8 box and 128-byte swizzle (pass-2
// element bricks); dims / byte strides as given (dimension 0 contiguous).
// cuTensorMapEncodeTiled comes from the driver entry point, so the library
// does not link libcuda.
void encode_brick_map(CUtensorMap* map, double* base, const std::vector<int64_t>& dims,
                      const std::vector<int64_t>& strides) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) fail(PASD_ERR_CUDA, "pasd_b200: cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t gdim[3] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2]};
  const cuuint64_t gstride[2] = {(cuuint64_t)strides[0], (cuuint64_t)strides[1]};
  const cuuint32_t box[3] = {P2_B1, P2_B2, P2_B3};
  const cuuint32_t estride[3] = {1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, gdim, gstride, box, estride,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(PASD_ERR_CUDA, "pasd_b200: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

bool trace_on() {
  static const bool on = std::getenv("PASD_B200_TRACE") != nullptr;
  return on;
}
double trace_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

pasd_solver* create_solver(const pasd_options* o, const pasd_shard* shard) {
  const double tc0 = trace_on() ? trace_ms() : 0.0;
  validate_options(o);
  auto s = std::make_unique<pasd_solver>();
  s->N = o->order;
  s->dims.assign(o->dims, o->dims + o->order);
  s->gdims = s->dims;
  if (shard) {  // slab along the last mode
    if (o->order != 3) fail(PASD_ERR_ARGUMENT, "pasd_b200: slab sharding supports order-3 tensors only");
    if (shard->nranks < 1 || shard->rank < 0 || shard->rank >= shard->nranks)
      fail(PASD_ERR_ARGUMENT, "pasd_b200: invalid rank/nranks");
    if (!(0 <= shard->slab_begin && shard->slab_begin < shard->slab_end && shard->slab_end <= s->dims[2]))
      fail(PASD_ERR_ARGUMENT, "pasd_b200: slab [" + std::to_string(shard->slab_begin) + ", " +
                                  std::to_string(shard->slab_end) + ") outside mode 3 of size " +
                                  std::to_string(s->dims[2]));
    for (int n = 0; n < 3; ++n)
      if (o->ranks[n] > PASD_MAX_RANK) fail(PASD_ERR_ARGUMENT, "pasd_b200: rank exceeds 64");
    s->sharded = true;
    s->rank = shard->rank;
    s->nranks = shard->nranks;
    s->slab_b = shard->slab_begin;
    s->slab_e = shard->slab_end;
    s->dims[2] = s->slab_e - s->slab_b;
  }
  s->S = dims_product(s->dims);
  s->ranks.assign(o->ranks, o->ranks + o->order);
  s->lambdas.assign(o->lambdas, o->lambdas + o->order);
  if (o->output_weights)
    s->alphas.assign(o->output_weights, o->output_weights + o->order);
  else
    s->alphas = s->lambdas;  // PasdConfig::alphas (pasd.hpp:26)
  s->mu0 = o->mu0;
  s->mu_max = o->mu_max;
  s->rho = o->rho;
  s->eps = o->eps;
  s->maxiter = o->maxiter;
  s->flags = o->flags;
  s->f32 = (o->flags & PASD_FLAG_FP32) != 0;
  s->esz = s->f32 ? sizeof(float) : sizeof(double);
  if (s->f32 && s->N != 3) fail(PASD_ERR_ARGUMENT, "pasd_b200: the fp32 mode supports order-3 tensors");
  s->poll_every = o->poll_every > 0 ? o->poll_every : 8;
  s->device = o->device;
  CK(cudaSetDevice(s->device));
  CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s->xfer, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&s->ev_xfork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s->ev_xjoin, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s->ev_p1fork, cudaEventDisableTiming));
  for (int n = 0; n < s->N; ++n) {
    CK(cudaStreamCreateWithFlags(&s->p1s[n], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&s->ev_p1join[n], cudaEventDisableTiming));
  }
  const int64_t S = s->S;
  // element tensors: S float64, or S float32 in the fp32 mode (held through double*)
  auto elem = [&]() { return s->f32 ? reinterpret_cast<double*>(s->alloc<float>(S)) : s->alloc<double>(S); };
  s->T = elem();
  s->E[0] = elem();
  s->E[1] = elem();
  s->D = elem();
  for (int n = 0; n < s->N; ++n) s->Y.push_back(elem());
  int maxR = 1;
  for (int n = 0; n < s->N; ++n) {
    ModeDev m{};
    m.mode = n;
    m.I = s->dims[n];
    m.inner = 1;
    for (int l = 0; l < n; ++l) m.inner *= s->dims[l];
    m.outer = 1;
    for (int l = n + 1; l < s->N; ++l) m.outer *= s->dims[l];
    m.J = m.inner * m.outer;
    m.Ifull = s->gdims[n];
    m.ioff = (s->sharded && n == s->N - 1) ? s->slab_b : 0;
    m.R = (int)s->ranks[n];
    maxR = std::max(maxR, m.R);
    m.lambda = s->lambdas[n];
    const int64_t IR = m.I * m.R, RR = (int64_t)m.R * m.R, IRf = m.Ifull * m.R;
    m.U = s->alloc<double>(IRf);
    m.UM = s->alloc<double>(IRf);
    m.M = s->alloc<double>(RR);
    m.A = s->alloc<double>((size_t)m.J * m.R);
    m.Wt = s->alloc<double>(IRf);
    m.nib_w = (int)((m.I + CW_IT - 1) / CW_IT);
    const int64_t kchunks = (m.J + CW_KC - 1) / CW_KC;
    m.nkc_w = (int)std::max<int64_t>(1, std::min<int64_t>(kchunks, std::max(1, 592 / m.nib_w)));
    m.Wpart = s->alloc<double>((size_t)m.nkc_w * IR);
    m.gpart = s->alloc<double>((size_t)m.nkc_w * m.nib_w);
    m.nkc_g = (int)std::max<int64_t>(1, std::min<int64_t>((m.J + GM_KC - 1) / GM_KC, 148));
    // slab partials of A_1, A_2 (sharded) cannot feed the SVT's small-value refinement
    m.refine_ok = !(s->sharded && n < s->N - 1);
    m.Gpart = s->alloc<double>((size_t)m.nkc_g * RR);
    m.Gram = s->alloc<double>(RR);
    m.sig = s->alloc<double>(m.R);
    m.P = s->alloc<double>(RR);
    m.Qp = s->alloc<double>(RR);
    m.scratch = s->alloc<double>(3 * IRf);
    s->modes.push_back(m);
  }
  if (s->sharded) {
    const ModeDev& m3 = s->modes[2];
    s->A3_partial = s->alloc<double>((size_t)m3.J * m3.R);
    for (int n = 0; n < 3; ++n) {
      const ModeDev& m = s->modes[n];
      s->gram_partial.push_back(s->alloc<double>((size_t)m.R * m.R));
      s->wt_partial.push_back(s->alloc<double>((size_t)m.Ifull * m.R));
    }
    s->g2_partial = s->alloc<double>(PASD_MAX_ORDER);
    s->red_local = s->alloc<double>(PASD_MAX_ORDER + 1);
    s->red = s->alloc<double>(PASD_MAX_ORDER + 1);
    if (shard->loopback) {  // ranks of one group share this device (pasd_comm.cuh)
      auto* g = reinterpret_cast<LoopbackGroup*>(shard->loopback);
      if (g->nranks != s->nranks)
        fail(PASD_ERR_ARGUMENT, "pasd_b200: loopback group of " + std::to_string(g->nranks) + " ranks, shard says " +
                                    std::to_string(s->nranks));
      s->comm = std::make_unique<LoopbackComm>(g, s->rank);
      s->loop_group = g;
    } else {
      ncclUniqueId id;
      if (shard->nccl_unique_id)
        std::memcpy(&id, shard->nccl_unique_id, sizeof(id));
      else if (s->nranks == 1)
        NK(ncclGetUniqueId(&id));
      else
        fail(PASD_ERR_ARGUMENT, "pasd_b200: nccl_unique_id is required for nranks > 1");
      s->comm = std::make_unique<NcclComm>(s->nranks, s->rank, id);
    }
    s->check_replicas = (o->flags & PASD_FLAG_CHECK_REPLICAS) != 0 || std::getenv("PASD_CHECK_REPLICAS") != nullptr;
    CK(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
  }
  std::memset(&s->h_pack, 0, sizeof(ModePack));
  s->h_pack.order = s->N;
  for (int n = 0; n < s->N; ++n) {
    s->h_pack.m[n] = s->modes[n];
    s->h_pack.Y[n] = s->Y[n];
  }
  s->d_pack = s->alloc<ModePack>(1);
  CK(cudaMemcpy(s->d_pack, &s->h_pack, sizeof(ModePack), cudaMemcpyHostToDevice));
  s->d_ctl = s->alloc<Ctl>(1);
  CK(cudaMallocHost(&s->h_ctl, sizeof(Ctl)));
  s->d_hist = s->alloc<double>(std::max(1, s->maxiter));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
  s->sms = sms;
  s->nblk_update = (int)std::max<int64_t>(1, std::min<int64_t>((S + kThreads - 1) / kThreads, (int64_t)sms * 8));
  s->d_resid_part = s->alloc<double>((size_t)s->nblk_update * PASD_MAX_ORDER);
  s->d_bad_part = s->alloc<int>(s->nblk_update);
  s->small_smem = small_ws_bytes(maxR);
  s->gram_rp = (maxR + 7) / 8 * 8;
  s->gram_grid = 0;
  int64_t gram_entries = 0;
  for (const ModeDev& m : s->modes) {
    s->gram_grid += m.nkc_g;
    gram_entries += (int64_t)m.R * m.R;
  }
  s->gram_red_grid = (int)std::min<int64_t>((gram_entries + 7) / 8, 8 * s->sms);  // one warp per entry
  ensure_small_smem_attr();
  if (s->N == 3) {
    s->fused = true;
    Pass2Args& a = s->p2;
    for (int n = 0; n < 3; ++n) {
      a.m[n] = s->modes[n];
      if (s->sharded) a.m[n].Wt = s->wt_partial[n];  // reduced across ranks by the comm
      a.Y[n] = s->Y[n];
    }
    a.T = s->T;
    a.E0 = s->E[0];
    a.E1 = s->E[1];
    a.D = s->D;
    s->p2_rp = pass2_rp(s->modes[0].R, s->modes[1].R, s->modes[2].R);
    s->use_m8 = (m8_supported(s->p2_rp) && std::getenv("PASD_PASS2_M16") == nullptr) || std::getenv("PASD_PASS2_M8") != nullptr;
    if (s->f32) s->use_m8 = m8_supported(s->p2_rp);  // float kernels exist for the default variant only
    a.b1 = s->use_m8 ? M8_B : P2_B1;
    a.n1b = (int)((s->dims[0] + a.b1 - 1) / a.b1);
    a.n3b = (int)((s->dims[2] + P2_B3 - 1) / P2_B3);
    a.npencils = a.n1b * a.n3b;
    // Split each pencil's i2 sweep into nseg segments when the pencil count
    // would leave the last wave of CTAs mostly empty (C1: 169 pencils on 296
    // slots of k_pass2_m8, C2: 625; C3: 1250 on 148 of k_pass2_fused).
    // Segments keep >= 4 steps each so the pencil-resident A_2 slice is reused.
    a.nseg = 1;
    const char* nseg_env = std::getenv("PASD_P2_NSEG");  // test hook: force the segment count (1..8)
    if (nseg_env && std::atoi(nseg_env) >= 1 && std::atoi(nseg_env) <= 8) {
      a.nseg = std::atoi(nseg_env);
    } else {
      const int slots = (s->use_m8 ? M8_CTAS : 1) * sms;
      const int64_t steps = (s->dims[1] + (s->use_m8 ? M8_B : P2_B2) - 1) / (s->use_m8 ? M8_B : P2_B2);
      // modelled time ~ waves x (steps per item + per-item overhead), the
      // overhead (pencil-resident staging, Wt_1 / Wt_3 partial reductions)
      // measured at ~2 steps for the 16x8x8 kernel and ~1 for the 8x8x8 one
      const double c0 = s->use_m8 ? 1.0 : 2.0;
      double best = 1e300;
      for (int sg = 1; sg <= 8 && (steps + sg - 1) / sg >= 4; ++sg) {
        if ((int64_t)(sg - 1) * ((steps + sg - 1) / sg) >= steps) continue;  // would leave the last segment empty
        const double waves = std::ceil((double)a.npencils * sg / slots);
        const double t = waves * ((double)((steps + sg - 1) / sg) + c0);
        if (t < best * 0.99) {  // fewer segments unless clearly better
          best = t;
          a.nseg = sg;
        }
      }
    }
    s->p2_grid = std::max(1, (int)std::min<int64_t>((int64_t)a.npencils * a.nseg, (s->use_m8 ? M8_CTAS : 1) * sms));
    // TMA element streams (PASD_P2_TIO=1; needs 16-byte global strides, i.e. I1 even, and the
    // bricks within 227 KB).  Parity-green but slower at C5 (45.7 vs 42.3 ms per launch: the
    // CTA moves to the 228 KB carve-out, the Wt_2/Wt_3 operands are formed from D and Y in the
    // fragment load, and L2 re-fetches of the A slices grow by 8.5 GB), so LDG/STG is the default.
    const char* tio_env = std::getenv("PASD_P2_TIO");
    s->p2_tio = !s->f32 && !s->use_m8 && (s->dims[0] % 2 == 0) && pass2_smem(s->p2_rp, true) <= 227u * 1024u &&
                (tio_env && tio_env[0] == '1');
    if (s->p2_tio) {
      const int64_t I1 = s->dims[0], I2 = s->dims[1], I3 = s->dims[2];
      const std::vector<int64_t> da = {I1, I2, I3}, db = {I1, I3, I2};
      const std::vector<int64_t> sa = {I1 * 8, I1 * I2 * 8}, sb = {I1 * I2 * 8, I1 * 8};
      encode_brick_map(&s->p2_tmaps.t, s->T, da, sa);
      encode_brick_map(&s->p2_tmaps.y1, s->Y[0], da, sa);
      encode_brick_map(&s->p2_tmaps.y2, s->Y[1], da, sa);
      encode_brick_map(&s->p2_tmaps.y3b, s->Y[2], db, sb);
      encode_brick_map(&s->p2_tmaps.y3a, s->Y[2], da, sa);
      encode_brick_map(&s->p2_tmaps.e0, s->E[0], da, sa);
      encode_brick_map(&s->p2_tmaps.e1, s->E[1], da, sa);
      encode_brick_map(&s->p2_tmaps.d, s->D, da, sa);
    }
    s->p2_smem = s->use_m8 ? 0 : pass2_smem(s->p2_rp, s->p2_tio);
    a.W1p = s->alloc<double>((size_t)a.npencils * a.nseg * a.b1 * s->modes[0].R);
    a.W3p = s->alloc<double>((size_t)a.npencils * a.nseg * 8 * s->modes[2].R);
    // Wt_2 partials: one per K-half of each CTA while they stay small next to L2
    // (C3 38 MB, C4 18 MB: one barrier per step fewer, -2..5% pass 2); at C5 the
    // 118 MB they would take thrash L2 (+1 ms), so one per CTA there.
    const double w2_split_bytes = 2.0 * s->p2_grid * (double)s->dims[1] * s->modes[1].R * sizeof(double);
    s->p2_bulk = !s->use_m8 && !s->p2_tio && pass2_bulk<false>();
    a.n2b = (int)((s->dims[1] + P2_B2 - 1) / P2_B2);
    if (s->p2_bulk) {  // tiled, padded copies of A_n / UM_2 (k_retile), ~1.17x the bytes of A_n each
      const RetileSizes z = retile_sizes(s->p2_rp, a.n1b, a.n2b, a.n3b);
      a.At1 = s->alloc<double>(z.at1);
      a.At2 = s->alloc<double>(z.at2);
      a.At3 = s->alloc<double>(z.at3);
      a.U2t = s->alloc<double>(z.u2t);
    }
    const bool ws = !s->use_m8 && (!s->p2_tio || PASD_P2_TIL) && PASD_P2_WS && s->p2_rp >= 48 &&
                    !s->p2_bulk;  // pass2_ws<RP, TIO>()
    a.nw2 = (!s->use_m8 && !s->p2_tio && !ws && w2_split_bytes <= 48e6) ? 2 * s->p2_grid : s->p2_grid;
    a.W2part = s->alloc<double>((size_t)a.nw2 * s->dims[1] * s->modes[1].R);
    a.gpart = s->alloc<double>((size_t)s->p2_grid * 3);
    s->p2_resid = s->alloc<double>((size_t)s->p2_grid * PASD_MAX_ORDER);
    s->p2_bad = s->alloc<int>(s->p2_grid);
    a.resid_part = s->p2_resid;
    a.bad_part = s->p2_bad;
    a.history = s->d_hist;
    if (!s->sharded) {  // the last pass-2 CTA runs the finish (sharded: after the NCCL max-reduce)
      a.finish_ticket = s->alloc<int>(1);
      CK(cudaMemset(a.finish_ticket, 0, sizeof(int)));
    }
    {
      const char* ts_env = std::getenv("PASD_P2_TS");
      // opt-in (PASD_P2_TS=1): parity-green, measured slower (C5 47.2 vs 37.0 ms per launch)
      s->p2_ts = s->p2_bulk && PASD_P2_TS && ts_supported(s->p2_rp) && ts_env && ts_env[0] == '1';
    }
    if (s->use_m8)
      m8_setup(s->p2_rp);
    else
      pass2_setup(s->p2_rp);
    if (s->p2_ts) ts_setup(s->p2_rp);
    CK(cudaGetLastError());
  }
  s->d_stats = s->alloc<double>(2 * 2048);
  s->d_flag = s->alloc<int>(1);
  const double tc1 = trace_on() ? trace_ms() : 0.0;
  reset_state(s.get());
  CK(cudaStreamSynchronize(s->stream));
  if (trace_on())
    std::fprintf(stderr, "create_solver: buffers/streams %.2f ms, reset %.2f ms\n", tc1 - tc0, trace_ms() - tc1);
  return s.release();
}

void ensure_scratch(pasd_solver* s);

void build_graph(pasd_solver* s) {
  if (s->graph_exec) return;
  const double t0 = trace_on() ? trace_ms() : 0.0;
  CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  launch_iteration(s, s->stream);
  CK(cudaStreamEndCapture(s->stream, &s->graph));
  CK(cudaGraphInstantiate(&s->graph_exec, s->graph, 0));
  static const bool unroll = [] {
    const char* e = std::getenv("PASD_GRAPH_UNROLL");
    return e && e[0] == '1';
  }();
  if (unroll && s->poll_every > 1 && s->poll_every <= 64) {
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < s->poll_every; ++k) launch_iteration(s, s->stream);
    CK(cudaStreamEndCapture(s->stream, &s->graph_k));
    CK(cudaGraphInstantiate(&s->graph_exec_k, s->graph_k, 0));
    s->graph_k_iters = s->poll_every;
  }
  if (trace_on()) std::fprintf(stderr, "build_graph: %.2f ms\n", trace_ms() - t0);
}

void sync_ctl(pasd_solver* s) {
  CK(cudaMemcpyAsync(s->h_ctl, s->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
}

// Upload T on the transfer stream (forked from the solver stream's current
// point), so state resets queued on the solver stream afterwards overlap it.
void ensure_scratch(pasd_solver* s);

// fp32 mode: float64 input lands in the scratch zbuf and is rounded into T by load_tensor
double* upload_target(pasd_solver* s) {
  if (!s->f32) return s->T;
  ensure_scratch(s);
  return s->zbuf;
}

void begin_upload(pasd_solver* s, const double* t) {
  CK(cudaEventRecord(s->ev_xfork, s->stream));
  CK(cudaStreamWaitEvent(s->xfer, s->ev_xfork, 0));
  CK(cudaMemcpyAsync(upload_target(s), t, s->S * sizeof(double), cudaMemcpyHostToDevice, s->xfer));
  CK(cudaEventRecord(s->ev_xjoin, s->xfer));
}

// uploaded: T already issued by begin_upload (the solver stream joins it here)
void load_tensor(pasd_solver* s, const double* t, int is_device, bool uploaded = false) {
  double* t64 = upload_target(s);  // float64 copy of the input on the device
  if (uploaded)
    CK(cudaStreamWaitEvent(s->stream, s->ev_xjoin, 0));
  else if (!(s->f32 && is_device))
    CK(cudaMemcpyAsync(t64, t, s->S * sizeof(double), is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       s->stream));
  else
    t64 = const_cast<double*>(t);  // fp32 mode, device input: read it in place
  CK(cudaMemsetAsync(s->d_flag, 0, sizeof(int), s->stream));
  k_nonfinite<<<1184, 256, 0, s->stream>>>(t64, s->S, s->d_flag);
  if (s->f32) {
    k_to_float<<<1184, 256, 0, s->stream>>>(t64, as_el<float>(s->T), s->S);
    k_tsub<<<1184, 256, 0, s->stream>>>(as_el<float>(s->D), as_el<float>(s->T), as_el<float>(s->E[0]),
                                        as_el<float>(s->E[1]), s->S, s->d_ctl);
  } else {
    k_tsub<<<1184, 256, 0, s->stream>>>(s->D, s->T, s->E[0], s->E[1], s->S, s->d_ctl);  // keep D = T - E
  }
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, s->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (flag) fail(PASD_ERR_ARGUMENT, "pasd: input tensor contains non-finite entries");  // pasd.cpp:135-136
  s->loaded = true;
}

__global__ void k_state_ctl(Ctl* ctl, ModePack* mp, double mu, int iter, const double* vn2) {
  ctl->mu = mu;
  ctl->mu_used_last = mu;
  ctl->iter = iter;
  ctl->done = 0;
  ctl->converged = 0;
  ctl->nan_flag = 0;
  ctl->ecur = 0;
  for (int n = 0; n < mp->order; ++n) {
    ctl->vnorm2[n] = vn2[n];
    const int R = mp->m[n].R;
    for (int i = 0; i < R * R; ++i) mp->m[n].M[i] = (i % (R + 1) == 0) ? 1.0 : 0.0;  // M = I: V = A
  }
}

void set_state(pasd_solver* s, const double* e, const double* const* y, const double* const* u,
               const double* const* v, double mu, int iter) {
  if (!s->loaded) fail(PASD_ERR_STATE, "pasd_b200: no tensor loaded");
  if (s->sharded) fail(PASD_ERR_STATE, "pasd_b200: set_state is not available on a sharded solver");
  if (s->f32) fail(PASD_ERR_STATE, "pasd_b200: set_state is not available in the fp32 mode");
  if (!e || !y || !u || !v) fail(PASD_ERR_ARGUMENT, "pasd_b200: null state buffer");
  if (iter >= s->maxiter) fail(PASD_ERR_ARGUMENT, "pasd_b200: state iteration must be below maxiter");
  cudaStream_t st = s->stream;
  const int64_t S = s->S;
  CK(cudaMemcpyAsync(s->E[0], e, S * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(s->E[1], e, S * sizeof(double), cudaMemcpyHostToDevice, st));
  k_tsub<<<1184, 256, 0, st>>>(s->D, s->T, s->E[0], s->E[1], S, s->d_ctl);
  std::vector<double> vn2(s->N, 0.0);
  double* d_vn2 = s->d_stats;  // scratch (finalisation reuses it later)
  ensure_scratch(s);
  for (int n = 0; n < s->N; ++n) {
    const ModeDev& m = s->modes[n];
    CK(cudaMemcpyAsync(s->Y[n], y[n], S * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(m.U, u[n], m.I * m.R * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(s->xbuf, v[n], m.J * m.R * sizeof(double), cudaMemcpyHostToDevice, st));
    k_load_v_as_a<<<1184, 256, 0, st>>>(m, s->xbuf);
    k_sumsq<<<1, 1024, 0, st>>>(s->xbuf, m.J * m.R, d_vn2 + n);
  }
  k_state_ctl<<<1, 1, 0, st>>>(s->d_ctl, s->d_pack, mu, iter, d_vn2);
  // Wt_n = G_(n) V_n^T from the injected state (the product the next Procrustes needs)
  for (int n = 0; n < s->N; ++n) {
    const ModeDev& m = s->modes[n];
    const dim3 grid(m.nkc_w, m.nib_w);
    switch (rpt_for(m.R)) {
      case 2: k_contract_W<2><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
      case 4: k_contract_W<4><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
      case 8: k_contract_W<8><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
      default: k_contract_W<16><<<grid, kThreads, 0, st>>>(m, s->T, s->E[0], s->E[1], s->Y[n], s->d_ctl); break;
    }
  }
  k_wreduce_generic<<<dim3(64, s->N), 256, 0, st>>>(s->d_pack, s->d_ctl);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
}

// Observer snapshot (recovery.hpp:38-48): host copies of e, z, y, u, v.
struct HostView {
  std::vector<double> e;
  std::vector<std::vector<double>> z, y, u, v;
};

// A float64 view of an element tensor: itself, or (fp32 mode) its conversion into `scratch` on `st`.
const double* elem_f64(pasd_solver* s, const double* x, double* scratch, cudaStream_t st) {
  if (!s->f32) return x;
  k_to_double<<<1184, 256, 0, st>>>(reinterpret_cast<const float*>(x), scratch, s->S);
  CK(cudaGetLastError());
  return scratch;
}

void deliver_observer(pasd_solver* s, pasd_observer_fn fn, void* user, HostView& hv) {
  const int N = s->N;
  const int64_t S = s->S;
  const Ctl& c = *s->h_ctl;
  hv.e.resize(S);
  hv.z.resize(N);
  hv.y.resize(N);
  hv.u.resize(N);
  hv.v.resize(N);
  CK(cudaMemcpyAsync(hv.e.data(), elem_f64(s, s->E[c.ecur], s->ebuf, s->stream), S * sizeof(double),
                     cudaMemcpyDeviceToHost, s->stream));
  for (int n = 0; n < N; ++n) {
    const ModeDev& m = s->modes[n];
    hv.z[n].resize(S);
    hv.y[n].resize(S);
    hv.u[n].resize(m.I * m.R);
    hv.v[n].resize(m.J * m.R);
    k_materialize_z<<<1184, 256, 0, s->stream>>>(m, s->zbuf, S);
    CK(cudaMemcpyAsync(hv.z[n].data(), s->zbuf, S * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(hv.y[n].data(), elem_f64(s, s->Y[n], s->ebuf, s->stream), S * sizeof(double),
                       cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(hv.u[n].data(), m.U, m.I * m.R * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    k_materialize_v<<<1184, 256, 0, s->stream>>>(m, s->xbuf);
    CK(cudaMemcpyAsync(hv.v[n].data(), s->xbuf, m.J * m.R * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  }
  CK(cudaStreamSynchronize(s->stream));
  std::vector<const double*> zp, yp, up, vp;
  for (int n = 0; n < N; ++n) {
    zp.push_back(hv.z[n].data());
    yp.push_back(hv.y[n].data());
    up.push_back(hv.u[n].data());
    vp.push_back(hv.v[n].data());
  }
  pasd_iteration_view view{c.iter, c.mu_used_last, c.mu, c.resid, hv.e.data(), zp.data(), yp.data(), up.data(),
                           vp.data()};
  fn(&view, user);
}

void ensure_scratch(pasd_solver* s) {
  if (!s->zbuf) s->zbuf = s->alloc<double>(s->S);
  if (s->f32 && !s->ebuf) s->ebuf = s->alloc<double>(s->S);
  if (!s->xbuf) {
    int64_t need = s->S;
    for (const auto& m : s->modes) need = std::max<int64_t>(need, m.J * m.R);
    s->xbuf = s->alloc<double>(need);
  }
}

// Order-independent 64-bit hash of the replicated small state (U_n, M_n of
// every mode): sum over entries of bits * (2 idx + 1) mod 2^64.  Written as
// [hi, lo, -hi, -lo] (exact doubles) so one MAX all-reduce gives max and min.
__global__ void k_replica_hash(const ModePack* mp, double* out) {
  __shared__ unsigned long long acc;
  if (threadIdx.x == 0) acc = 0ull;
  __syncthreads();
  unsigned long long h = 0ull, base = 0ull;
  for (int n = 0; n < mp->order; ++n) {
    const ModeDev& m = mp->m[n];
    const int64_t nu = m.Ifull * m.R, nm = (int64_t)m.R * m.R;
    for (int64_t i = threadIdx.x; i < nu; i += blockDim.x)
      h += (unsigned long long)__double_as_longlong(m.U[i]) * (2ull * (base + i) + 1ull);
    base += nu;
    for (int64_t i = threadIdx.x; i < nm; i += blockDim.x)
      h += (unsigned long long)__double_as_longlong(m.M[i]) * (2ull * (base + i) + 1ull);
    base += nm;
  }
  atomicAdd(&acc, h);
  __syncthreads();
  if (threadIdx.x == 0) {
    const double hi = (double)(acc >> 32), lo = (double)(acc & 0xffffffffull);
    out[0] = hi;
    out[1] = lo;
    out[2] = -hi;
    out[3] = -lo;
  }
}

// Debug check of SURVEY 8(e): every rank holds bit-identical U_n and M_n.
void check_replicas(pasd_solver* s) {
  cudaStream_t st = s->stream;
  k_replica_hash<<<1, 256, 0, st>>>(s->d_pack, s->d_stats);
  s->comm->allreduce(s->d_stats, s->d_stats + 4, 4, RedOp::Max, st);
  double h[4];
  CK(cudaMemcpyAsync(h, s->d_stats + 4, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h[0] != -h[2] || h[1] != -h[3])
    fail(PASD_ERR_NUMERICAL, "pasd_b200: replicated U_n / M_n differ across ranks at iteration " +
                                 std::to_string(s->h_ctl->iter));
}

// Runs until stop or `iters` more iterations.
void run_solver(pasd_solver* s, int iters, pasd_observer_fn obs, void* user) {
  if (!s->loaded) fail(PASD_ERR_STATE, "pasd_b200: no tensor loaded");
  if (obs && s->sharded) fail(PASD_ERR_STATE, "pasd_b200: observers are not available on a sharded solver");
  sync_ctl(s);
  if (s->h_ctl->done) return;
  const bool eager = s->comm && !s->comm->capturable();  // loopback ranks: host-sequenced launches
  if (!eager) build_graph(s);
  HostView hv;
  if (obs) ensure_scratch(s);
  int launched = 0;
  s->launches_last_run = 0;
  while (launched < iters) {
    const int chunk = obs ? 1 : std::min(s->poll_every, iters - launched);
    if (!eager && s->graph_exec_k && chunk == s->graph_k_iters) {
      CK(cudaGraphLaunch(s->graph_exec_k, s->stream));  // the whole polling period in one launch
    } else {
      for (int k = 0; k < chunk; ++k) {
        if (eager)
          launch_iteration_marked(s, s->stream, [](int, bool) {});
        else
          CK(cudaGraphLaunch(s->graph_exec, s->stream));
      }
    }
    launched += chunk;
    s->launches_last_run += (int64_t)chunk * s->launches_per_iter;
    sync_ctl(s);
    const Ctl& c = *s->h_ctl;
    if (c.nan_flag)  // pasd.cpp:230-232
      fail(PASD_ERR_NUMERICAL, "pasd: non-finite iterate at iteration " + std::to_string(c.iter));
    if (obs) deliver_observer(s, obs, user, hv);
    if (c.done) break;
  }
  if (s->sharded && s->check_replicas) check_replicas(s);
}

void profile_solver(pasd_solver* s, int iters, double* ms, int64_t* cnt, double* bytes, double* flops) {
  if (!s->loaded) fail(PASD_ERR_STATE, "pasd_b200: no tensor loaded");
  for (int k = 0; k < PASD_NUM_KERNEL_CLASSES; ++k) {
    ms[k] = 0.0;
    cnt[k] = 0;
  }
  std::vector<cudaEvent_t> ev;
  std::vector<int> cls;
  auto mark = [&](int c, bool begin) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, s->stream));
    ev.push_back(e);
    if (begin) cls.push_back(c);
  };
  for (int it = 0; it < iters; ++it) launch_iteration_marked(s, s->stream, mark);
  CK(cudaStreamSynchronize(s->stream));
  for (size_t j = 0; j < cls.size(); ++j) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ev[2 * j], ev[2 * j + 1]));
    ms[cls[j]] += t;
    cnt[cls[j]] += 1;
  }
  for (cudaEvent_t e : ev) cudaEventDestroy(e);
  kernel_work(s, bytes, flops);
  sync_ctl(s);
  if (s->h_ctl->nan_flag)
    fail(PASD_ERR_NUMERICAL, "pasd: non-finite iterate at iteration " + std::to_string(s->h_ctl->iter));
}

void finalize_solver(pasd_solver* s, pasd_outputs* out) {
  sync_ctl(s);
  const Ctl c = *s->h_ctl;
  const int N = s->N;
  const int64_t S = s->S;
  ensure_scratch(s);
  cudaStream_t st = s->stream;
  const double* e = s->E[c.ecur];
  const double* ep = s->E[c.ecur ^ 1];
  const double mu_used = c.mu_used_last;
  // iteration bookkeeping
  out->iters = c.iter;
  out->converged = c.converged;
  if (out->residual_history && c.iter > 0)
    CK(cudaMemcpyAsync(out->residual_history, s->d_hist, c.iter * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (out->final_residuals)
    for (int n = 0; n < N; ++n) out->final_residuals[n] = c.resid[n];
  // X = weighted mean of Z_n (recovery.cpp:7-25) and optional Z_n
  double wsum = 0.0;
  for (double w : s->alphas) wsum += w;
  const int blocks = 1184;
  const bool want_x = out->x != nullptr;
  if (out->e) {  // E is final: its download overlaps the X materialisation below
    const double* e64 = elem_f64(s, e, s->ebuf, st);
    CK(cudaEventRecord(s->ev_xfork, st));
    CK(cudaStreamWaitEvent(s->xfer, s->ev_xfork, 0));
    CK(cudaMemcpyAsync(out->e, e64, S * sizeof(double), cudaMemcpyDeviceToHost, s->xfer));
    CK(cudaEventRecord(s->ev_xjoin, s->xfer));
  }
  for (int n = 0; n < N; ++n) {
    const bool want_z = out->z && out->z[n];
    if (!want_x && !want_z) continue;
    if (want_z) {
      k_materialize_z<<<blocks, 256, 0, st>>>(s->modes[n], s->zbuf, S);
      if (want_x) k_accum_x<<<blocks, 256, 0, st>>>(s->xbuf, s->zbuf, s->alphas[n] / wsum, n == 0, S);
      CK(cudaMemcpyAsync(out->z[n], s->zbuf, S * sizeof(double), cudaMemcpyDeviceToHost, st));
    } else {
      k_materialize_accum_x<<<blocks, 256, 0, st>>>(s->modes[n], s->xbuf, s->alphas[n] / wsum, n == 0, S);
    }
  }
  if (want_x) CK(cudaMemcpyAsync(out->x, s->xbuf, S * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (out->e) CK(cudaStreamWaitEvent(st, s->ev_xjoin, 0));
  // objective = ||E||_1 + sum_n lambda_n ||V_n||_*  (pasd.cpp:263-266)
  std::vector<double> sums(blocks), maxs(blocks);
  auto abs_stats = [&](const double* x, double* sum, double* mx, bool elem) {
    if (elem && s->f32)
      k_abs_stats<<<blocks, 256, 0, st>>>(reinterpret_cast<const float*>(x), S, s->d_stats, s->d_stats + 2048);
    else
      k_abs_stats<<<blocks, 256, 0, st>>>(x, S, s->d_stats, s->d_stats + 2048);
    CK(cudaMemcpyAsync(sums.data(), s->d_stats, blocks * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(maxs.data(), s->d_stats + 2048, blocks * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double a = 0.0, m = 0.0;
    for (int b = 0; b < blocks; ++b) {
      a += sums[b];
      m = std::max(m, maxs[b]);
    }
    if (sum) *sum = a;
    if (mx) *mx = m;
  };
  CK(cudaStreamSynchronize(st));
  double l1 = 0.0;
  abs_stats(e, &l1, nullptr, true);
  auto allreduce_scalar = [&](double v, RedOp op) {
    if (!s->sharded) return v;
    CK(cudaMemcpyAsync(s->d_stats, &v, sizeof(double), cudaMemcpyHostToDevice, st));
    s->comm->allreduce(s->d_stats, s->d_stats + 1, 1, op, st);
    double r = 0.0;
    CK(cudaMemcpyAsync(&r, s->d_stats + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return r;
  };
  l1 = allreduce_scalar(l1, RedOp::Sum);  // ||E||_1 over all slabs
  double obj = l1;
  for (int n = 0; n < N; ++n) obj += s->lambdas[n] * c.nuclear[n];
  out->objective = obj;
  // Yhat and certificate (pasd.cpp:246-258, 277-309)
  const bool want_cert = c.converged && !(s->flags & PASD_FLAG_NO_CERTIFICATE);
  for (int n = 0; n < N; ++n) {
    const bool want_yh = out->y_hat && out->y_hat[n];
    if (out->y && out->y[n])
      CK(cudaMemcpyAsync(out->y[n], elem_f64(s, s->Y[n], s->ebuf, st), S * sizeof(double), cudaMemcpyDeviceToHost,
                         st));
    if (!want_yh && !want_cert) continue;
    if (s->f32)
      k_yhat<<<blocks, 256, 0, st>>>(as_el<float>(s->Y[n]), reinterpret_cast<const float*>(e),
                                     reinterpret_cast<const float*>(ep), mu_used, s->zbuf,
                                     want_cert ? s->xbuf : nullptr, n == 0, S);
    else
      k_yhat<<<blocks, 256, 0, st>>>(s->Y[n], e, ep, mu_used, s->zbuf, want_cert ? s->xbuf : nullptr, n == 0, S);
    if (want_yh) CK(cudaMemcpyAsync(out->y_hat[n], s->zbuf, S * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  out->has_certificate = 0;
  out->cert_epsilon_hat = out->cert_c = out->cert_bound = 0.0;
  if (want_cert) {
    double eps_hat = 0.0, tl1 = 0.0;
    abs_stats(s->xbuf, nullptr, &eps_hat, false);
    abs_stats(s->T, &tl1, nullptr, true);
    eps_hat = allreduce_scalar(eps_hat, RedOp::Max);
    tl1 = allreduce_scalar(tl1, RedOp::Sum);
    const int k_star = c.iter - 1;
    const double geom = s->rho * (1.0 + s->rho) / (s->rho - 1.0) + 0.5 / std::pow(s->rho, k_star);
    double dim_sum = 0.0, lam_term = 0.0;
    double Sg = 1.0;
    for (int64_t d : s->gdims) Sg *= (double)d;
    for (int n = 0; n < N; ++n) {
      dim_sum += Sg;
      lam_term += s->lambdas[n] * Sg * s->eps;
    }
    const double nn = (double)N;
    const double cc = dim_sum * geom / (s->mu0 * nn * nn) + tl1;
    out->has_certificate = 1;
    out->cert_epsilon_hat = eps_hat;
    out->cert_c = cc;
    out->cert_bound = cc * eps_hat + lam_term;
  }
  CK(cudaStreamSynchronize(st));
}

int guarded_call(char* err, size_t errlen, const std::function<void()>& f) {
  try {
    f();
    return PASD_OK;
  } catch (const PasdError& e) {
    set_err(err, errlen, e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_err(err, errlen, "pasd_b200: host allocation failed");
    return PASD_ERR_CUDA;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return PASD_ERR_CUDA;
  }
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

int pasd_b200_abi_version(void) { return PASD_B200_ABI_VERSION; }

int pasd_b200_nccl_unique_id(void* out128, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!out128) fail(PASD_ERR_ARGUMENT, "pasd_b200: null output");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
  });
}

const char* pasd_b200_build_info(void) {
  return "pasd_b200 sm_100a fp64; kernels: polar,pass1,gram,svt,retile,pass2,finish,pass2_reduce; comm: nccl,loopback";
}

int pasd_b200_loopback_create(int32_t nranks, void** out, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null output handle");
    if (nranks < 1 || nranks > kLoopbackMaxRanks)
      fail(PASD_ERR_ARGUMENT, "pasd_b200: loopback groups hold 1.." + std::to_string(kLoopbackMaxRanks) + " ranks");
    *out = new LoopbackGroup(nranks);
  });
}

void pasd_b200_loopback_destroy(void* group) { delete reinterpret_cast<LoopbackGroup*>(group); }

#if PASD_P2_TIMING
// probe builds only: per-phase cycle sums of k_pass2_fused's warp 0 over all CTAs since the last call
extern "C" int pasd_b200_debug_p2_phases(double* out12) {
  unsigned long long h[12];
  if (cudaMemcpyFromSymbol(h, g_p2_phase, sizeof(h)) != cudaSuccess) return 5;
  const unsigned long long z[12] = {};
  cudaMemcpyToSymbol(g_p2_phase, z, sizeof(z));
  for (int k = 0; k < 12; ++k) out12[k] = (double)h[k];
  return 0;
}
#endif

int64_t pasd_b200_guard_report(int64_t* checked, int64_t* live) {
  GuardState& g = guard_state();
  std::lock_guard<std::mutex> lk(g.mu);
  if (checked) *checked = g.checked;
  if (live) *live = (int64_t)g.live.size();
  return g.violations;
}

int pasd_b200_validate(const pasd_options* opt, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] { validate_options(opt); });
}

int pasd_b200_default_lambdas(int32_t order, const int64_t* dims, double* out, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (order < 1 || !dims) fail(PASD_ERR_ARGUMENT, "tensor order must be at least 1");
    std::vector<int64_t> d(dims, dims + order);
    const int64_t total = dims_product(d);  // pasd.cpp:51-60
    const double n_modes = (double)order;
    for (int n = 0; n < order; ++n) {
      const double big = (double)std::max(d[n], total / d[n]);
      out[n] = std::sqrt(big) / n_modes;
    }
  });
}

int pasd_b200_default_rank_bound(int64_t target_rank, int64_t* out, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (target_rank < 1) fail(PASD_ERR_ARGUMENT, "target rank must be positive");  // pasd.cpp:62-66
    *out = (12 * target_rank) / 10;
  });
}

int pasd_b200_solver_create(const pasd_options* opt, const pasd_shard* shard, pasd_solver** out, char* errbuf,
                            size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null output handle");
    *out = create_solver(opt, shard);
  });
}

int pasd_b200_solver_load(pasd_solver* s, const double* t, int t_is_device, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!s || !t) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    CK(cudaSetDevice(s->device));
    load_tensor(s, t, t_is_device);
  });
}

int pasd_b200_solver_reset(pasd_solver* s, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!s) fail(PASD_ERR_ARGUMENT, "pasd_b200: null solver");
    CK(cudaSetDevice(s->device));
    reset_state(s);
    CK(cudaStreamSynchronize(s->stream));
  });
}

int pasd_b200_solver_run(pasd_solver* s, int32_t iters, int32_t* iters_done, int32_t* converged, char* errbuf,
                         size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!s) fail(PASD_ERR_ARGUMENT, "pasd_b200: null solver");
    CK(cudaSetDevice(s->device));
    try {
      run_solver(s, iters, nullptr, nullptr);
    } catch (...) {
      if (s->loop_group) s->loop_group->abort();  // release the other ranks' barriers
      throw;
    }
    if (iters_done) *iters_done = s->h_ctl->iter;
    if (converged) *converged = s->h_ctl->converged;
  });
}

int pasd_b200_solver_finalize(pasd_solver* s, pasd_outputs* out, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!s || !out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    CK(cudaSetDevice(s->device));
    try {
      finalize_solver(s, out);
    } catch (...) {
      if (s->loop_group) s->loop_group->abort();
      throw;
    }
  });
}

int pasd_b200_solver_set_state(pasd_solver* s, const double* e, const double* const* y, const double* const* u,
                               const double* const* v, double mu, int32_t iter, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!s) fail(PASD_ERR_ARGUMENT, "pasd_b200: null solver");
    CK(cudaSetDevice(s->device));
    set_state(s, e, y, u, v, mu, iter);
  });
}

int pasd_b200_solver_profile(pasd_solver* s, int32_t iters, double* kernel_ms, int64_t* kernel_launches,
                             double* kernel_bytes, double* kernel_flops, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!s || !kernel_ms || !kernel_launches || !kernel_bytes || !kernel_flops)
      fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    CK(cudaSetDevice(s->device));
    profile_solver(s, iters, kernel_ms, kernel_launches, kernel_bytes, kernel_flops);
  });
}

const double* pasd_b200_solver_device_e(const pasd_solver* s) {
  if (!s) return nullptr;
  return s->E[s->h_ctl ? s->h_ctl->ecur : 0];
}

void* pasd_b200_solver_stream(const pasd_solver* s) { return s ? (void*)s->stream : nullptr; }

int64_t pasd_b200_solver_launches(const pasd_solver* s) { return s ? s->launches_last_run : 0; }

int pasd_b200_solver_ranks(pasd_solver* s, int32_t* svt_keep, int32_t* polar_rank, char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!s || !svt_keep || !polar_rank) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    CK(cudaSetDevice(s->device));
    sync_ctl(s);
    for (int n = 0; n < s->N; ++n) {
      svt_keep[n] = s->h_ctl->keep[n];
      polar_rank[n] = s->h_ctl->polar_rank[n];
    }
  });
}

void pasd_b200_solver_destroy(pasd_solver* s) {
  if (s) {
    const double t0 = trace_on() ? trace_ms() : 0.0;
    cudaSetDevice(s->device);
    delete s;
    if (trace_on()) std::fprintf(stderr, "solver_destroy: %.2f ms\n", trace_ms() - t0);
  }
}

// Opt-in reuse (PASD_FLAG_REUSE_SOLVER): a one-shot solve may keep its solver
// (device buffers, captured graph) keyed on the complete options struct, so a
// repeated call with the same problem shape and options skips allocation,
// graph capture and teardown.  This is the library's only global state; it
// is never used unless the caller sets the flag, and it holds the solver's
// HBM (about (N+4) S doubles plus A_n: ~64 GB at 1000^3, R = 50) until
// pasd_b200_release_cache() or process exit.  On a miss the stale entry is
// freed BEFORE the new solver is allocated, so peak HBM is one solver.
namespace {
std::mutex g_cache_mu;
pasd_solver* g_cache = nullptr;
std::vector<char> g_cache_key;

std::vector<char> options_key(const pasd_options* o) {
  std::vector<char> k;
  auto put = [&](const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    k.insert(k.end(), c, c + n);
  };
  put(&o->order, sizeof(o->order));
  const int n = std::max(0, std::min<int>(o->order, PASD_MAX_ORDER));
  if (o->dims) put(o->dims, sizeof(int64_t) * n);
  if (o->ranks) put(o->ranks, sizeof(int64_t) * n);
  const char has_l = o->lambdas != nullptr, has_w = o->output_weights != nullptr;
  put(&has_l, 1);
  put(&has_w, 1);
  if (o->lambdas) put(o->lambdas, sizeof(double) * n);
  if (o->output_weights) put(o->output_weights, sizeof(double) * n);
  put(&o->mu0, sizeof(o->mu0));
  put(&o->mu_max, sizeof(o->mu_max));
  put(&o->rho, sizeof(o->rho));
  put(&o->eps, sizeof(o->eps));
  put(&o->maxiter, sizeof(o->maxiter));
  put(&o->device, sizeof(o->device));
  put(&o->flags, sizeof(o->flags));
  put(&o->poll_every, sizeof(o->poll_every));
  return k;
}
}  // namespace

int pasd_b200_recover(const double* t, const pasd_options* opt, pasd_outputs* out, pasd_observer_fn observer,
                      void* user, char* errbuf, size_t errlen) {
  static const bool trace = std::getenv("PASD_B200_TRACE") != nullptr;
  const bool use_cache = opt && (opt->flags & PASD_FLAG_REUSE_SOLVER);
  pasd_solver* s = nullptr;
  std::vector<char> key;
  const int rc = guarded_call(errbuf, errlen, [&] {
    if (!t || !out || !opt) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    if (use_cache) {
      key = options_key(opt);
      pasd_solver* stale = nullptr;
      {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        if (g_cache && key == g_cache_key) {
          std::swap(s, g_cache);  // take it (concurrent calls build their own)
        } else if (g_cache) {
          stale = g_cache;        // a miss: free the old solver before allocating a new one
          g_cache = nullptr;
          g_cache_key.clear();
        }
      }
      pasd_b200_solver_destroy(stale);
    }
    bool uploaded = false;
    if (s) {
      validate_options(opt);
      CK(cudaSetDevice(s->device));
      begin_upload(s, t);         // H2D of T ...
      reset_state(s, false);      // ... overlaps the E / Y resets
      uploaded = true;
    } else {
      s = create_solver(opt, nullptr);
    }
    const auto t1 = now();
    load_tensor(s, t, 0, uploaded);
    const auto t2 = now();
    run_solver(s, s->maxiter, observer, user);
    const auto t3 = now();
    finalize_solver(s, out);
    const auto t4 = now();
    if (trace)
      std::fprintf(stderr, "pasd_b200_recover: setup %.2f load %.2f run %.2f finalize %.2f ms\n", ms(t0, t1),
                   ms(t1, t2), ms(t2, t3), ms(t3, t4));
  });
  if (rc == PASD_OK && s && use_cache) {
    pasd_solver* old = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      old = g_cache;
      g_cache = s;
      g_cache_key = std::move(key);
    }
    pasd_b200_solver_destroy(old);
  } else {
    pasd_b200_solver_destroy(s);
  }
  return rc;
}

void pasd_b200_release_cache(void) {
  pasd_solver* old = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    old = g_cache;
    g_cache = nullptr;
    g_cache_key.clear();
  }
  pasd_b200_solver_destroy(old);
}

}  // extern "C"

// ---------------------------------------------------------------- linops ABI
namespace {

struct TmpDev {
  std::vector<void*> ptrs;
  ~TmpDev() {
    for (void* p : ptrs) dfree(p);
  }
  template <class T>
  T* alloc(size_t n) {
    T* p = dalloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
};

__global__ void k_set_ctl(Ctl* ctl, double mu, double vnorm2) {
  ctl->mu = mu;
  ctl->mu_used_last = mu;
  ctl->done = 0;
  ctl->ecur = 0;
  ctl->order = 1;
  ctl->vnorm2[0] = vnorm2;
}

// m_is_device: m is a device pointer on `device` (the spec helpers form U^T G there).
void device_svt(const double* m_h, int64_t rows, int64_t cols, double tau, double* out_h, int32_t* kept, int device,
                bool m_is_device = false, double* sig_out = nullptr) {
  if (tau < 0.0 || !std::isfinite(tau)) fail(PASD_ERR_ARGUMENT, "svt: threshold must be a nonnegative finite number");
  if (rows < 1 || cols < 1) fail(PASD_ERR_ARGUMENT, "thin_svd: matrix must be nonempty");
  if (m_is_device) {
    CK(cudaSetDevice(device));
    TmpDev f;
    int* flag = f.alloc<int>(1);
    CK(cudaMemset(flag, 0, sizeof(int)));
    k_nonfinite<<<256, 256>>>(m_h, rows * cols, flag);
    int h = 0;
    CK(cudaMemcpy(&h, flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (h) fail(PASD_ERR_ARGUMENT, "thin_svd: input contains non-finite entries");
  } else {
    for (int64_t i = 0; i < rows * cols; ++i)
      if (!std::isfinite(m_h[i])) fail(PASD_ERR_ARGUMENT, "thin_svd: input contains non-finite entries");
  }
  if (tau == 0.0) {  // linops.cpp:80-81
    if (m_is_device)
      CK(cudaMemcpy(out_h, m_h, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost));
    else
      std::memcpy(out_h, m_h, sizeof(double) * rows * cols);
    if (kept) *kept = (int32_t)std::min(rows, cols);
    return;
  }
  if (rows > PASD_MAX_RANK)
    fail(PASD_ERR_ARGUMENT, "pasd_b200: svt supports at most " + std::to_string(PASD_MAX_RANK) + " rows");
  CK(cudaSetDevice(device));
  TmpDev t;
  ModeDev m{};
  m.inner = 1;
  m.I = rows;
  m.Ifull = rows;
  m.ioff = 0;
  m.outer = cols;
  m.J = cols;
  m.R = (int)rows;
  m.lambda = tau;
  const int R = m.R;
  m.A = t.alloc<double>(rows * cols);
  m.U = t.alloc<double>(R * R);
  m.UM = t.alloc<double>(R * R);
  m.M = t.alloc<double>(R * R);
  m.Gram = t.alloc<double>(R * R);
  m.P = t.alloc<double>(R * R);
  m.Qp = t.alloc<double>(R * R);
  m.sig = t.alloc<double>(R);
  m.nkc_g = (int)std::max<int64_t>(1, std::min<int64_t>((m.J + GR_KC - 1) / GR_KC, 296));
  m.refine_ok = 1;
  m.Gpart = t.alloc<double>((size_t)m.nkc_g * R * R);
  std::vector<double> eye(R * R, 0.0);
  for (int i = 0; i < R; ++i) eye[i + R * i] = 1.0;
  CK(cudaMemcpy(m.U, eye.data(), sizeof(double) * R * R, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(m.P, eye.data(), sizeof(double) * R * R, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(m.A, m_h, sizeof(double) * rows * cols, m_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  ModePack pack{};
  pack.order = 1;
  pack.m[0] = m;
  ModePack* d_pack = t.alloc<ModePack>(1);
  CK(cudaMemcpy(d_pack, &pack, sizeof(pack), cudaMemcpyHostToDevice));
  Ctl* ctl = t.alloc<Ctl>(1);
  k_set_ctl<<<1, 1>>>(ctl, 1.0, 0.0);
  k_gram<<<m.nkc_g, kThreads>>>(m, ctl);
  k_gram_reduce<<<8, 256>>>(m, m.Gram, ctl);
  const size_t smem = small_ws_bytes(R);
  ensure_small_smem_attr();
  k_svt<<<kSmallCluster, kSmallThreads, smem>>>(d_pack, ctl);
  if (out_h) {
    double* V = t.alloc<double>(rows * cols);
    k_materialize_v<<<256, 256>>>(m, V);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out_h, V, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost));
  }
  CK(cudaGetLastError());
  if (sig_out) CK(cudaMemcpy(sig_out, m.sig, sizeof(double) * R, cudaMemcpyDeviceToHost));  // descending
  Ctl hc;
  CK(cudaMemcpy(&hc, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  if (kept) *kept = hc.keep[0];
}

// g_is_device / v_is_device: g, v are device pointers.  xleft_dev (optional,
// device I x R): receives the left singular vectors of g v^T (first *rank
// columns; k_polar's rotated, normalised X) -- the nuclear-norm helper's basis.
void device_procrustes(const double* g_h, int64_t I, int64_t P, const double* v_h, int64_t R64, const double* u_prev,
                       double* u_out, int32_t* degenerate, int32_t* rank, int device, bool g_is_device = false,
                       bool v_is_device = false, double* xleft_dev = nullptr) {
  if (R64 > I) fail(PASD_ERR_ARGUMENT, "procrustes: v has more rows than g (R must not exceed I)");
  if (I < 1 || P < 1 || R64 < 1) fail(PASD_ERR_ARGUMENT, "thin_svd: matrix must be nonempty");
  if (R64 > PASD_MAX_RANK)
    fail(PASD_ERR_ARGUMENT, "pasd_b200: procrustes supports at most " + std::to_string(PASD_MAX_RANK) + " rows of v");
  CK(cudaSetDevice(device));
  const int R = (int)R64;
  TmpDev t;
  ModeDev m{};
  m.inner = 1;
  m.I = I;
  m.Ifull = I;
  m.ioff = 0;
  m.outer = P;
  m.J = P;
  m.R = R;
  const int64_t IR = I * R;
  double* G = t.alloc<double>(I * P);
  double* Z0 = t.alloc<double>(I * P);
  CK(cudaMemset(Z0, 0, sizeof(double) * I * P));
  CK(cudaMemcpy(G, g_h, sizeof(double) * I * P, g_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  m.A = t.alloc<double>(R * P);
  CK(cudaMemcpy(m.A, v_h, sizeof(double) * R * P, v_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  m.U = t.alloc<double>(IR);
  std::vector<double> up(IR, 0.0);
  if (u_prev)
    std::memcpy(up.data(), u_prev, sizeof(double) * IR);
  else
    for (int i = 0; i < R; ++i) up[i + I * i] = 1.0;
  CK(cudaMemcpy(m.U, up.data(), sizeof(double) * IR, cudaMemcpyHostToDevice));
  m.M = t.alloc<double>(R * R);
  std::vector<double> eye(R * R, 0.0);
  for (int i = 0; i < R; ++i) eye[i + R * i] = 1.0;
  CK(cudaMemcpy(m.M, eye.data(), sizeof(double) * R * R, cudaMemcpyHostToDevice));
  m.Qp = t.alloc<double>(R * R);
  CK(cudaMemcpy(m.Qp, eye.data(), sizeof(double) * R * R, cudaMemcpyHostToDevice));
  m.nib_w = (int)((I + CW_IT - 1) / CW_IT);
  m.nkc_w = (int)std::max<int64_t>(1, std::min<int64_t>((P + CW_KC - 1) / CW_KC, std::max(1, 592 / m.nib_w)));
  m.Wpart = t.alloc<double>((size_t)m.nkc_w * IR);
  m.gpart = t.alloc<double>((size_t)m.nkc_w * m.nib_w);
  m.scratch = t.alloc<double>(3 * IR);
  m.Wt = t.alloc<double>(IR);
  Ctl* ctl = t.alloc<Ctl>(1);
  double* vn = t.alloc<double>(1);
  k_sumsq<<<1, 1024>>>(m.A, R * P, vn);
  double vnorm2 = 0.0;
  CK(cudaMemcpy(&vnorm2, vn, sizeof(double), cudaMemcpyDeviceToHost));
  k_set_ctl<<<1, 1>>>(ctl, 1.0, vnorm2);
  const dim3 grid(m.nkc_w, m.nib_w);
  switch (rpt_for(R)) {
    case 2: k_contract_W<2><<<grid, kThreads>>>(m, G, Z0, Z0, Z0, ctl); break;
    case 4: k_contract_W<4><<<grid, kThreads>>>(m, G, Z0, Z0, Z0, ctl); break;
    case 8: k_contract_W<8><<<grid, kThreads>>>(m, G, Z0, Z0, Z0, ctl); break;
    default: k_contract_W<16><<<grid, kThreads>>>(m, G, Z0, Z0, Z0, ctl); break;
  }
  ModePack pack{};
  pack.order = 1;
  pack.m[0] = m;
  ModePack* d_pack = t.alloc<ModePack>(1);
  CK(cudaMemcpy(d_pack, &pack, sizeof(pack), cudaMemcpyHostToDevice));
  k_wreduce_generic<<<dim3(64, 1), 256>>>(d_pack, ctl);
  const size_t smem = small_ws_bytes(R);
  ensure_small_smem_attr();
  k_polar<<<kSmallCluster, kSmallThreads, smem>>>(d_pack, ctl);
  CK(cudaGetLastError());
  Ctl hc;
  CK(cudaMemcpy(&hc, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  if (degenerate) *degenerate = hc.degenerate[0];
  if (rank) *rank = hc.polar_rank[0];
  if (!hc.degenerate[0] && u_out) CK(cudaMemcpy(u_out, m.U, sizeof(double) * IR, cudaMemcpyDeviceToHost));
  if (!hc.degenerate[0] && xleft_dev)
    CK(cudaMemcpy(xleft_dev, m.scratch + IR, sizeof(double) * IR, cudaMemcpyDeviceToDevice));
}

}  // namespace

extern "C" {

int pasd_b200_svt(const double* m, int64_t rows, int64_t cols, double tau, double* out, int32_t* kept, int32_t device,
                  char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!m || !out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    device_svt(m, rows, cols, tau, out, kept, device);
  });
}

int pasd_b200_procrustes(const double* g, int64_t i_rows, int64_t p_cols, const double* v, int64_t r_rows,
                         const double* u_prev, double* u_out, int32_t* degenerate, int32_t* rank, int32_t device,
                         char* errbuf, size_t errlen) {
  return guarded_call(errbuf, errlen, [&] {
    if (!g || !v || !u_out) fail(PASD_ERR_ARGUMENT, "pasd_b200: null argument");
    device_procrustes(g, i_rows, p_cols, v, r_rows, u_prev, u_out, degenerate, rank, device);
  });
}

}  // extern "C"

#include "pasd_spec.cuh"
#include "pasd_synth.cuh"
#include "pasd_snn.cuh"
