// pasd_comm.cuh — the collectives of the slab-sharded iteration.
//
// Every exchange of the sharded PASD iteration is an all-reduce of fp64
// partials (A_3, Gram_1/2, Wt_n, ||G_n||^2: SUM; residual maxima + NaN flag:
// MAX; finalisation scalars).  The solver issues them through this interface:
//
//   NcclComm      one process (or thread) per GPU, NCCL over NVLink/NVSwitch;
//                 the calls are stream-ordered and are captured into the
//                 iteration's CUDA graph.
//   LoopbackComm  every rank of a group in one process on ONE device (one host
//                 thread per rank), for running the library's own sharded code
//                 path with nranks > 1 without more GPUs.  Ranks meet at host
//                 barriers: a rank synchronises its stream, posts its send
//                 buffers, and after the barrier reduces all ranks' buffers in
//                 rank order with an ordinary kernel; a second barrier keeps
//                 the send buffers alive until every rank has read them.  No
//                 kernel ever waits on another rank's kernel (they may or may
//                 not run concurrently), so nothing can hang the device.  Not
//                 capturable: a loopback solver launches its iterations eagerly.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace pasd {

enum class RedOp { Sum, Max };

class Comm {
 public:
  virtual ~Comm() = default;
  virtual void group_start() = 0;
  virtual void group_end() = 0;
  virtual void allreduce(const double* send, double* recv, size_t count, RedOp op, cudaStream_t st) = 0;
  virtual bool capturable() const = 0;
  virtual const char* kind() const = 0;
};

constexpr int kLoopbackMaxRanks = 8;

struct LoopbackSrc {
  const double* p[kLoopbackMaxRanks];
};

// recv = fold over ranks 0..n-1 (fixed order: every rank gets the same bytes)
__global__ void k_loopback_reduce(LoopbackSrc src, int n, double* recv, int64_t count, int is_max) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double v = src.p[0][i];
    for (int q = 1; q < n; ++q) {
      const double x = src.p[q][i];
      v = is_max ? (x > v ? x : v) : v + x;
    }
    recv[i] = v;
  }
}

// Shared by the nranks LoopbackComm objects of one group.
struct LoopbackGroup {
  struct Op {
    const double* send;
    double* recv;
    size_t count;
    RedOp op;
    cudaStream_t st;
  };
  explicit LoopbackGroup(int n) : nranks(n), posted(n) {}
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool broken = false;
  std::vector<std::vector<Op>> posted;  // [rank] ops of the current round

  // Reusable barrier; a rank that never arrives (an error on its thread)
  // breaks the group after `timeout_s` instead of hanging the others.
  // Returns false when the group is broken.
  bool barrier(double timeout_s = 300.0) {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const uint64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                [&] { return generation != gen || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

}  // namespace pasd
