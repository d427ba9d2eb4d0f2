// host_cc.h -- the CC block on host cores (Stream-A of PAPER.md:161).
//
// The reference computes every block with numpy fp64 on one thread
// (slicing_kernel.py:119-123).  Here the CC block (hidden columns [0, b1)) is
// computed natively from the same pinned, chunk-interleaved layout the GPU
// streams from, on a persistent pool of host threads, in fp32 with AVX-512:
//   a[t, h]  = act(<W1t[h], x[t]>) [* <W3t[h], x[t]>]      rows split over threads
//   y[t, n]  = sum_chunks <W2t_chunk[n, :rc], a[t, r0:r0+rc]>  outputs split over threads
#pragma once

#include <stdint.h>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace sp {

class ThreadPool {
 public:
  explicit ThreadPool(int n_threads);
  ~ThreadPool();
  int size() const { return n_; }
  // Run fn(tid, n) on n = min(want, size()) threads; the caller is tid 0.
  void run(int want, const std::function<void(int, int)>& fn);

 private:
  void worker(int tid);
  int n_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_start_, cv_done_;
  const std::function<void(int, int)>* job_ = nullptr;
  int job_n_ = 0;
  uint64_t generation_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

struct HostChunk {
  const void* w1t;  // [rc, ldm]
  const void* w3t;  // [rc, ldm] or null
  const void* w2t;  // [N, ldc]
  int64_t r0, rc, ldc;
};

struct CCProblem {
  int wdtype;      // 0 f32, 1 bf16
  int gated, act;
  int64_t M, N, ldm;
  const HostChunk* chunks;
  int n_chunks;    // covering hidden rows [0, b1)
  int64_t b1;
  const float* x;  // [T, ldx] fp32, zero padded to ldx >= roundup(M, 64)
  int64_t ldx;
  int64_t T;
  float* a;        // scratch [T, lda], lda >= roundup(b1, 64), zero padded
  int64_t lda;
  float* y;        // [T, N] output
};

void cc_forward(const CCProblem& p, ThreadPool& pool, int threads);
bool host_has_avx512();

}  // namespace sp
