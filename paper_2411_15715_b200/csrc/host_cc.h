// host_cc.h -- the CC block on host cores (Stream-A of PAPER.md:161).
//
// The reference computes every block with numpy fp64 on one thread
// (slicing_kernel.py:119-123).  Here the CC block (hidden units [0, b1)) is
// computed natively from the same pinned, chunk-interleaved layout the GPU
// streams from, on a persistent pool of host threads, in fp32 with AVX-512.
// Thread i owns a contiguous range of hidden units and streams their rows once:
//   a[t, h]     = act(<W1t[h], x[t]>) [* <W3t[h], x[t]>]
//   y_i[t, :]  += a[t, h] * W2[h, :]
// then y = sum_i y_i in thread order (deterministic), split over columns.
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
  const void* w2;   // [rc, ldn]
  int64_t r0, rc;
};

struct CCProblem {
  int wdtype;      // 0 f32, 1 bf16
  int gated, act;
  int64_t M, N, ldm, ldn;
  const HostChunk* chunks;
  int n_chunks;    // covering hidden rows [0, b1)
  int64_t b1;
  const float* x;  // [T, ldx] fp32, zero padded to ldx >= roundup(M, 64)
  int64_t ldx;
  int64_t T;
  float* y;        // [T, N] output
  // AMX down phase: W2 of the CC rows already in VNNI pairs, one block per
  // 128-column round (amx_prepack_w2), or null (each round repacks it)
  const uint16_t* w2p = nullptr;
};

void cc_forward(const CCProblem& p, ThreadPool& pool, int threads);
// Several problems (the active experts of a decode step) in ONE pass: their row
// blocks share one dynamic queue and one reduce, so the pool joins once per
// step instead of twice per expert.  Each problem's result is bit-identical to
// cc_forward's (same blocks, same block-order sums).  AMX-eligible problems run
// through cc_forward one after another.
void cc_forward_batch(const CCProblem* ps, int n, ThreadPool& pool, int threads);
bool host_has_avx512();
// AMX tile path for bf16 weights and prompt-size token counts (host_cc_amx.cpp);
// cc_forward dispatches to it when T >= SP_AMX_MIN_T (default 4) and the host
// has AMX-BF16 (SP_AMX=0 disables it).
bool host_has_amx();
void cc_forward_amx(const CCProblem& p, ThreadPool& pool, int threads);
// true when cc_forward / cc_forward_batch run this problem on AMX tiles
bool cc_uses_amx(const CCProblem& p);
// elements (bf16) of the prepacked W2 of p's CC rows, and the prepack itself
size_t amx_w2_prepack_elems(const CCProblem& p);
void amx_prepack_w2(const CCProblem& p, uint16_t* out, ThreadPool& pool, int threads);

}  // namespace sp
