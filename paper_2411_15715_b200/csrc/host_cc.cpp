// host_cc.cpp -- CC block on host threads (see host_cc.h).
#include "host_cc.h"

#include <immintrin.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <pthread.h>
#include <sched.h>
#include <stdlib.h>

namespace sp {

// Software prefetch distance (bytes ahead on each weight stream; 0 = off).
// Measured on the box (scripts/gpu_cc_pf.sh, 16 threads, T = 1): 130-149 GB/s
// without, 171-199 GB/s at 4-8 KB.
// Consecutive hidden units' rows are contiguous inside a chunk, so "ahead" runs
// into the next row: the L2 streamer stops at every 4 KB page, this does not.
static int env_or(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
static const int g_cc_pf = env_or("SP_CC_PREFETCH", 8192);
static const int g_amx = env_or("SP_AMX", 1);
static const int g_amx_min_t = env_or("SP_AMX_MIN_T", 4);

bool cc_uses_amx(const CCProblem& p) { return p.wdtype == 1 && g_amx && p.T >= g_amx_min_t && host_has_amx(); }

// ---------------------------------------------------------------------------
// thread pool: persistent workers, the caller participates as tid 0

ThreadPool::ThreadPool(int n_threads) : n_(std::max(1, n_threads)) {
  for (int t = 1; t < n_; ++t) threads_.emplace_back([this, t] { worker(t); });
  // SP_PIN_THREADS=1: worker t on the t-th CPU of the process affinity mask
  if (env_or("SP_PIN_THREADS", 0)) {
    cpu_set_t allowed;
    CPU_ZERO(&allowed);
    if (sched_getaffinity(0, sizeof(allowed), &allowed) == 0) {
      std::vector<int> cpus;
      for (int c = 0; c < CPU_SETSIZE; ++c)
        if (CPU_ISSET(c, &allowed)) cpus.push_back(c);
      for (int t = 1; t < n_ && !cpus.empty(); ++t) {
        cpu_set_t one;
        CPU_ZERO(&one);
        CPU_SET(cpus[size_t(t) % cpus.size()], &one);
        pthread_setaffinity_np(threads_[size_t(t - 1)].native_handle(), sizeof(one), &one);
      }
    }
  }
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_start_.notify_all();
  for (auto& th : threads_) th.join();
}

void ThreadPool::worker(int tid) {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(int, int)>* job;
    int n;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_start_.wait(lk, [&] { return stop_ || generation_ != seen; });
      if (stop_) return;
      seen = generation_;
      job = job_;
      n = job_n_;
    }
    if (tid < n) (*job)(tid, n);
    {
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) cv_done_.notify_one();
    }
  }
}

void ThreadPool::run(int want, const std::function<void(int, int)>& fn) {
  const int n = std::max(1, std::min(want, n_));
  if (n == 1 || n_ == 1) {
    fn(0, 1);
    return;
  }
  {
    std::lock_guard<std::mutex> g(mu_);
    job_ = &fn;
    job_n_ = n;
    pending_ = n_ - 1;
    ++generation_;
  }
  cv_start_.notify_all();
  fn(0, n);
  std::unique_lock<std::mutex> lk(mu_);
  cv_done_.wait(lk, [&] { return pending_ == 0; });
}

// ---------------------------------------------------------------------------
// dot tiles: out[r * NT + t] = <rows[r][0:K16), x[t * ldx + 0:K16)>

bool host_has_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                         __builtin_cpu_supports("fma");
  return ok;
}

template <int WD>
__attribute__((target("avx512f,avx512bw,fma"))) static inline __m512 load16(const void* base,
                                                                             int64_t k) {
  if constexpr (WD == 1) {
    const __m256i h = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(
        static_cast<const uint16_t*>(base) + k));
    return _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(h), 16));
  } else {
    return _mm512_loadu_ps(static_cast<const float*>(base) + k);
  }
}

template <int WD, int NR, int NT>
__attribute__((target("avx512f,avx512bw,fma"))) static void dot_tile_avx512(
    const void* const* rows, int64_t k16, const float* x, int64_t ldx, float* out) {
  __m512 acc[NR][NT];
  for (int r = 0; r < NR; ++r)
    for (int t = 0; t < NT; ++t) acc[r][t] = _mm512_setzero_ps();
  constexpr int64_t kEsz = WD == 1 ? 2 : 4;
  for (int64_t k = 0; k < k16; k += 16) {
    if (g_cc_pf && ((k * kEsz) & 63) == 0)
      for (int r = 0; r < NR; ++r)
        _mm_prefetch(static_cast<const char*>(rows[r]) + k * kEsz + g_cc_pf, _MM_HINT_T0);
    __m512 w[NR];
    for (int r = 0; r < NR; ++r) w[r] = load16<WD>(rows[r], k);
    for (int t = 0; t < NT; ++t) {
      const __m512 xv = _mm512_loadu_ps(x + t * ldx + k);
      for (int r = 0; r < NR; ++r) acc[r][t] = _mm512_fmadd_ps(w[r], xv, acc[r][t]);
    }
  }
  for (int r = 0; r < NR; ++r)
    for (int t = 0; t < NT; ++t) out[r * NT + t] = _mm512_reduce_add_ps(acc[r][t]);
}

static inline float to_f(const void* base, int64_t k, int wd) {
  if (wd == 1) {
    uint32_t u = uint32_t(static_cast<const uint16_t*>(base)[k]) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
  }
  return static_cast<const float*>(base)[k];
}

template <int NR>
static void dot_tile_scalar(const void* const* rows, int64_t k16, const float* x, int64_t ldx,
                            int nt, int wd, float* out) {
  for (int r = 0; r < NR; ++r)
    for (int t = 0; t < nt; ++t) {
      float s = 0.f;
      for (int64_t k = 0; k < k16; ++k) s += to_f(rows[r], k, wd) * x[t * ldx + k];
      out[r * nt + t] = s;
    }
}

// rows: NR row pointers; tokens t in [0, T) processed 4 at a time.
// out[r * T + t]
template <int NR>
static void dot_rows(const void* const* rows, int64_t k16, const float* x, int64_t ldx, int64_t T,
                     int wd, float* out) {
  float tile[NR * 4];
  for (int64_t t0 = 0; t0 < T; t0 += 4) {
    const int nt = int(std::min<int64_t>(4, T - t0));
    const float* xt = x + t0 * ldx;
    if (host_has_avx512()) {
#define SP_TILE(WDV, NTV) dot_tile_avx512<WDV, NR, NTV>(rows, k16, xt, ldx, tile)
      if (wd == 1) {
        switch (nt) {
          case 4: SP_TILE(1, 4); break;
          case 3: SP_TILE(1, 3); break;
          case 2: SP_TILE(1, 2); break;
          default: SP_TILE(1, 1); break;
        }
      } else {
        switch (nt) {
          case 4: SP_TILE(0, 4); break;
          case 3: SP_TILE(0, 3); break;
          case 2: SP_TILE(0, 2); break;
          default: SP_TILE(0, 1); break;
        }
      }
#undef SP_TILE
    } else {
      dot_tile_scalar<NR>(rows, k16, xt, ldx, nt, wd, tile);
    }
    for (int r = 0; r < NR; ++r)
      for (int t = 0; t < nt; ++t) out[r * T + t0 + t] = tile[r * nt + t];
  }
}

static inline float act_host(int act, float z) {
  if (act == 1) return z / (1.0f + expf(-z));
  if (act == 2) return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));
  return z;
}

static inline int64_t round16(int64_t v) { return (v + 15) / 16 * 16; }

// y[t, 0:n16) += sum_r a[r][t] * W2[r][0:n16) for NR rows at once (ybuf is [T, ldy])
template <int WD, int NR>
__attribute__((target("avx512f,avx512bw,fma"))) static void axpy_rows_avx512(
    const void* const* rows, const float* a /*[NR][T]*/, int64_t T, float* ybuf, int64_t ldy, int64_t n16) {
  constexpr int64_t kEsz = WD == 1 ? 2 : 4;
  for (int64_t n = 0; n < n16; n += 16) {
    if (g_cc_pf && ((n * kEsz) & 63) == 0)
      for (int r = 0; r < NR; ++r)
        _mm_prefetch(static_cast<const char*>(rows[r]) + n * kEsz + NR * g_cc_pf, _MM_HINT_T0);
    __m512 w[NR];
    for (int r = 0; r < NR; ++r) w[r] = load16<WD>(rows[r], n);
    for (int64_t t = 0; t < T; ++t) {
      float* yp = ybuf + t * ldy + n;
      __m512 acc = _mm512_loadu_ps(yp);
      for (int r = 0; r < NR; ++r) acc = _mm512_fmadd_ps(w[r], _mm512_set1_ps(a[r * T + t]), acc);
      _mm512_storeu_ps(yp, acc);
    }
  }
}

static void axpy_rows_scalar(const void* const* rows, int nr, const float* a, int64_t T, float* ybuf,
                             int64_t ldy, int64_t n16, int wd) {
  for (int r = 0; r < nr; ++r)
    for (int64_t t = 0; t < T; ++t) {
      const float at = a[r * T + t];
      for (int64_t n = 0; n < n16; ++n) ybuf[t * ldy + n] += at * to_f(rows[r], n, wd);
    }
}

static void axpy_rows(const void* const* rows, int nr, const float* a, int64_t T, float* ybuf,
                      int64_t ldy, int64_t n16, int wd) {
  if (!host_has_avx512()) return axpy_rows_scalar(rows, nr, a, T, ybuf, ldy, n16, wd);
  while (nr > 0) {
    const int take = nr >= 4 ? 4 : nr >= 2 ? 2 : 1;
    if (wd == 1) {
      if (take == 4) axpy_rows_avx512<1, 4>(rows, a, T, ybuf, ldy, n16);
      else if (take == 2) axpy_rows_avx512<1, 2>(rows, a, T, ybuf, ldy, n16);
      else axpy_rows_avx512<1, 1>(rows, a, T, ybuf, ldy, n16);
    } else {
      if (take == 4) axpy_rows_avx512<0, 4>(rows, a, T, ybuf, ldy, n16);
      else if (take == 2) axpy_rows_avx512<0, 2>(rows, a, T, ybuf, ldy, n16);
      else axpy_rows_avx512<0, 1>(rows, a, T, ybuf, ldy, n16);
    }
    rows += take;
    a += take * T;
    nr -= take;
  }
}

// ---------------------------------------------------------------------------

namespace {

// One problem's share of a (batched) CC pass: its row blocks and partial slices.
struct CCPlan {
  const CCProblem* p;
  int64_t k_up, n16, slice, nb;
  int64_t blk0;   // first global block index
  size_t ybuf0;   // offset of its slices in the shared partial buffer
  std::vector<int> chunk_of;
};

CCPlan plan_cc(const CCProblem& p, int n_thr) {
  CCPlan c{&p, round16(p.M), round16(p.N), 0, 0, 0, 0, {}};
  c.slice = p.T * c.n16;
  // Hidden rows are processed in blocks claimed dynamically (an atomic
  // cursor), so a preempted or slow thread does not hold up the block: with
  // 16 threads on a shared 16-vCPU host the static split's tail was the CC
  // block's largest jitter.  Each row block accumulates into its own partial
  // slice and the slices are summed in block order -- the result does not
  // depend on which thread ran which block (deterministic).
  const int64_t budget = (int64_t(8) << 20) / (c.slice * 4);  // partial slices within 8 MB
  c.nb = std::max<int64_t>(1, std::min<int64_t>(p.b1, std::max<int64_t>(n_thr, std::min<int64_t>(budget, 8 * n_thr))));
  c.chunk_of.resize(size_t(p.b1));
  for (int k = 0; k < p.n_chunks; ++k)
    for (int64_t r = 0; r < p.chunks[k].rc; ++r) c.chunk_of[size_t(p.chunks[k].r0 + r)] = k;
  return c;
}

// rows [h0, h1) of one problem into its partial slice ybuf
void cc_rows(const CCPlan& c, int64_t h0, int64_t h1, float* ybuf, float* s, float* a) {
  const CCProblem& p = *c.p;
  const int64_t T = p.T;
  const int wd = p.wdtype;
  const size_t esz = wd == 1 ? 2 : 4;
  const void* w2rows[4];
  std::fill(ybuf, ybuf + c.slice, 0.f);
  int pend = 0;
  for (int64_t h = h0; h < h1; ++h) {
    const HostChunk& ch = p.chunks[c.chunk_of[size_t(h)]];
    const int64_t off1 = (h - ch.r0) * p.ldm * int64_t(esz);
    const void* rows[2] = {static_cast<const char*>(ch.w1t) + off1,
                           p.gated ? static_cast<const char*>(ch.w3t) + off1 : nullptr};
    if (p.gated) {
      dot_rows<2>(rows, c.k_up, p.x, p.ldx, T, wd, s);
      for (int64_t t = 0; t < T; ++t) a[pend * T + t] = act_host(p.act, s[t]) * s[T + t];
    } else {
      dot_rows<1>(rows, c.k_up, p.x, p.ldx, T, wd, s);
      for (int64_t t = 0; t < T; ++t) a[pend * T + t] = act_host(p.act, s[t]);
    }
    w2rows[pend++] = static_cast<const char*>(ch.w2) + (h - ch.r0) * p.ldn * int64_t(esz);
    if (pend == 4 || h + 1 == h1) {
      axpy_rows(w2rows, pend, a, T, ybuf, c.n16, c.n16, wd);
      pend = 0;
    }
  }
}

}  // namespace

void cc_forward_batch(const CCProblem* ps, int n, ThreadPool& pool, int threads) {
  std::vector<CCPlan> plans;
  int64_t t_max = 1;
  for (int i = 0; i < n; ++i) {
    const CCProblem& p = ps[i];
    if (p.b1 <= 0 || p.T <= 0) {
      for (int64_t k = 0; k < p.T * p.N; ++k) p.y[k] = 0.f;
      continue;
    }
    if (cc_uses_amx(p)) {
      cc_forward_amx(p, pool, threads);
      continue;
    }
    plans.reserve(size_t(n));
    const int n_thr = int(std::max<int64_t>(1, std::min<int64_t>(std::min(threads, pool.size()), p.b1)));
    plans.push_back(plan_cc(p, n_thr));
    t_max = std::max(t_max, p.T);
  }
  if (plans.empty()) return;
  int64_t blocks = 0, most_rows = 1;
  size_t floats = 0;
  for (CCPlan& c : plans) {
    c.blk0 = blocks;
    c.ybuf0 = floats;
    blocks += c.nb;
    floats += size_t(c.nb * c.slice);
    most_rows = std::max(most_rows, c.p->b1);
  }
  const int n_thr = int(std::max<int64_t>(1, std::min<int64_t>(std::min(threads, pool.size()), most_rows)));
  // persistent across calls (no page faults on fresh mmap'd memory every call)
  // (a thread_local is per thread: the workers below must use this pointer)
  static thread_local std::vector<float> tl_ybufs;
  tl_ybufs.resize(std::max(tl_ybufs.size(), floats));
  float* const ybufs = tl_ybufs.data();
  std::atomic<int64_t> cursor{0};

  auto rows_pass = [&](int, int) {
    std::vector<float> s(size_t(2 * t_max)), a(size_t(4 * t_max));
    size_t pi = 0;
    for (;;) {
      const int64_t g = cursor.fetch_add(1, std::memory_order_relaxed);
      if (g >= blocks) break;
      while (g >= plans[pi].blk0 + plans[pi].nb) ++pi;  // blocks are claimed in increasing order
      const CCPlan& c = plans[pi];
      const int64_t blk = g - c.blk0, b1 = c.p->b1;
      cc_rows(c, b1 * blk / c.nb, b1 * (blk + 1) / c.nb, ybufs + c.ybuf0 + size_t(blk) * c.slice, s.data(), a.data());
    }
  };
  pool.run(n_thr, rows_pass);

  auto reduce = [&](int tid, int nt) {
    std::vector<float> acc;
    for (const CCPlan& c : plans) {
      const CCProblem& p = *c.p;
      const int64_t c0 = (c.n16 / 16) * tid / nt * 16;
      const int64_t c1 = std::min<int64_t>((c.n16 / 16) * (tid + 1) / nt * 16, p.N);
      if (c1 <= c0) continue;
      acc.resize(size_t(c1 - c0));
      for (int64_t t = 0; t < p.T; ++t) {
        std::fill(acc.begin(), acc.end(), 0.f);
        for (int64_t i = 0; i < c.nb; ++i) {  // block order: deterministic
          const float* src = ybufs + c.ybuf0 + size_t(i) * c.slice + t * c.n16;
          for (int64_t col = c0; col < c1; ++col) acc[size_t(col - c0)] += src[col];
        }
        std::copy(acc.begin(), acc.end(), p.y + t * p.N + c0);
      }
    }
  };
  pool.run(threads, reduce);
}

void cc_forward(const CCProblem& p, ThreadPool& pool, int threads) { cc_forward_batch(&p, 1, pool, threads); }

}  // namespace sp
