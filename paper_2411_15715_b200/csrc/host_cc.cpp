// host_cc.cpp -- CC block on host threads (see host_cc.h).
#include "host_cc.h"

#include <immintrin.h>
#include <math.h>
#include <string.h>

#include <algorithm>

namespace sp {

// ---------------------------------------------------------------------------
// thread pool: persistent workers, the caller participates as tid 0

ThreadPool::ThreadPool(int n_threads) : n_(std::max(1, n_threads)) {
  for (int t = 1; t < n_; ++t) threads_.emplace_back([this, t] { worker(t); });
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
  for (int64_t k = 0; k < k16; k += 16) {
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
  for (int64_t n = 0; n < n16; n += 16) {
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

void cc_forward(const CCProblem& p, ThreadPool& pool, int threads) {
  const int64_t T = p.T;
  if (p.b1 <= 0 || T <= 0) {
    for (int64_t i = 0; i < T * p.N; ++i) p.y[i] = 0.f;
    return;
  }
  const int wd = p.wdtype;
  const size_t esz = wd == 1 ? 2 : 4;
  const int64_t k_up = round16(p.M);
  const int64_t n16 = round16(p.N);  // W2 rows are zero padded to ldn >= roundup(N, 64)
  const int n_thr = int(std::max<int64_t>(1, std::min<int64_t>(std::min(threads, pool.size()), p.b1)));

  // hidden row -> chunk
  std::vector<int> chunk_of(size_t(p.b1));
  for (int c = 0; c < p.n_chunks; ++c)
    for (int64_t r = 0; r < p.chunks[c].rc; ++r) chunk_of[size_t(p.chunks[c].r0 + r)] = c;

  // per-thread partial outputs [n_thr][T][n16]
  std::vector<float> ybufs(size_t(n_thr) * T * n16, 0.f);

  auto rows_pass = [&](int tid, int n) {
    const int64_t h0 = p.b1 * tid / n, h1 = p.b1 * (tid + 1) / n;
    float* ybuf = ybufs.data() + size_t(tid) * T * n16;
    std::vector<float> s(size_t(2 * T)), a(size_t(4 * T));
    const void* w2rows[4];
    int pend = 0;
    for (int64_t h = h0; h < h1; ++h) {
      const HostChunk& c = p.chunks[chunk_of[size_t(h)]];
      const int64_t off1 = (h - c.r0) * p.ldm * int64_t(esz);
      const void* rows[2] = {static_cast<const char*>(c.w1t) + off1,
                             p.gated ? static_cast<const char*>(c.w3t) + off1 : nullptr};
      if (p.gated) {
        dot_rows<2>(rows, k_up, p.x, p.ldx, T, wd, s.data());
        for (int64_t t = 0; t < T; ++t) a[pend * T + t] = act_host(p.act, s[t]) * s[T + t];
      } else {
        dot_rows<1>(rows, k_up, p.x, p.ldx, T, wd, s.data());
        for (int64_t t = 0; t < T; ++t) a[pend * T + t] = act_host(p.act, s[t]);
      }
      w2rows[pend++] = static_cast<const char*>(c.w2) + (h - c.r0) * p.ldn * int64_t(esz);
      if (pend == 4 || h + 1 == h1) {
        axpy_rows(w2rows, pend, a.data(), T, ybuf, n16, n16, wd);
        pend = 0;
      }
    }
  };
  pool.run(n_thr, rows_pass);

  auto reduce = [&](int tid, int n) {
    const int64_t c0 = (n16 / 16) * tid / n * 16, c1 = (n16 / 16) * (tid + 1) / n * 16;
    for (int64_t t = 0; t < T; ++t)
      for (int64_t col = c0; col < c1; ++col) {
        if (col >= p.N) break;
        float v = 0.f;
        for (int i = 0; i < n_thr; ++i) v += ybufs[(size_t(i) * T + t) * n16 + col];
        p.y[t * p.N + col] = v;
      }
  };
  pool.run(threads, reduce);
}

}  // namespace sp
