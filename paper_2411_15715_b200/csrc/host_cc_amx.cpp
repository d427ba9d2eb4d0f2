// host_cc_amx.cpp -- the CC block on Intel AMX tiles (prompt-size token counts).
//
// With tens of tokens per expert (the prompt rows the token assigner keeps on
// the host, token_assigner.py:33-137) the CC block is compute bound on
// AVX-512 FP32 FMA (~0.5 TFLOP/s on 16 cores): it paced the whole prefill
// layer.  AMX TDPBF16PS does a 16x16x32 bf16 tile product per instruction
// with fp32 accumulation, enough to make the block host-DRAM bound again at
// 128 tokens.  Same math as the GPU tensor-core path: x and the hidden
// activation a = act(x W1t^T) [* x W3t^T] are rounded to bf16, all sums fp32.
//
//   up   (per 16 hidden rows h, per 2 token groups g):
//        C[h][t] += W1t[h][k:k+32] . xp[g][k/2..][t]          A = weight rows (natural layout)
//                                                              B = x packed in VNNI pairs once
//   act  a[t][h] = bf16(act(C1) [* C3])
//   down (per 256 output columns, per 2 n-tiles, per token group):
//        Y[t][n] += a[t][h:h+32] . W2p[h/2][n]                 B = W2 rows interleaved in pairs
//                                                              (repacked per block into L2)
// Hidden rows are claimed in 32-row-aligned blocks by an atomic cursor; each
// block accumulates into its own partial slice and the slices are summed in
// block order (deterministic, as the AVX-512 path).
#include <immintrin.h>
#include <math.h>
#include <string.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <vector>
#include <stdio.h>
#include <stdlib.h>
#include <x86intrin.h>

#include "host_cc.h"

namespace sp {

namespace {

constexpr long kArchReqXcompPerm = 0x1023;
constexpr long kXfeatureXtiledata = 18;

struct alignas(64) TileConfig {
  uint8_t palette;
  uint8_t start_row;
  uint8_t reserved[14];
  uint16_t colsb[16];
  uint8_t rows[16];
};

inline uint16_t f2bf(float f) {  // round to nearest even (finite inputs)
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

inline float act_f(int act, float z) {
  if (act == 1) return z / (1.0f + expf(-z));
  if (act == 2) return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));
  return z;
}

struct AmxShared {
  const CCProblem& p;
  int64_t T16, G16, K32, KP, n16, ldm_b, ldn, n32, nb, slice, hb_max;
  const uint16_t* xp;
  const int* chunk_of;
  float* ybufs;
  std::atomic<int64_t>* cursor;
};

constexpr int64_t NR = 1024;     // output columns per W2 repack (2 KB contiguous per row)
constexpr int64_t kUpPf = 1024;  // up-GEMM weight prefetch distance (bytes per row)

__attribute__((target("amx-tile,amx-bf16,avx512f,avx512bw"))) void amx_worker(const AmxShared& S) {
  const CCProblem& p = S.p;
  const int64_t T = p.T, T16 = S.T16, G16 = S.G16, K32 = S.K32, KP = S.KP, n16 = S.n16, ldm_b = S.ldm_b,
                ldn = S.ldn, n32 = S.n32, nb = S.nb, slice = S.slice, hb_max = S.hb_max;
  const uint16_t* xpd = S.xp;
  const int* chunk_of = S.chunk_of;
  // scratch lives across calls: fresh large allocations are mmap'd and every
  // first touch is a page fault (expensive under a hypervisor)
  static thread_local std::vector<uint16_t> a_bf, w2p, pad1, pad3;
  TileConfig cfg{};
  cfg.palette = 1;
  for (int i = 0; i < 8; ++i) {
    cfg.colsb[i] = 64;
    cfg.rows[i] = 16;
  }
  _tile_loadconfig(&cfg);
  alignas(64) float z1[2][256], z3[2][256];
  a_bf.resize(std::max(a_bf.size(), size_t(T16 * hb_max)));
  w2p.resize(std::max(w2p.size(), size_t(hb_max / 2 * NR * 2)));
  pad1.resize(std::max(pad1.size(), size_t(16 * p.ldm)));
  pad3.resize(std::max(pad3.size(), size_t(16 * p.ldm)));
  // SP_AMX_PROF=1: per-thread cycle split printed to stderr (tuning aid)
  static const bool prof = getenv("SP_AMX_PROF") != nullptr;
  unsigned long long c_up = 0, c_act = 0, c_rep = 0, c_dn = 0, tq = 0;
  for (;;) {
    const int64_t blk = S.cursor->fetch_add(1, std::memory_order_relaxed);
    if (blk >= nb) break;
    const int64_t s0 = n32 * blk / nb, s1 = n32 * (blk + 1) / nb;
    const int64_t r0 = 32 * s0, r1 = std::min<int64_t>(32 * s1, p.b1);
    const int64_t hbp = 32 * (s1 - s0);  // padded rows of this block
    float* ybuf = S.ybufs + size_t(blk) * slice;
    std::fill(ybuf, ybuf + slice, 0.f);

    // ---- up: a[t][h - r0] for the block's rows ----
    for (int64_t sb = 0; sb < hbp / 16; ++sb) {
      const int64_t h = r0 + 16 * sb;
      const int64_t valid = std::min<int64_t>(16, r1 - h);
      if (valid <= 0) {
        for (int64_t t = 0; t < T16; ++t)
          memset(&a_bf[size_t(t * hbp + 16 * sb)], 0, 32);
        continue;
      }
      const HostChunk& c = p.chunks[chunk_of[size_t(h)]];
      const char* w1 = static_cast<const char*>(c.w1t) + (h - c.r0) * ldm_b;
      const char* w3 = p.gated ? static_cast<const char*>(c.w3t) + (h - c.r0) * ldm_b : nullptr;
      if (valid < 16) {  // last rows of the CC block: never read past them
        std::fill(pad1.begin(), pad1.begin() + 16 * p.ldm, 0);
        memcpy(pad1.data(), w1, size_t(valid * ldm_b));
        w1 = reinterpret_cast<const char*>(pad1.data());
        if (p.gated) {
          std::fill(pad3.begin(), pad3.begin() + 16 * p.ldm, 0);
          memcpy(pad3.data(), w3, size_t(valid * ldm_b));
          w3 = reinterpret_cast<const char*>(pad3.data());
        }
      }
      for (int64_t g0 = 0; g0 < G16; g0 += 2) {
        const bool two = g0 + 1 < G16;
        _tile_zero(4);
        _tile_zero(5);
        _tile_zero(6);
        _tile_zero(7);
        const uint16_t* xg0 = xpd + size_t(g0 * KP * 32);
        const uint16_t* xg1 = xpd + size_t((g0 + 1) * KP * 32);
        if (prof) tq = __rdtsc();
        for (int64_t k = 0; k < K32; k += 32) {
          // Tile registers are not renamed: a tile load waits for the last
          // product reading that tile, so each k step would eat a full DRAM
          // latency.  Prefetch the 16 (32) weight rows kUpPf bytes ahead.
          if (g0 == 0)
            for (int i = 0; i < 16; ++i) {
              _mm_prefetch(w1 + i * ldm_b + k * 2 + kUpPf, _MM_HINT_T0);
              if (p.gated) _mm_prefetch(w3 + i * ldm_b + k * 2 + kUpPf, _MM_HINT_T0);
            }
          _tile_loadd(0, w1 + k * 2, ldm_b);
          if (p.gated) _tile_loadd(1, w3 + k * 2, ldm_b);
          _tile_loadd(2, xg0 + (k / 2) * 32, 64);
          _tile_dpbf16ps(4, 0, 2);
          if (p.gated) _tile_dpbf16ps(6, 1, 2);
          if (two) {
            _tile_loadd(3, xg1 + (k / 2) * 32, 64);
            _tile_dpbf16ps(5, 0, 3);
            if (p.gated) _tile_dpbf16ps(7, 1, 3);
          }
        }
        if (prof) {
          c_up += __rdtsc() - tq;
          tq = __rdtsc();
        }
        _tile_stored(4, z1[0], 64);
        _tile_stored(5, z1[1], 64);
        _tile_stored(6, z3[0], 64);
        _tile_stored(7, z3[1], 64);
        for (int q = 0; q < (two ? 2 : 1); ++q)
          for (int i = 0; i < 16; ++i)      // hidden row h + i
            for (int j = 0; j < 16; ++j) {  // token 16 (g0 + q) + j
              const int64_t t = 16 * (g0 + q) + j;
              float a = 0.f;
              if (i < valid && t < T) {
                a = act_f(p.act, z1[q][i * 16 + j]);
                if (p.gated) a *= z3[q][i * 16 + j];
              }
              a_bf[size_t(t * hbp + 16 * sb + i)] = f2bf(a);
            }
        if (prof) c_act += __rdtsc() - tq;
      }
    }

    // ---- down: Y[t][n] += a[t][:] . W2[r0:r1][n] ----
    for (int64_t n0 = 0; n0 < n16; n0 += NR) {
      const int64_t nr = std::min<int64_t>(NR, n16 - n0);
      if (prof) tq = __rdtsc();
      // W2 rows in VNNI pairs: w2p[pr][n][e] = W2[r0 + 2 pr + e][n0 + n], zero past r1
      for (int64_t pr = 0; pr < hbp / 2; ++pr) {
        const int64_t ha = r0 + 2 * pr, hb2 = ha + 1;
        const uint16_t* ra = nullptr;
        const uint16_t* rb = nullptr;
        if (ha < r1) {
          const HostChunk& c = p.chunks[chunk_of[size_t(ha)]];
          ra = static_cast<const uint16_t*>(c.w2) + (ha - c.r0) * ldn + n0;
        }
        if (hb2 < r1) {
          const HostChunk& c = p.chunks[chunk_of[size_t(hb2)]];
          rb = static_cast<const uint16_t*>(c.w2) + (hb2 - c.r0) * ldn + n0;
        }
        uint16_t* dst = w2p.data() + size_t(pr * nr * 2);
        if (pr + 2 < hbp / 2 && ha + 5 < r1) {  // rows two pairs ahead
          const HostChunk& c = p.chunks[chunk_of[size_t(ha + 4)]];
          if (ha + 5 < c.r0 + c.rc) {
            const char* q = reinterpret_cast<const char*>(static_cast<const uint16_t*>(c.w2) + (ha + 4 - c.r0) * ldn + n0);
            for (int64_t off = 0; off < nr * 2; off += 64) {
              _mm_prefetch(q + off, _MM_HINT_T0);
              _mm_prefetch(q + ldn * 2 + off, _MM_HINT_T0);
            }
          }
        }
        for (int64_t n = 0; n < nr; n += 16) {
          const __m512i va = ra ? _mm512_cvtepu16_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(ra + n)))
                                : _mm512_setzero_si512();
          const __m512i vb = rb ? _mm512_slli_epi32(
                                      _mm512_cvtepu16_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(rb + n))), 16)
                                : _mm512_setzero_si512();
          _mm512_storeu_si512(reinterpret_cast<void*>(dst + n * 2), _mm512_or_si512(va, vb));
        }
      }
      // 2 token groups x 2 column tiles per pass: four independent accumulator
      // chains, every A and B tile feeds two products
      if (prof) {
        c_rep += __rdtsc() - tq;
        tq = __rdtsc();
      }
      const int64_t njt = nr / 16;
      for (int64_t jn = 0; jn < njt; jn += 2) {
        const bool j2 = jn + 1 < njt;
        for (int64_t g = 0; g < G16; g += 2) {
          const bool g2 = g + 1 < G16;
          float* y0 = ybuf + (16 * g) * n16 + n0 + 16 * jn;
          float* y1 = y0 + 16 * n16;
          _tile_loadd(0, y0, n16 * 4);
          if (j2) _tile_loadd(1, y0 + 16, n16 * 4);
          if (g2) _tile_loadd(2, y1, n16 * 4);
          if (g2 && j2) _tile_loadd(3, y1 + 16, n16 * 4);
          const uint16_t* a0 = a_bf.data() + (16 * g) * hbp;
          const uint16_t* a1 = a0 + 16 * hbp;
          const uint16_t* b0 = w2p.data() + jn * 32;
          for (int64_t sl = 0; sl < hbp / 32; ++sl) {
            _tile_loadd(4, a0 + 32 * sl, hbp * 2);
            _tile_loadd(6, b0 + (16 * sl) * nr * 2, nr * 4);
            _tile_dpbf16ps(0, 4, 6);
            if (j2) {
              _tile_loadd(7, b0 + (16 * sl) * nr * 2 + 32, nr * 4);
              _tile_dpbf16ps(1, 4, 7);
            }
            if (g2) {
              _tile_loadd(5, a1 + 32 * sl, hbp * 2);
              _tile_dpbf16ps(2, 5, 6);
              if (j2) _tile_dpbf16ps(3, 5, 7);
            }
          }
          _tile_stored(0, y0, n16 * 4);
          if (j2) _tile_stored(1, y0 + 16, n16 * 4);
          if (g2) _tile_stored(2, y1, n16 * 4);
          if (g2 && j2) _tile_stored(3, y1 + 16, n16 * 4);
        }
      }
      if (prof) c_dn += __rdtsc() - tq;
    }
  }
  _tile_release();
  if (prof)
    fprintf(stderr, "amx kcycles: up %llu act %llu repack %llu down %llu\n", c_up >> 10, c_act >> 10, c_rep >> 10,
            c_dn >> 10);
}

}  // namespace

bool host_has_amx() {
  static const bool ok = [] {
    if (!__builtin_cpu_supports("amx-tile") || !__builtin_cpu_supports("amx-bf16") ||
        !__builtin_cpu_supports("avx512f") || !__builtin_cpu_supports("avx512bw"))
      return false;
    // Linux hands out the 8 KB tile state only on request (per process)
    return syscall(SYS_arch_prctl, kArchReqXcompPerm, kXfeatureXtiledata) == 0;
  }();
  return ok;
}

void cc_forward_amx(const CCProblem& p, ThreadPool& pool, int threads) {
  const int64_t T = p.T, M = p.M, N = p.N;
  const int64_t T16 = (T + 15) / 16 * 16, G16 = T16 / 16;
  const int64_t K32 = (M + 31) / 32 * 32;  // W rows are zero padded to ldm >= roundup(M, 64)
  const int64_t KP = K32 / 2;              // k pairs
  const int64_t n16 = (N + 15) / 16 * 16;  // W2 rows zero padded to ldn >= roundup(N, 64)
  const int64_t ldm_b = p.ldm * 2, ldn = p.ldn;
  const int n_thr = int(std::max<int64_t>(1, std::min<int64_t>(std::min(threads, pool.size()), (p.b1 + 31) / 32)));

  // x -> bf16 VNNI pairs: xp[g][kp][j][e] = x[16 g + j][2 kp + e]
  // (thread_locals of the calling thread: workers get raw pointers)
  static thread_local std::vector<uint16_t> tl_xp;
  static thread_local std::vector<float> tl_ybufs;
  tl_xp.resize(std::max(tl_xp.size(), size_t(G16 * KP * 32)));
  uint16_t* const xp = tl_xp.data();
  std::fill(xp, xp + G16 * KP * 32, 0);
  for (int64_t t = 0; t < T; ++t) {
    const float* xr = p.x + t * p.ldx;
    const int64_t g = t / 16, j = t % 16;
    for (int64_t k = 0; k < M; ++k) xp[size_t(((g * KP + k / 2) * 16 + j) * 2 + (k & 1))] = f2bf(xr[k]);
  }

  // hidden row -> chunk
  std::vector<int> chunk_of(size_t(p.b1));
  for (int c = 0; c < p.n_chunks; ++c)
    for (int64_t r = 0; r < p.chunks[c].rc; ++r) chunk_of[size_t(p.chunks[c].r0 + r)] = c;

  const int64_t n32 = (p.b1 + 31) / 32;
  const int64_t slice = T16 * n16;
  const int64_t budget = (int64_t(64) << 20) / (slice * 4);  // partial slices within 64 MB
  int64_t nb = std::min<int64_t>(n32, std::max<int64_t>(n_thr, std::min<int64_t>(budget, 4 * n_thr)));
  nb = std::max<int64_t>(1, nb);
  const int64_t max_slabs = (n32 + nb - 1) / nb;
  const int64_t hb_max = 32 * max_slabs;
  tl_ybufs.resize(std::max(tl_ybufs.size(), size_t(nb * slice)));
  float* const ybufs = tl_ybufs.data();
  std::atomic<int64_t> cursor{0};
  AmxShared S{p, T16, G16, K32, KP, n16, ldm_b, ldn, n32, nb, slice, hb_max, xp, chunk_of.data(), ybufs,
              &cursor};
  pool.run(n_thr, [&](int, int) { amx_worker(S); });

  auto reduce = [&](int tid, int n) {
    const int64_t c0 = (n16 / 16) * tid / n * 16;
    const int64_t c1 = std::min<int64_t>((n16 / 16) * (tid + 1) / n * 16, N);
    if (c1 <= c0) return;
    std::vector<float> acc(size_t(c1 - c0));
    for (int64_t t = 0; t < T; ++t) {
      std::fill(acc.begin(), acc.end(), 0.f);
      for (int64_t i = 0; i < nb; ++i) {  // block order: deterministic
        const float* src = ybufs + size_t(i) * slice + t * n16;
        for (int64_t col = c0; col < c1; ++col) acc[size_t(col - c0)] += src[col];
      }
      std::copy(acc.begin(), acc.end(), p.y + t * N + c0);
    }
  };
  pool.run(threads, reduce);
}

}  // namespace sp
