// host_cc_amx.cpp -- the CC block on Intel AMX tiles (prompt-size token counts).
//
// With tens to hundreds of tokens per expert (the prompt rows the token
// assigner keeps on the host, token_assigner.py:33-137) the CC block is
// compute bound; AMX TDPBF16PS does a 16x16x32 bf16 tile product per
// instruction with fp32 accumulation.  Same math as the GPU tensor-core path:
// x and the hidden activation a = act(x W1t^T) [* x W3t^T] are rounded to
// bf16, every sum is fp32.  Three phases on the host pool:
//
//   pack  x -> bf16 VNNI pairs xp[g][kp][j][e] = x[16 g + j][2 kp + e]   (all threads)
//   up    per 16-row hidden slab (dynamic cursor), per 2 token groups:
//           C[h][t] += W1t[h][k:k+32] . xp[g][k/2..][t]   A = weight rows as stored
//         a[t][h] = bf16(act(C1) [* C3])  (AVX-512, into one shared [T16][b1p] array)
//   down  rounds of 128 output columns (dynamic cursor), W2 rows repacked in
//         VNNI pairs per round; 4 accumulator tiles (2 token groups x 2 column
//         tiles) run over the WHOLE hidden range before one store:
//           Y[t][n] = sum_h a[t][h] W2[h][n]
// The down phase splits columns, not hidden rows, so there are no partial
// slices to reduce and each output element is summed in one fixed hidden order
// whatever the thread count (deterministic).
//
// SP_AMX_EMULATE (tests only): the tile operations run as plain C++ on
// software tiles, so the index arithmetic is checked on hosts without AMX
// (tests/test_amx_emulated.py builds this file with it).
#include <immintrin.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <x86intrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <vector>

#include "host_cc.h"

namespace sp {

namespace {

constexpr long kArchReqXcompPerm = 0x1023;
constexpr long kXfeatureXtiledata = 18;
constexpr int64_t kRoundCols = 128;  // W2 columns repacked per down-phase round (b1p x 512 B)
constexpr int64_t kUpPf = 1024;      // up-phase weight prefetch distance (bytes ahead per row)

struct alignas(64) TileConfig {
  uint8_t palette;
  uint8_t start_row;
  uint8_t reserved[14];
  uint16_t colsb[16];
  uint8_t rows[16];
};

#ifdef SP_AMX_EMULATE
// ---- software tiles (16 rows x 64 bytes each) ----
struct EmuTile {
  alignas(64) unsigned char d[16 * 64];
};
thread_local EmuTile emu[8];
inline float bf2f(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
inline void emu_zero(int t) { memset(emu[t].d, 0, sizeof(emu[t].d)); }
inline void emu_load(int t, const void* p, int64_t stride) {
  for (int r = 0; r < 16; ++r) memcpy(emu[t].d + r * 64, static_cast<const char*>(p) + r * stride, 64);
}
inline void emu_store(int t, void* p, int64_t stride) {
  for (int r = 0; r < 16; ++r) memcpy(static_cast<char*>(p) + r * stride, emu[t].d + r * 64, 64);
}
inline void emu_dp(int c, int a, int b) {  // C[m][n] += sum_k A[m][2k..] . B[k][2n..]
  float* C = reinterpret_cast<float*>(emu[c].d);
  const uint16_t* A = reinterpret_cast<const uint16_t*>(emu[a].d);
  const uint16_t* B = reinterpret_cast<const uint16_t*>(emu[b].d);
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 16; ++n) {
      float s = C[m * 16 + n];
      for (int k = 0; k < 16; ++k)
        s += bf2f(A[m * 32 + 2 * k]) * bf2f(B[k * 32 + 2 * n]) + bf2f(A[m * 32 + 2 * k + 1]) * bf2f(B[k * 32 + 2 * n + 1]);
      C[m * 16 + n] = s;
    }
}
#define TZERO(t) emu_zero(t)
#define TLOAD(t, p, s) emu_load(t, p, s)
#define TSTORE(t, p, s) emu_store(t, p, s)
#define TDP(c, a, b) emu_dp(c, a, b)
#define TCONFIG(cfg) ((void)(cfg))
#define TRELEASE() ((void)0)
#define AMX_TARGET __attribute__((target("avx512f,avx512bw,avx512vl")))
#else
#define TZERO(t) _tile_zero(t)
#define TLOAD(t, p, s) _tile_loadd(t, p, s)
#define TSTORE(t, p, s) _tile_stored(t, p, s)
#define TDP(c, a, b) _tile_dpbf16ps(c, a, b)
#define TCONFIG(cfg) _tile_loadconfig(cfg)
#define TRELEASE() _tile_release()
#define AMX_TARGET __attribute__((target("amx-tile,amx-bf16,avx512f,avx512bw,avx512vl")))
#endif

inline uint16_t f2bf(float f) {  // round to nearest even (finite inputs)
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

// 16 fp32 -> 16 bf16 (round to nearest even, finite inputs), as f2bf
AMX_TARGET inline __m256i cvt_bf16(__m512 v) {
  const __m512i u = _mm512_castps_si512(v);
  const __m512i r = _mm512_add_epi32(
      u, _mm512_add_epi32(_mm512_set1_epi32(0x7fff), _mm512_and_si512(_mm512_srli_epi32(u, 16), _mm512_set1_epi32(1))));
  return _mm512_cvtepi32_epi16(_mm512_srli_epi32(r, 16));
}

// e^x, |rel err| ~ 2e-7 on the clamped range: 2^n e^r with |r| <= ln2 / 2
AMX_TARGET inline __m512 exp16(__m512 x) {
  x = _mm512_min_ps(_mm512_max_ps(x, _mm512_set1_ps(-87.3f)), _mm512_set1_ps(88.3f));
  const __m512 n = _mm512_roundscale_ps(_mm512_mul_ps(x, _mm512_set1_ps(1.44269504088896341f)),
                                        _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  __m512 r = _mm512_fnmadd_ps(n, _mm512_set1_ps(0.693145751953125f), x);
  r = _mm512_fnmadd_ps(n, _mm512_set1_ps(1.428606765330187e-06f), r);
  __m512 q = _mm512_set1_ps(1.0f / 5040.0f);
  q = _mm512_fmadd_ps(q, r, _mm512_set1_ps(1.0f / 720.0f));
  q = _mm512_fmadd_ps(q, r, _mm512_set1_ps(1.0f / 120.0f));
  q = _mm512_fmadd_ps(q, r, _mm512_set1_ps(1.0f / 24.0f));
  q = _mm512_fmadd_ps(q, r, _mm512_set1_ps(1.0f / 6.0f));
  q = _mm512_fmadd_ps(q, r, _mm512_set1_ps(0.5f));
  q = _mm512_fmadd_ps(q, r, _mm512_set1_ps(1.0f));
  q = _mm512_fmadd_ps(q, r, _mm512_set1_ps(1.0f));
  return _mm512_scalef_ps(q, n);
}

// erf(x), Abramowitz & Stegun 7.1.26 (|abs err| <= 1.5e-7)
AMX_TARGET inline __m512 erf16(__m512 x) {
  const __m512 ax = _mm512_abs_ps(x);
  const __m512 t = _mm512_div_ps(_mm512_set1_ps(1.0f), _mm512_fmadd_ps(_mm512_set1_ps(0.3275911f), ax,
                                                                         _mm512_set1_ps(1.0f)));
  __m512 p = _mm512_set1_ps(1.061405429f);
  p = _mm512_fmadd_ps(p, t, _mm512_set1_ps(-1.453152027f));
  p = _mm512_fmadd_ps(p, t, _mm512_set1_ps(1.421413741f));
  p = _mm512_fmadd_ps(p, t, _mm512_set1_ps(-0.284496736f));
  p = _mm512_fmadd_ps(p, t, _mm512_set1_ps(0.254829592f));
  p = _mm512_mul_ps(p, t);
  const __m512 e = exp16(_mm512_mul_ps(_mm512_sub_ps(_mm512_setzero_ps(), ax), ax));
  const __m512 y = _mm512_fnmadd_ps(p, e, _mm512_set1_ps(1.0f));
  return _mm512_mask_sub_ps(y, _mm512_cmp_ps_mask(x, _mm512_setzero_ps(), _CMP_LT_OQ), _mm512_setzero_ps(), y);
}

AMX_TARGET inline __m512 act16(int act, __m512 z) {
  if (act == 1)  // SiLU z / (1 + e^-z)
    return _mm512_div_ps(z, _mm512_add_ps(_mm512_set1_ps(1.0f), exp16(_mm512_sub_ps(_mm512_setzero_ps(), z))));
  if (act == 2)  // GELU 0.5 z (1 + erf(z / sqrt 2))
    return _mm512_mul_ps(_mm512_mul_ps(_mm512_set1_ps(0.5f), z),
                         _mm512_add_ps(_mm512_set1_ps(1.0f), erf16(_mm512_mul_ps(z, _mm512_set1_ps(0.70710678118654752f)))));
  return z;
}

// 64-byte aligned scratch that only grows (tile rows are 64 bytes: an
// unaligned row straddles two cache lines and doubles the L2 traffic)
struct Scratch {
  uint16_t* p = nullptr;
  size_t n = 0;
  uint16_t* get(size_t elems) {
    if (elems > n) {
      free(p);
      n = std::max(elems, n * 2);
      p = static_cast<uint16_t*>(aligned_alloc(64, (n * 2 + 63) / 64 * 64));
    }
    return p;
  }
  ~Scratch() { free(p); }
};

struct AmxShared {
  const CCProblem& p;
  int64_t T16, G16, K32, KP, n16, b1p, ldm_b, ldn, n_slabs;
  uint16_t* xp;  // [G16][KP][16][2]
  uint16_t* a;   // [T16][b1p]
  const int* chunk_of;
  std::atomic<int64_t>* cursor;
};

AMX_TARGET void tile_config() {
  TileConfig cfg{};
  cfg.palette = 1;
  for (int i = 0; i < 8; ++i) {
    cfg.colsb[i] = 64;
    cfg.rows[i] = 16;
  }
  TCONFIG(&cfg);
}

// K is walked in chunks of kKc so that one chunk's tiles (weights, x or `a`,
// the W2 repack) stay in L2 -- with an SMT sibling on the same core only about
// half of it -- while the accumulators are parked in a small fp32 buffer
// between chunks.  Each output is still summed in one fixed order.
constexpr int64_t kKc = 1024;

// ---- phase 1: the up GEMM and the activation, one 16-row hidden slab at a time ----
AMX_TARGET void up_worker(const AmxShared& S) {
  const CCProblem& p = S.p;
  const int64_t T = p.T, G16 = S.G16, K32 = S.K32, KP = S.KP, b1p = S.b1p, ldm_b = S.ldm_b;
  static thread_local Scratch pad1s, pad3s, zs;
  uint16_t* const pad1 = pad1s.get(size_t(16 * p.ldm));
  uint16_t* const pad3 = pad3s.get(size_t(16 * p.ldm));
  // accumulators of every token-group pair: [pair][W1 g0, W1 g1, W3 g0, W3 g1][16 x 16] fp32
  float* const zbuf = reinterpret_cast<float*>(zs.get(size_t((G16 + 1) / 2 * 4 * 256 * 2)));
  tile_config();
  alignas(64) uint16_t ab[16][16];  // [hidden row][token] of one 16 x 16 activation block
  static const bool prof = getenv("SP_AMX_PROF") != nullptr;
  unsigned long long c_up = 0, c_act = 0, tc = 0;
  int slabs = 0;
  for (;;) {
    const int64_t s = S.cursor->fetch_add(1, std::memory_order_relaxed);
    if (s >= S.n_slabs) break;
    const int64_t h0 = 16 * s;
    const int64_t valid = std::min<int64_t>(16, p.b1 - h0);
    const HostChunk& c = p.chunks[S.chunk_of[size_t(h0)]];  // chunks start at multiples of 64 rows
    const char* w1 = static_cast<const char*>(c.w1t) + (h0 - c.r0) * ldm_b;
    const char* w3 = p.gated ? static_cast<const char*>(c.w3t) + (h0 - c.r0) * ldm_b : nullptr;
    if (valid < 16) {  // last rows of the CC block: never read past them
      std::fill(pad1, pad1 + 16 * p.ldm, 0);
      memcpy(pad1, w1, size_t(valid * ldm_b));
      w1 = reinterpret_cast<const char*>(pad1);
      if (p.gated) {
        std::fill(pad3, pad3 + 16 * p.ldm, 0);
        memcpy(pad3, w3, size_t(valid * ldm_b));
        w3 = reinterpret_cast<const char*>(pad3);
      }
    }
    ++slabs;
    if (prof) tc = __rdtsc();
    for (int64_t kc = 0; kc < K32; kc += kKc) {
      const int64_t ke = std::min(K32, kc + kKc);
      for (int64_t g0 = 0; g0 < G16; g0 += 2) {
        const bool two = g0 + 1 < G16;
        float* zc = zbuf + (g0 / 2) * 4 * 256;
        if (kc == 0) {
          TZERO(4);
          TZERO(5);
          TZERO(6);
          TZERO(7);
        } else {
          TLOAD(4, zc, 64);
          TLOAD(5, zc + 256, 64);
          TLOAD(6, zc + 512, 64);
          TLOAD(7, zc + 768, 64);
        }
        const uint16_t* xg0 = S.xp + size_t(g0 * KP * 32);
        const uint16_t* xg1 = S.xp + size_t((g0 + 1) * KP * 32);
        // Tile registers are not renamed: a load into a tile waits for every
        // product still reading it.  So the loop is software pipelined -- each
        // tile of the NEXT k step is loaded right after its last reader in this
        // step (W1 after its two products, x0 after the W3 x0 product, x1 and W3
        // at the end), and those loads run under the remaining products instead
        // of in front of the next step's.  The weight rows are also prefetched
        // ahead (first token-group pass only; later passes find them in L2).
        TLOAD(0, w1 + kc * 2, ldm_b);
        if (p.gated) TLOAD(1, w3 + kc * 2, ldm_b);
        TLOAD(2, xg0 + (kc / 2) * 32, 64);
        if (two) TLOAD(3, xg1 + (kc / 2) * 32, 64);
        for (int64_t k = kc; k < ke; k += 32) {
          const int64_t kn = k + 32;
          const bool nx = kn < ke;
          if (g0 == 0)
            for (int i = 0; i < 16; ++i) {
              _mm_prefetch(w1 + i * ldm_b + k * 2 + kUpPf, _MM_HINT_T0);
              if (p.gated) _mm_prefetch(w3 + i * ldm_b + k * 2 + kUpPf, _MM_HINT_T0);
            }
          TDP(4, 0, 2);
          if (two) TDP(5, 0, 3);
          if (nx) TLOAD(0, w1 + kn * 2, ldm_b);
          if (p.gated) TDP(6, 1, 2);
          if (nx) TLOAD(2, xg0 + (kn / 2) * 32, 64);
          if (p.gated && two) TDP(7, 1, 3);
          if (nx) {
            if (two) TLOAD(3, xg1 + (kn / 2) * 32, 64);
            if (p.gated) TLOAD(1, w3 + kn * 2, ldm_b);
          }
        }
        TSTORE(4, zc, 64);
        TSTORE(5, zc + 256, 64);
        TSTORE(6, zc + 512, 64);
        TSTORE(7, zc + 768, 64);
      }
    }
    if (prof) {
      c_up += __rdtsc() - tc;
      tc = __rdtsc();
    }
    for (int64_t g = 0; g < G16; ++g) {
      const float* z1 = zbuf + (g / 2) * 4 * 256 + (g & 1) * 256;
      const float* z3 = z1 + 512;
      const int64_t t0 = 16 * g;
      for (int i = 0; i < 16; ++i) {  // hidden row h0 + i: 16 tokens at once
        __m512 v = _mm512_setzero_ps();
        if (i < valid) {
          v = act16(p.act, _mm512_load_ps(z1 + i * 16));
          if (p.gated) v = _mm512_mul_ps(v, _mm512_load_ps(z3 + i * 16));
          if (t0 + 16 > T)  // padded tokens stay exactly zero
            v = _mm512_maskz_mov_ps(__mmask16((1u << (T - t0 > 0 ? T - t0 : 0)) - 1u), v);
        }
        _mm256_store_si256(reinterpret_cast<__m256i*>(ab[i]), cvt_bf16(v));
      }
      for (int j = 0; j < 16; ++j) {  // a[t][h0 .. h0 + 16): the 16 x 16 block transposed
        uint16_t* dst = S.a + size_t((t0 + j) * b1p + h0);
        for (int i = 0; i < 16; ++i) dst[i] = ab[i][j];
      }
    }
    if (prof) c_act += __rdtsc() - tc;
  }
  TRELEASE();
  if (prof && slabs)
    fprintf(stderr, "  up thread: %d slabs, kcycles tiles %llu act %llu\n", slabs, c_up >> 10, c_act >> 10);
}

// W2 rows of columns [n0, n0 + nr) in VNNI pairs: dst[kp][n][e] = W2[2 kp + e][n0 + n],
// zero past b1 (b1p / 2 pairs)
AMX_TARGET void repack_w2_round(const CCProblem& p, const int* chunk_of, int64_t b1p, int64_t n0, int64_t nr,
                                uint16_t* w2p) {
  const int64_t ldn = p.ldn;
  for (int64_t kp = 0; kp < b1p / 2; ++kp) {
    const int64_t ha = 2 * kp, hb = ha + 1;
    uint16_t* dst = w2p + size_t(kp * nr * 2);
    const uint16_t* ra = nullptr;
    const uint16_t* rb = nullptr;
    if (ha < p.b1) {
      const HostChunk& c = p.chunks[chunk_of[size_t(ha)]];
      ra = static_cast<const uint16_t*>(c.w2) + (ha - c.r0) * ldn + n0;
    }
    if (hb < p.b1) {
      const HostChunk& c = p.chunks[chunk_of[size_t(hb)]];
      rb = static_cast<const uint16_t*>(c.w2) + (hb - c.r0) * ldn + n0;
    }
    if (ha + 6 < p.b1) {  // the rows three pairs ahead
      const HostChunk& c = p.chunks[chunk_of[size_t(ha + 6)]];
      const char* q = reinterpret_cast<const char*>(static_cast<const uint16_t*>(c.w2) + (ha + 6 - c.r0) * ldn + n0);
      for (int64_t off = 0; off < nr * 2; off += 64) _mm_prefetch(q + off, _MM_HINT_T0);
      if (ha + 7 < p.b1)
        for (int64_t off = 0; off < nr * 2; off += 64) _mm_prefetch(q + ldn * 2 + off, _MM_HINT_T0);
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
}

// ---- phase 2: the down GEMM, kRoundCols output columns at a time ----
AMX_TARGET void down_worker(const AmxShared& S, std::atomic<int64_t>* rounds, int tid) {
  const CCProblem& p = S.p;
  const int64_t T = p.T, N = p.N, T16 = S.T16, G16 = S.G16, n16 = S.n16, b1p = S.b1p, ldn = S.ldn;
  const int64_t ntiles = n16 / 16, per = kRoundCols / 16;
  static thread_local Scratch w2ps, ys;
  uint16_t* const w2p = p.w2p ? nullptr : w2ps.get(size_t(b1p / 2 * kRoundCols * 2));
  float* const ybuf = reinterpret_cast<float*>(ys.get(size_t(T16 * kRoundCols * 2)));  // [T16][nr] fp32
  tile_config();
  static const bool prof = getenv("SP_AMX_PROF") != nullptr;
  unsigned long long c_rep = 0, c_dn = 0, tc = 0;
  for (;;) {  // rounds of kRoundCols output columns, claimed dynamically (the host's vCPUs differ in speed)
    const int64_t jr = per * rounds->fetch_add(1, std::memory_order_relaxed);
    if (jr >= ntiles) break;
    if (prof) tc = __rdtsc();
    const int64_t je = std::min(ntiles, jr + per);
    const int64_t n0 = 16 * jr, nr = 16 * (je - jr);
    // W2 rows of the round's columns in VNNI pairs: prepacked once per layer
    // (amx_prepack_w2), else repacked here
    const uint16_t* w2r = w2p;
    if (p.w2p)
      w2r = p.w2p + size_t(b1p) * size_t(n0);
    else
      repack_w2_round(p, S.chunk_of, b1p, n0, nr, w2p);
    if (prof) {
      c_rep += __rdtsc() - tc;
      tc = __rdtsc();
    }
    // 2 token groups x 2 column tiles per pass; the hidden range in kKc chunks,
    // the accumulators parked in ybuf [T16][nr] between chunks
    for (int64_t kc = 0; kc < b1p; kc += kKc) {
      const int64_t ke = std::min(b1p, kc + kKc);
      for (int64_t g = 0; g < G16; g += 2) {
        const bool g2 = g + 1 < G16;
        const uint16_t* a0 = S.a + size_t(16 * g * b1p);
        const uint16_t* a1 = a0 + 16 * b1p;
        for (int64_t jn = 0; jn < nr / 16; jn += 2) {
          const bool j2 = jn + 1 < nr / 16;
          float* y0 = ybuf + (16 * g) * nr + 16 * jn;  // tile (g, jn); +16: jn + 1; +16 nr rows: g + 1
          if (kc == 0) {
            TZERO(0);
            TZERO(1);
            TZERO(2);
            TZERO(3);
          } else {
            TLOAD(0, y0, nr * 4);
            if (j2) TLOAD(1, y0 + 16, nr * 4);
            if (g2) TLOAD(2, y0 + 16 * nr, nr * 4);
            if (g2 && j2) TLOAD(3, y0 + 16 * nr + 16, nr * 4);
          }
          const uint16_t* b0 = w2r + jn * 32;
          // software pipelined like the up loop: each tile of the next hidden
          // step is loaded right after its last reader in this one
          const int64_t s0 = kc / 32, se = ke / 32;
          TLOAD(4, a0 + 32 * s0, b1p * 2);
          TLOAD(6, b0 + (16 * s0) * nr * 2, nr * 4);
          if (j2) TLOAD(7, b0 + (16 * s0) * nr * 2 + 32, nr * 4);
          if (g2) TLOAD(5, a1 + 32 * s0, b1p * 2);
          for (int64_t sl = s0; sl < se; ++sl) {
            const int64_t sn = sl + 1;
            const bool nx = sn < se;
            TDP(0, 4, 6);
            if (j2) TDP(1, 4, 7);
            if (nx) TLOAD(4, a0 + 32 * sn, b1p * 2);
            if (g2) TDP(2, 5, 6);
            if (nx) TLOAD(6, b0 + (16 * sn) * nr * 2, nr * 4);
            if (g2 && j2) TDP(3, 5, 7);
            if (nx) {
              if (j2) TLOAD(7, b0 + (16 * sn) * nr * 2 + 32, nr * 4);
              if (g2) TLOAD(5, a1 + 32 * sn, b1p * 2);
            }
          }
          TSTORE(0, y0, nr * 4);
          if (j2) TSTORE(1, y0 + 16, nr * 4);
          if (g2) TSTORE(2, y0 + 16 * nr, nr * 4);
          if (g2 && j2) TSTORE(3, y0 + 16 * nr + 16, nr * 4);
        }
      }
    }
    for (int64_t t = 0; t < T; ++t) {  // the round's valid rows and columns
      const int64_t nv = std::min(nr, N - n0);
      memcpy(p.y + t * N + n0, ybuf + t * nr, size_t(nv) * 4);
    }
    if (prof) c_dn += __rdtsc() - tc;
  }
  TRELEASE();
  if (prof && tid == 0) fprintf(stderr, "  down thread 0 kcycles: repack %llu tiles %llu\n", c_rep >> 10, c_dn >> 10);
}

}  // namespace

bool host_has_amx() {
#ifdef SP_AMX_EMULATE
  return true;
#else
  static const bool ok = [] {
    if (!__builtin_cpu_supports("amx-tile") || !__builtin_cpu_supports("amx-bf16") ||
        !__builtin_cpu_supports("avx512f") || !__builtin_cpu_supports("avx512bw"))
      return false;
    // Linux hands out the 8 KB tile state only on request (per process)
    return syscall(SYS_arch_prctl, kArchReqXcompPerm, kXfeatureXtiledata) == 0;
  }();
  return ok;
#endif
}

size_t amx_w2_prepack_elems(const CCProblem& p) {
  const int64_t b1p = (p.b1 + 31) / 32 * 32, n16 = (p.N + 15) / 16 * 16;
  return size_t(b1p) * size_t(n16);
}

// round r (columns [128 r, 128 r + nr_r)) at out + b1p * 128 r, laid out as the
// down phase's repack: [b1p / 2][nr_r][2]
void amx_prepack_w2(const CCProblem& p, uint16_t* out, ThreadPool& pool, int threads) {
  const int64_t b1p = (p.b1 + 31) / 32 * 32, n16 = (p.N + 15) / 16 * 16;
  std::vector<int> chunk_of(size_t(b1p), 0);
  for (int c = 0; c < p.n_chunks; ++c)
    for (int64_t r = 0; r < p.chunks[c].rc; ++r) chunk_of[size_t(p.chunks[c].r0 + r)] = c;
  const int64_t n_rounds = (n16 + kRoundCols - 1) / kRoundCols;
  std::atomic<int64_t> next{0};
  pool.run(int(std::min<int64_t>(std::max(1, std::min(threads, pool.size())), n_rounds)), [&](int, int) {
    for (int64_t r; (r = next.fetch_add(1)) < n_rounds;) {
      const int64_t n0 = r * kRoundCols, nr = std::min(kRoundCols, n16 - n0);
      repack_w2_round(p, chunk_of.data(), b1p, n0, nr, out + size_t(b1p) * size_t(n0));
    }
  });
}

void cc_forward_amx(const CCProblem& p, ThreadPool& pool, int threads) {
  const int64_t T = p.T, M = p.M;
  const int64_t T16 = (T + 15) / 16 * 16, G16 = T16 / 16;
  const int64_t K32 = (M + 31) / 32 * 32;  // W rows are zero padded to ldm >= roundup(M, 64)
  const int64_t KP = K32 / 2;              // k pairs
  const int64_t n16 = (p.N + 15) / 16 * 16;
  const int64_t b1p = (p.b1 + 31) / 32 * 32;
  const int nthr = std::max(1, std::min(threads, pool.size()));
  const auto t0 = std::chrono::steady_clock::now();

  // persistent scratch of the calling thread (workers get raw pointers): fresh
  // large allocations are mmap'd and every first touch is a page fault
  static thread_local Scratch tl_xp, tl_a;
  uint16_t* const xp = tl_xp.get(size_t(G16 * KP * 32));
  uint16_t* const a = tl_a.get(size_t(T16 * b1p));
  std::vector<int> chunk_of(size_t(b1p), 0);  // hidden row -> chunk
  for (int c = 0; c < p.n_chunks; ++c)
    for (int64_t r = 0; r < p.chunks[c].rc; ++r) chunk_of[size_t(p.chunks[c].r0 + r)] = c;

  // pack: x -> bf16 VNNI pairs xp[g][kp][j][e] = x[16 g + j][2 kp + e] (zero past T and M)
  pool.run(nthr, [&](int tid, int n) {
    const int64_t k0 = KP * tid / n, k1 = KP * (tid + 1) / n;
    for (int64_t g = 0; g < G16; ++g)
      for (int64_t kp = k0; kp < k1; ++kp) {
        uint16_t* dst = xp + size_t((g * KP + kp) * 32);
        for (int64_t j = 0; j < 16; ++j) {
          const int64_t t = 16 * g + j;
          for (int e = 0; e < 2; ++e) {
            const int64_t k = 2 * kp + e;
            dst[j * 2 + e] = (t < T && k < M) ? f2bf(p.x[t * p.ldx + k]) : uint16_t(0);
          }
        }
      }
  });
  // the hidden columns past b1 (to the next multiple of 32) stay zero in `a`
  if (b1p > p.b1)
    for (int64_t t = 0; t < T16; ++t) std::fill(a + t * b1p + p.b1, a + (t + 1) * b1p, uint16_t(0));

  // SP_AMX_PROF=1: phase wall times to stderr (tuning aid)
  static const bool prof = getenv("SP_AMX_PROF") != nullptr;
  const auto t1 = std::chrono::steady_clock::now();
  std::atomic<int64_t> cursor{0};
  AmxShared S{p, T16, G16, K32, KP, n16, b1p, p.ldm * 2, p.ldn, (p.b1 + 15) / 16, xp, a, chunk_of.data(), &cursor};
  pool.run(int(std::min<int64_t>(nthr, S.n_slabs)), [&](int, int) { up_worker(S); });
  const auto t2 = std::chrono::steady_clock::now();
  std::atomic<int64_t> rounds{0};
  pool.run(int(std::min<int64_t>(nthr, (n16 / 16 + kRoundCols / 16 - 1) / (kRoundCols / 16))),
           [&](int tid, int) { down_worker(S, &rounds, tid); });
  if (prof) {
    const auto t3 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    fprintf(stderr, "amx T=%lld: pack %.0f us  up %.0f us  down %.0f us\n", (long long)T, us(t0, t1), us(t1, t2),
            us(t2, t3));
  }
}

}  // namespace sp
