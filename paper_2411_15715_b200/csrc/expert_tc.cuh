// expert_tc.cuh -- one persistent tcgen05 kernel per HBM-resident block at
// prefill token counts (T <= 128): up GEMM + activation/gate + down GEMM.
//
// Why: at 16-128 tokens per expert a block is HBM-bound (one 4096 x 14336
// SwiGLU expert is 352 MB of weights, ~54 us at the measured copy rate), and the
// four-kernel chain of gemm_tc.cuh (gather -> up -> swiglu_reduce -> down ->
// finalize of the down splits) loses ~25 us to what lies between the weight
// streams: the up GEMM has 112 row tiles for 148 SMs, each kernel ramps up and
// drains, and the down splits round-trip through output slices.
//
// This kernel runs ONE CTA per SM for the whole block and streams the block's
// weights exactly once, back to back:
//   phase U (up)  : units (row tile j of 128 hidden units, k-block of 64 of M);
//                   D[h, t] = W1t[h, :] . x[t, :]  and  W3t  (two TMEM accumulators)
//   phase D (down): units (column tile c of 256 outputs, k-block of 64 hidden units);
//                   D[n, t] = W2[:, n] . a[t, :]   (W2 MN-major, two 128-column sub-tiles)
// Each phase's units are cut into G equal contiguous ranges, one per CTA
// (stream-K), so every SM streams the same number of weight bytes.  A range
// covers whole tiles and at most two partial ones; a tile split across CTAs is
// finished by a fix-up through fp32 partials in global memory (L2), ordered by
// per-launch epoch flags -- all sums in a fixed order, so the result depends only
// on (shape, T, G), never on timing:
//   * up tile j: the CTA holding its first k-block (it reaches it LAST in its
//     range) adds the other contributors' partials to its TMEM accumulator in
//     contributor order, applies act * gate, stores bf16 `a`, and publishes
//     ready[j];
//   * down tile c: every contributor stores its partial [t][256] and then sums a
//     1/n share of the tile over all n partials (contributor order) into the
//     output slice y -- the reduction is spread over the tile's CTAs.
// The producer streams the W2 boxes of the down phase as soon as ring slots
// free up (they depend on nothing) and waits on ready[j] only before the box
// of `a` it needs, so the phase change costs no bubble in the weight stream.
//
// Deadlock freedom: all G <= #SMs CTAs are co-resident (1 CTA per SM by shared
// memory, and the kernel never triggers dependent launches early).  Up
// partials are written before any wait of their CTA's epilogue; owners wait
// only on up partials; down waits only on up `ready` flags and on down tiles'
// partials, which by induction over the tile index are all written.
//
// Roles (320 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 2..9 epilogue (TMEM lane quarter = warp % 4, two warps per
// quarter splitting the token chunks).  TMEM holds two
// accumulator buffers (2 x 2 x NT columns), so a tile's epilogue overlaps the
// next tile's MMAs.
#pragma once

#include "gemm_tc.cuh"

namespace sp {
namespace tc {

constexpr int kFusedMaxNT = 128;
constexpr int kFusedEpiWarps = 8;
constexpr int kFusedL2Ahead = 8;  // down units whose W2 is pulled into L2 beyond the smem ring
constexpr int kFusedEpiThreads = kFusedEpiWarps * 32;
constexpr int kFusedThreads = 64 + kFusedEpiThreads;  // producer warp, MMA warp, epilogue warps
constexpr int kDownCols = 2 * BM;  // output columns per down tile (two sub-tiles)

struct FusedArgs {
  int R, M, N, T;      // hidden rows of the block, model dim (up K), output columns, tokens
  int act, gated;
  int G;               // CTAs
  int GU, GD;          // CTAs with work in the up / down phase (min(G, units): every range non-empty)
  int nkU, mU, U;      // up: k-blocks per tile, tiles, units (= mU * nkU)
  int nkD, mD, D;      // down: k-blocks per tile, tiles, units
  int QU, QD;          // partial slots per up / down tile
  int stages;
  uint32_t epoch;      // flags equal to `epoch` were written by this launch
  __nv_bfloat16* a_out;  // [T][lda] bf16 hidden activations
  int64_t lda;
  float* y;            // [T][ldy] fp32 output slice (stored, every column < N of every token < T)
  int64_t ldy;
  float* ws_up;        // [mU][QU][2][NT][128]  fp32 partial pre-activations
  float* ws_dn;        // [mD][QD][NT][256]     fp32 partial outputs
  uint32_t* up_flag;   // [mU][QU]
  uint32_t* ready;     // [mU]
  uint32_t* dn_flag;   // [mD][QD]
  unsigned long long* stamps;  // debug (SP_KSTAMPS=1): [G][16] %globaltimer phase stamps, or null
};

// CTA i owns units [range_begin(i), range_begin(i + 1)) of a phase with `units` units
__host__ __device__ __forceinline__ int range_begin(int i, int units, int G) {
  return int((int64_t(i) * units) / G);
}
// the CTA whose range holds unit u
__host__ __device__ __forceinline__ int cta_of(int u, int units, int G) {
  return int((int64_t(u + 1) * G + units - 1) / units) - 1;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_epoch(const uint32_t* p, uint32_t epoch) {
  while (ld_acquire_u32(p) != epoch) __nanosleep(32);
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void fused_epi_sync() {
  asm volatile("bar.sync 2, %0;" ::"n"(kFusedEpiThreads) : "memory");
}
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

#define SP_FSTAMP(i)                                                     \
  do {                                                                   \
    if (g.stamps) g.stamps[size_t(blockIdx.x) * 16 + (i)] = global_ns(); \
  } while (0)

__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

// Walk a CTA's segments (maximal runs of its range inside one tile) in order:
// f(down, tile, k0, k1, seg) for up segments then down segments.
template <typename F>
__device__ __forceinline__ void for_each_segment(const FusedArgs& g, int cta, F&& f) {
  int seg = 0;
  if (cta < g.GU) {
    const int u1 = range_begin(cta + 1, g.U, g.GU);
    for (int u = range_begin(cta, g.U, g.GU); u < u1;) {
      const int tile = u / g.nkU, e = min(u1, (tile + 1) * g.nkU);
      f(false, tile, u - tile * g.nkU, e - tile * g.nkU, seg++);
      u = e;
    }
  }
  if (cta < g.GD) {
    const int d1 = range_begin(cta + 1, g.D, g.GD);
    for (int d = range_begin(cta, g.D, g.GD); d < d1;) {
      const int tile = d / g.nkD, e = min(d1, (tile + 1) * g.nkD);
      f(true, tile, d - tile * g.nkD, e - tile * g.nkD, seg++);
      d = e;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(kFusedThreads, 1)
    expert_tc_kernel(const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW3,
                     const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW2,
                     const __grid_constant__ CUtensorMap tmA, const FusedArgs g) {
  static_assert(NT % 16 == 0 && NT <= kFusedMaxNT, "token tile");
  constexpr int A_BYTES = BM * BK * 2;  // 16 KB: one 128-row weight box (or 2 x 64-column W2 boxes)
  constexpr int B_BYTES = NT * BK * 2;  // x / a box
  constexpr int STAGE = 2 * A_BYTES + B_BYTES;
  constexpr int BUF_COLS = 2 * NT;      // one accumulator buffer: two NT-column accumulators
  constexpr int TMEM_COLS = 2 * BUF_COLS <= 32 ? 32 : 2 * BUF_COLS <= 64 ? 64 : 2 * BUF_COLS <= 128 ? 128
                            : 2 * BUF_COLS <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * STAGE);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2] accumulator buffer b complete
  uint64_t* tempty = tfull + 2;  // [2] accumulator buffer b drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int na_up = g.gated ? 2 : 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW2)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int u0 = cta < g.GU ? range_begin(cta, g.U, g.GU) : 0, u1 = cta < g.GU ? range_begin(cta + 1, g.U, g.GU) : 0;
  const int d0 = cta < g.GD ? range_begin(cta, g.D, g.GD) : 0, d1 = cta < g.GD ? range_begin(cta + 1, g.D, g.GD) : 0;
  const int nU = u1 - u0, n_all = nU + (d1 - d0);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_w = evict_first_policy();  // weights: streamed once
      int ready_tile = -1;                          // last up tile seen ready
      auto issue_w = [&](int i) {
        const int s = i % S;
        unsigned char* st = smem + size_t(s) * STAGE;
        if (i < nU) {
          const int u = u0 + i, tile = u / g.nkU, kb = u - tile * g.nkU;
          mbar_expect_tx(&full[s], na_up * A_BYTES + B_BYTES);
          tma_load_2d_hint(st, &tmW1, &full[s], kb * BK, tile * BM, pol_w);
          if (na_up == 2) tma_load_2d_hint(st + A_BYTES, &tmW3, &full[s], kb * BK, tile * BM, pol_w);
        } else {
          const int d = d0 + (i - nU), tile = d / g.nkD, kb = d - tile * g.nkD;
          const int c0 = tile * kDownCols;
          mbar_expect_tx(&full[s], 2 * A_BYTES + B_BYTES);
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            tma_load_2d_hint(st + a * A_BYTES, &tmW2, &full[s], c0 + a * BM, kb * BK, pol_w);
            tma_load_2d_hint(st + a * A_BYTES + BK * 128, &tmW2, &full[s], c0 + a * BM + 64, kb * BK, pol_w);
          }
        }
      };
      // the box of x / `a` for unit i; false (nothing issued) while the up tile
      // a down unit reads is not published yet
      auto try_issue_b = [&](int i) -> bool {
        const int s = i % S;
        unsigned char* st = smem + size_t(s) * STAGE + 2 * A_BYTES;
        if (i < nU) {
          const int u = u0 + i, kb = u % g.nkU;
          tma_load_2d(st, &tmX, &full[s], kb * BK, 0);
          return true;
        }
        const int d = d0 + (i - nU), kb = d % g.nkD;
        const int need = (kb * BK) / BM;  // up tile holding hidden units [kb * 64, kb * 64 + 64)
        if (need != ready_tile) {
          if (ld_acquire_u32(g.ready + need) != g.epoch) return false;
          fence_proxy_async_global();  // the generic-proxy `a` stores before the TMA read
          ready_tile = need;
        }
        tma_load_2d(st, &tmA, &full[s], kb * BK, 0);
        return true;
      };
      // Weights run up to S units ahead of the x / `a` boxes: at the phase change
      // the W2 boxes fill the ring while the producer waits for the up tiles'
      // `ready` flags.  Waiting on a slot of unit iw >= S needs only unit iw - S
      // consumed, whose box was issued (iw - ib < S), so this never deadlocks.
      SP_FSTAMP(0);
      int iw = 0, ib = 0, ip = 0;  // next unit: weights to smem, x / `a` box, W2 to L2
      while (iw < n_all && iw < S) issue_w(iw++);
      grid_dep_wait();  // x is written by the predecessor grid
      while (ib < n_all) {
        if (ib < iw) {
          if (try_issue_b(ib)) {
            if (ib == nU - 1) SP_FSTAMP(1);
            if (ib == nU) SP_FSTAMP(2);
            ++ib;
            continue;
          }
        }
        if (iw < n_all && iw - ib < S) {
          if (iw >= S) mbar_wait(&empty[iw % S], ((iw / S) - 1) & 1);
          issue_w(iw++);
          continue;
        }
        // blocked on an up tile with the ring full of W2: keep DRAM busy by
        // pulling the next units' W2 boxes into L2 (they are read from there)
        if (ip < iw) ip = iw;
        if (ip < n_all && ip < ib + S + kFusedL2Ahead) {
          const int d = d0 + (ip - nU), tile = d / g.nkD, kb = d - tile * g.nkD;
          const int c0 = tile * kDownCols;
#pragma unroll
          for (int a = 0; a < 4; ++a) tma_prefetch_l2_2d(&tmW2, c0 + a * 64, kb * BK);
          ++ip;
          continue;
        }
        __nanosleep(64);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int it = 0;
    for_each_segment(g, cta, [&](bool down, int, int k0, int k1, int seg) {
      const int buf = seg & 1;
      if (seg >= 2) mbar_wait(&tempty[buf], ((seg >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d_acc = tmem + uint32_t(buf * BUF_COLS);
      const uint32_t idesc = umma_idesc(BM, NT, down);
      const int na = down ? 2 : na_up;
      for (int k = k0; k < k1; ++k, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const unsigned char* st = smem + size_t(s) * STAGE;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t b = umma_desc(st + 2 * A_BYTES + kk * 32, 16, 1024);
            for (int a = 0; a < na; ++a) {
              const uint64_t ad = down ? umma_desc(st + a * A_BYTES + kk * UK * 128, BK * 128, 1024)
                                       : umma_desc(st + a * A_BYTES + kk * 32, 16, 1024);
              umma_bf16(d_acc + uint32_t(a * NT), ad, b, idesc, (k > k0 || kk > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) {
        umma_commit(&tfull[buf]);
        SP_FSTAMP(down ? 5 : 3);
      }
      __syncwarp();
    });
  } else {
    // ---------------- epilogue: warps 2..9; warp w owns TMEM lanes 32 * (w % 4) ----------------
    // Two warps per lane quarter split a tile's 8-token chunks (half h takes
    // chunks h, h + 2, ...), so both have work from T = 9 on and twice the L2
    // loads of a fix-up are in flight.
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;  // weight row (up) / output column (down) inside the tile
    const int et = threadIdx.x - 64;      // 0 .. kFusedEpiThreads - 1
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const int tcap = NT < g.T ? NT : g.T;  // tokens of the tile that exist
    auto contributors = [&](bool down, int tile, int& q, int& n) {
      const int nk = down ? g.nkD : g.nkU;
      const int units = down ? g.D : g.U, gp = down ? g.GD : g.GU;
      const int first = cta_of(tile * nk, units, gp);
      n = cta_of(tile * nk + nk - 1, units, gp) - first + 1;
      q = cta - first;  // this CTA's contributor index in the tile (0 holds k-block 0)
    };
    int n_useg = 0;  // this CTA's up segments (its first down segment has index n_useg)
    for_each_segment(g, cta, [&](bool down, int, int, int, int) { n_useg += down ? 0 : 1; });
    grid_dep_wait();  // no store before the predecessor grid is complete
    // pass 1: drain every accumulator -- up tiles finished (owner) or handed on
    // as partials, down partials stored and published.  No down fix-up waits
    // here, so a CTA's second down tile never waits behind its first one's.
    for_each_segment(g, cta, [&](bool down, int tile, int, int, int seg) {
      const int buf = seg & 1;
      const uint32_t acc = lane_base + uint32_t(buf * BUF_COLS);
      int q, n;
      contributors(down, tile, q, n);
      const bool first_down = down && seg == n_useg;
      if (first_down && et == 0) SP_FSTAMP(11);
      mbar_wait(&tfull[buf], (seg >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (first_down && et == 0) SP_FSTAMP(12);
      auto release_tmem = [&]() {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        fused_epi_sync();
        if (et == 0) mbar_arrive(&tempty[buf]);
      };
      if (!down && q == 0) {
        // owner: TMEM + the other contributors' partials (in order), act * gate, bf16 `a`
        const int m = tile * BM + row;
        const float* wsp = g.ws_up + size_t(tile) * g.QU * 2 * NT * BM + row;
        if (n > 1) {
          if (et == 0)
            for (int qq = 1; qq < n; ++qq) wait_epoch(g.up_flag + size_t(tile) * g.QU + qq, g.epoch);
          fused_epi_sync();
        }
#pragma unroll 1
        for (int c = half * 8; c < tcap; c += 16) {
          uint32_t r0[8], r1[8];
          tmem_ld8_nw(acc + uint32_t(c), r0);
          if (na_up == 2) tmem_ld8_nw(acc + uint32_t(NT + c), r1);
          tmem_ld_wait();
          float z0[8], z1[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            z0[e] = __uint_as_float(r0[e]);
            z1[e] = na_up == 2 ? __uint_as_float(r1[e]) : 1.0f;
          }
          for (int qq = 1; qq < n; ++qq) {
            // all 16 loads of this partial in flight at once (slots hold NT token rows)
            const float* src = wsp + size_t(qq) * 2 * NT * BM + size_t(c) * BM;
            float p0[8], p1[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              p0[e] = __ldcg(src + size_t(e) * BM);
              p1[e] = na_up == 2 ? __ldcg(src + (size_t(NT) + e) * BM) : 0.0f;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              z0[e] += p0[e];
              z1[e] += p1[e];
            }
          }
          if (m < g.R) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              if (c + e < g.T) {
                float v = act_fn(g.act, z0[e]);
                if (na_up == 2) v *= z1[e];
                g.a_out[int64_t(c + e) * g.lda + m] = __float2bfloat16_rn(v);
              }
            }
          }
        }
        release_tmem();
        fence_proxy_async_global();
        __threadfence();
        fused_epi_sync();
        if (et == 0) {
          st_release_u32(g.ready + tile, g.epoch);
          SP_FSTAMP(4);
        }
        return;
      }
      // a partial: up [a][t][128 rows] for the tile's owner, down [t][256 columns]
      float* dst;
      uint32_t* flag;
      int ld1, off1;  // token stride, offset of the second accumulator
      if (!down) {
        dst = g.ws_up + (size_t(tile) * g.QU + q) * 2 * NT * BM + row;
        flag = g.up_flag + size_t(tile) * g.QU + q;
        ld1 = BM;
        off1 = NT * BM;
      } else {
        dst = g.ws_dn + (size_t(tile) * g.QD + q) * NT * kDownCols + row;
        flag = g.dn_flag + size_t(tile) * g.QD + q;
        ld1 = kDownCols;
        off1 = BM;
      }
      const int na = down ? 2 : na_up;
#pragma unroll 1
      for (int c = half * 8; c < tcap; c += 16) {
        uint32_t r0[8], r1[8];
        tmem_ld8_nw(acc + uint32_t(c), r0);
        if (na == 2) tmem_ld8_nw(acc + uint32_t(NT + c), r1);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (c + e < g.T) {
            dst[size_t(c + e) * ld1] = __uint_as_float(r0[e]);
            if (na == 2) dst[size_t(c + e) * ld1 + off1] = __uint_as_float(r1[e]);
          }
      }
      release_tmem();
      __threadfence();
      fused_epi_sync();
      if (et == 0) {
        st_release_u32(flag, g.epoch);
        if (down) SP_FSTAMP(6);
        if (first_down) SP_FSTAMP(8);
      }
    });
    bool first_fix = true;
    // pass 2: each down tile's fix-up, spread over its contributors -- this CTA
    // sums share q of the tile over all n partials (contributor order) into y
    for_each_segment(g, cta, [&](bool down, int tile, int, int, int) {
      if (!down) return;
      int q, n;
      contributors(true, tile, q, n);
      if (et == 0)
        for (int qq = 0; qq < n; ++qq) wait_epoch(g.dn_flag + size_t(tile) * g.QD + qq, g.epoch);
      if (first_fix && et == 0) SP_FSTAMP(9);
      fused_epi_sync();
      const float* wsd = g.ws_dn + size_t(tile) * g.QD * NT * kDownCols;
      constexpr int V = kDownCols / 4;  // float4 per token row of a tile
      const int E = g.T * V;
      const int e0 = int(int64_t(q) * E / n), e1 = int(int64_t(q + 1) * E / n);
      const int col0 = tile * kDownCols;
      for (int e = e0 + et; e < e1; e += kFusedEpiThreads) {
        const int t = e / V, c4 = (e - t * V) * 4;
        const float* src = wsd + size_t(t) * kDownCols + c4;
        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int qb = 0; qb < n; qb += 8) {
          // eight partials in flight, summed in contributor order
          float4 v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (qb + j < n) v[j] = __ldcg(reinterpret_cast<const float4*>(src + size_t(qb + j) * NT * kDownCols));
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (qb + j < n) {
              sum.x += v[j].x;
              sum.y += v[j].y;
              sum.z += v[j].z;
              sum.w += v[j].w;
            }
        }
        const int col = col0 + c4;
        float* yr = g.y + int64_t(t) * g.ldy + col;
        if (col + 3 < g.N) {
          *reinterpret_cast<float4*>(yr) = sum;
        } else {
          const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
          for (int j = 0; j < 4 && col + j < g.N; ++j) yr[j] = sv[j];
        }
      }
      if (first_fix && et == 0) SP_FSTAMP(10);
      first_fix = false;
    });
    if (et == 0) SP_FSTAMP(7);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

}  // namespace tc
}  // namespace sp
