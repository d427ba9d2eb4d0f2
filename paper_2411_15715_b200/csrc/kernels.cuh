// kernels.cuh -- sm_100a kernels of the sliced FFN path.
//
// A "block" is a contiguous range of hidden units [h0, h0 + rows) of one FFN
// instance: the GG block (HBM resident) or one streamed CG chunk (in the HBM
// staging ring).  Its weights are packed as
//     W1t[rows, ldm] | W3t[rows, ldm] (gated only) | W2[rows, ldn]
// i.e. hidden unit h owns row h of each matrix: column h of the reference's
// W1 / W3 (slicing_kernel.py:75-76) and row h of its W2 (:77); rows are zero
// padded to a multiple of 64 elements (128-byte aligned).
//
// ffn_block_kernel computes, for every token t of the launch,
//     a[t, h]   = act(<W1t[h], x[t]>) [* <W3t[h], x[t]>]            (phase 1)
//     y_c[t, :] = sum_{h in CTA c's rows} a[t, h] * W2[h, :]          (phase 2)
// and writes y_c -- CTA c's partial of the block's output -- to its own slice
// of a partial buffer.  finalize_kernel sums the slices of every block of a
// call in a fixed order (deterministic), adds the CC partial, applies the MoE
// gates and casts.  The up/down dependency therefore never
// leaves the CTA: one launch per block, no grid-wide barrier, no `a` round trip.
//
// Decode is HBM-bound (~1 flop per weight byte).  Each CTA's rows are
// contiguous in memory, so one producer lane streams them with cp.async.bulk
// (TMA bulk-copy engine) through an NST-deep shared-memory ring with
// full/empty mbarriers; 8 consumer warps read weights only from shared memory:
//   phase 1: warp w owns k-slice w of every row (x slice staged once), warp
//            shuffles reduce each (row, matrix), partials parked in smem,
//            one named barrier combines the 8 slices + fused SiLU/GELU/gate;
//   phase 2: thread owns 8-element column vectors of W2 rows, FMAs a[t, h]
//            (smem broadcast) into fp32 registers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

constexpr int kPadElems = 64;          // row padding of every packed matrix
constexpr int kConsumers = 8;          // consumer warps per CTA
constexpr int kBlockThreads = (kConsumers + 1) * 32;
constexpr int kMaxStages = 8;
constexpr int kMaxVec = 4;             // W2 column vectors per thread (N <= 8192 bf16)

template <typename WT>
struct VecTraits;
template <>
struct VecTraits<float> {
  static constexpr int kElems = 4;
};
template <>
struct VecTraits<__nv_bfloat16> {
  static constexpr int kElems = 8;
};

// 16 weight bytes -> fp32
template <typename WT>
__device__ __forceinline__ void unpack(const uint4& u, float* f);
template <>
__device__ __forceinline__ void unpack<float>(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x);
  f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z);
  f[3] = __uint_as_float(u.w);
}
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xffff0000u);
}

// Shared-memory position of x element k inside one token's tile.  For bf16
// weights a lane consumes 8 consecutive k; storing them as two 4-float planes
// makes both float4 reads of a warp hit 32 distinct banks.
template <typename WT>
__device__ __forceinline__ int xs_pos(int k, int kt) {
  if constexpr (VecTraits<WT>::kElems == 8) {
    return ((k >> 2) & 1) * (kt >> 1) + ((k >> 3) << 2) + (k & 3);
  } else {
    return k;
  }
}

// The reference's activations (slicing_kernel.py:33-38) in fp32.
__device__ __forceinline__ float act_fn(int act, float z) {
  if (act == 1) return z / (1.0f + expf(-z));                                // SiLU
  if (act == 2) return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));  // GELU (erf)
  return z;
}

__device__ __forceinline__ float bf16_to_f(uint16_t b) { return __uint_as_float(uint32_t(b) << 16); }

// ---- mbarrier / bulk-copy primitives ---------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SP_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SP_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
}

// Warp-reduce C values per lane (C a power of two <= 32) with (C - 1) + (5 - log2 C)
// shuffles instead of 5 * C: every halving step swaps half of the values with
// the partner lane (offset 16, 8, ...), then a plain butterfly finishes.  After
// the call, value i's total is returned by every lane whose bits
// [5 - log2 C, 5) equal i.
template <int C>
__device__ __forceinline__ float warp_reduce_transposed(float* v, int lane) {
  int off = 16;
#pragma unroll
  for (int c = C; c > 1; c >>= 1, off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < c / 2; ++i) {
      const float send = upper ? v[i] : v[i + c / 2];
      const float keep = upper ? v[i + c / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  float r = v[0];
#pragma unroll
  for (; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
  return r;
}

struct FfnArgs {
  const void* w1t;     // [rows, ldm]
  const void* w3t;     // [rows, ldm] or null
  const void* w2;      // [rows, ldn]
  int64_t ldm, ldn;    // row strides (elements)
  int rows;            // hidden units in the block
  int M, N;
  // x row of token t: x + (ids ? ids[t0 + t] : t0 + t) * ldx
  const void* x;
  int xdtype;          // 0 f32, 1 bf16
  int64_t ldx;
  const int32_t* ids;  // device or null
  int t0, T;           // tokens [t0, t0 + T) of the call (T <= TT)
  int act;
  int kt;              // x tile: roundup(M, 256)
  int xvec;            // x rows 16-byte aligned and M a multiple of the 16-byte vector
  int tok[4];          // x rows of the launch's tokens (host-resolved ids), used when xvec
  // partial slices: part[(slice0 + cta) * slice_stride + (t0 + t) * N + n]
  float* part;
  int64_t slice0, slice_stride;
  unsigned long long* stamps;  // debug timing: [grid][8] %globaltimer stamps, or null
  unsigned long long* kspan0;  // trace: atomicMin of every CTA's start (%globaltimer ns), or null
  unsigned long long* kspan1;  // trace: atomicMax of every CTA's end
  int cta0, ncta;              // this block's CTAs inside a grouped launch
};

// Several blocks (e.g. the GG blocks of every active expert) in one launch:
// CTAs [a[c].cta0, a[c].cta0 + a[c].ncta) work on entry c.  One launch, one
// ramp and one tail per step instead of one per expert.
constexpr int kMaxGroup = 8;
struct FfnGroup {
  FfnArgs a[kMaxGroup];
  int n;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SP_STAMP(i)                                                            \
  do {                                                                         \
    if (p.stamps && threadIdx.x == 0) p.stamps[blockIdx.x * 8 + (i)] = global_ns(); \
  } while (0)

struct FfnPlan {
  int rs_up;        // hidden rows per phase-1 stage
  int rs_down;      // hidden rows per phase-2 stage
  int stages;       // ring depth NST
  int stage_bytes;  // bytes per ring slot
};

// smem: ring[NST][stage] | xs[TT][kt] | xraw[TT][M] (xvec) | part1[n_local][8][G][TT] |
//       a_loc[n_local][TT] | full[NST] | empty[NST] | xbar
template <typename WT, int TT, bool GATED, int NV>
__global__ void __launch_bounds__(kBlockThreads, 1) ffn_block_kernel(const __grid_constant__ FfnGroup grp,
                                                                     const FfnPlan fp) {
  int gi = 0;
  while (gi + 1 < grp.n && int(blockIdx.x) >= grp.a[gi + 1].cta0) ++gi;
  const FfnArgs& p = grp.a[gi];
  const int cta = int(blockIdx.x) - p.cta0;
  constexpr int VE = VecTraits<WT>::kElems;
  constexpr int G = GATED ? 2 : 1;
  constexpr int STEP = 32 * VE;
  // rows of a phase-1 stage reduced together (RSU * G * TT <= 32 values per lane)
  constexpr int RSU = (2 * G * TT <= 32) ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SP_STAMP(0);
  if (p.stamps && threadIdx.x == 0) {  // debug: the SM this CTA runs on
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.stamps[blockIdx.x * 8 + 7] = smid;
  }
  if (p.kspan0 && threadIdx.x == 0) atomicMin(p.kspan0, global_ns());
  const int64_t r_begin = (int64_t)p.rows * cta / p.ncta;
  const int64_t r_end = (int64_t)p.rows * (cta + 1) / p.ncta;
  const int n_local = int(r_end - r_begin);
  const int NST = fp.stages;
  const int n_up = (n_local + fp.rs_up - 1) / fp.rs_up;
  const int n_dn = (n_local + fp.rs_down - 1) / fp.rs_down;
  const int64_t row1 = p.ldm * int64_t(sizeof(WT)), row2 = p.ldn * int64_t(sizeof(WT));

  const int xel = p.xdtype == 1 ? 2 : 4;
  const int xraw_bytes = p.xvec ? (TT * p.M * xel + 15) / 16 * 16 : 0;
  unsigned char* ring = smem_raw;
  float* xs = reinterpret_cast<float*>(ring + size_t(NST) * fp.stage_bytes);
  unsigned char* xraw = reinterpret_cast<unsigned char*>(xs + TT * p.kt);
  float* part1 = reinterpret_cast<float*>(xraw + xraw_bytes);
  float* a_loc = part1 + n_local * kConsumers * G * TT;
  uint64_t* full = reinterpret_cast<uint64_t*>(a_loc + ((n_local * TT + 1) & ~1));
  uint64_t* empty = full + NST;
  uint64_t* xbar = empty + NST;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    mbar_init(xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  SP_STAMP(1);

  if (warp == kConsumers) {
    // ---------------- producer: one lane streams x, then the CTA's rows ----------------
    if (lane == 0 && p.xvec) {
      // x first: a load issued behind the weight stream would wait for ~NST stages per SM
      const uint32_t row_bytes_x = uint32_t(p.M * xel);
      mbar_expect_tx(xbar, row_bytes_x * p.T);
      for (int t = 0; t < p.T; ++t)
        bulk_g2s(xraw + size_t(t) * row_bytes_x,
                 static_cast<const char*>(p.x) + int64_t(p.tok[t]) * p.ldx * xel, row_bytes_x, xbar,
                 evict_first_policy());
    }
    if (lane == 0 && n_local > 0) {
      const uint64_t pol = evict_first_policy();
      const char* s1 = static_cast<const char*>(p.w1t) + r_begin * row1;
      const char* s3 = GATED ? static_cast<const char*>(p.w3t) + r_begin * row1 : nullptr;
      const char* s2 = static_cast<const char*>(p.w2) + r_begin * row2;
      for (int s = 0; s < n_up + n_dn; ++s) {
        const int slot = s % NST;
        if (s >= NST) mbar_wait(&empty[slot], ((s / NST) - 1) & 1);
        unsigned char* dst = ring + size_t(slot) * fp.stage_bytes;
        if (s < n_up) {
          const int rows_s = min(fp.rs_up, n_local - s * fp.rs_up);
          const uint32_t bytes = uint32_t(rows_s * row1);
          mbar_expect_tx(&full[slot], bytes * G);
          bulk_g2s(dst, s1 + int64_t(s) * fp.rs_up * row1, bytes, &full[slot], pol);
          if constexpr (GATED)
            bulk_g2s(dst + size_t(fp.rs_up) * row1, s3 + int64_t(s) * fp.rs_up * row1, bytes, &full[slot], pol);
        } else {
          const int d = s - n_up;
          const int rows_s = min(fp.rs_down, n_local - d * fp.rs_down);
          const uint32_t bytes = uint32_t(rows_s * row2);
          mbar_expect_tx(&full[slot], bytes);
          bulk_g2s(dst, s2 + int64_t(d) * fp.rs_down * row2, bytes, &full[slot], pol);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // x -> fp32 tile xs (zero beyond M and beyond T)
  if (p.xvec) {
    mbar_wait(xbar, 0);
    const int vx = p.xdtype == 1 ? 8 : 4;
    const int nvec = p.kt / vx;
    for (int i = threadIdx.x; i < TT * nvec; i += kConsumers * 32) {
      const int t = i / nvec, k = (i - t * nvec) * vx;
      float f[8];
      if (t < p.T && k < p.M) {
        const uint4 raw = *reinterpret_cast<const uint4*>(xraw + (size_t(t) * p.M + k) * xel);
        if (vx == 8) unpack<__nv_bfloat16>(raw, f); else unpack<float>(raw, f);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = 0.f;
      }
      float* xrow = xs + t * p.kt;
      for (int e = 0; e < vx; ++e) xrow[xs_pos<WT>(k + e, p.kt)] = f[e];
    }
  } else {
    for (int t = 0; t < TT; ++t) {
      const bool live_t = t < p.T;
      const int64_t row = live_t ? (p.ids ? p.ids[p.t0 + t] : int64_t(p.t0 + t)) : 0;
      const int64_t base = row * p.ldx;
      float* xrow = xs + t * p.kt;
      for (int k = threadIdx.x; k < p.kt; k += kConsumers * 32) {
        float v = 0.f;
        if (live_t && k < p.M)
          v = p.xdtype == 1 ? bf16_to_f(static_cast<const uint16_t*>(p.x)[base + k])
                            : static_cast<const float*>(p.x)[base + k];
        xrow[xs_pos<WT>(k, p.kt)] = v;
      }
    }
  }
  consumers_sync();
  SP_STAMP(2);

  // ---- phase 1: a[t, h] for the CTA's rows ----
  // vectors [k, k + VE) with k < M stay inside the zero-padded row and meet zero x beyond M
  const int steps_total = (p.M + STEP - 1) / STEP;
  const int per = (steps_total + kConsumers - 1) / kConsumers;
  const int kb = warp * per * STEP;
  const int ke = min((p.M + VE - 1) / VE * VE, kb + per * STEP);
  for (int s = 0; s < n_up; ++s) {
    const int slot = s % NST;
    mbar_wait(&full[slot], (s / NST) & 1);
    const int rows_s = min(fp.rs_up, n_local - s * fp.rs_up);
    const unsigned char* st = ring + size_t(slot) * fp.stage_bytes;
    // the stage's rows together: RSU x G x TT independent accumulators, updated
    // in pairs (W1 / W3 of a row, or two rows) by packed FFMA2 with x broadcast:
    // each lane of an FFMA2 is the same fma.rn as a scalar FFMA, so every
    // accumulator sees the identical sequence -- half the FMA instructions
    constexpr int NP = RSU * G / 2;  // accumulator pairs per token (RSU * G is even)
    static_assert(RSU * G % 2 == 0, "phase-1 accumulators are updated in pairs");
    for (int j0 = 0; j0 < rows_s; j0 += RSU) {
      float2 accp[NP][TT];
#pragma unroll
      for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int t = 0; t < TT; ++t) accp[q][t] = make_float2(0.f, 0.f);
      const bool live1 = RSU > 1 && j0 + 1 < rows_s;
#pragma unroll 2
      for (int k = kb + lane * VE; k < ke; k += STEP) {
        uint4 wv[RSU][G];
#pragma unroll
        for (int j = 0; j < RSU; ++j)
#pragma unroll
          for (int m = 0; m < G; ++m)
            wv[j][m] = (j == 0 || live1)
                           ? *reinterpret_cast<const uint4*>(st + (size_t(m) * fp.rs_up + j0 + j) * row1 +
                                                             size_t(k) * sizeof(WT))
                           : make_uint4(0, 0, 0, 0);
        float wf[RSU * G][VE];  // index j * G + m
#pragma unroll
        for (int j = 0; j < RSU; ++j)
#pragma unroll
          for (int m = 0; m < G; ++m) unpack<WT>(wv[j][m], wf[j * G + m]);
        const int pos = xs_pos<WT>(k, p.kt);
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          float xv[VE];
          const float* xrow = xs + t * p.kt;
          const float4 a = *reinterpret_cast<const float4*>(xrow + pos);
          xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
          if constexpr (VE == 8) {
            const float4 b = *reinterpret_cast<const float4*>(xrow + pos + (p.kt >> 1));
            xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
          }
#pragma unroll
          for (int q = 0; q < NP; ++q)
#pragma unroll
            for (int e = 0; e < VE; ++e)
              accp[q][t] = __ffma2_rn(make_float2(xv[e], xv[e]), make_float2(wf[2 * q][e], wf[2 * q + 1][e]),
                                      accp[q][t]);
        }
      }
      float acc[RSU * G * TT];  // (j * G + m) * TT + t
#pragma unroll
      for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          acc[(2 * q) * TT + t] = accp[q][t].x;
          acc[(2 * q + 1) * TT + t] = accp[q][t].y;
        }
      constexpr int CNT = RSU * G * TT;
      constexpr int LOGC = CNT == 1 ? 0 : CNT == 2 ? 1 : CNT == 4 ? 2 : CNT == 8 ? 3 : CNT == 16 ? 4 : 5;
      const float r = warp_reduce_transposed<CNT>(acc, lane);
      constexpr int SHIFT = 5 - LOGC;
      if ((lane & ((1 << SHIFT) - 1)) == 0) {
        const int idx = lane >> SHIFT;  // (j * G + m) * TT + t
        const int t = idx % TT, m = (idx / TT) % G, j = idx / (TT * G);
        if (j == 0 || live1)
          part1[(((s * fp.rs_up + j0 + j) * kConsumers + warp) * G + m) * TT + t] = r;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  consumers_sync();
  SP_STAMP(3);
  for (int i = threadIdx.x; i < n_local * TT; i += kConsumers * 32) {
    const int lr = i / TT, t = i - lr * TT;
    float v[G];
#pragma unroll
    for (int m = 0; m < G; ++m) {
      v[m] = 0.f;
#pragma unroll
      for (int q = 0; q < kConsumers; ++q) v[m] += part1[((lr * kConsumers + q) * G + m) * TT + t];
    }
    float a = act_fn(p.act, v[0]);
    if constexpr (GATED) a *= v[1];
    a_loc[lr * TT + t] = t < p.T ? a : 0.f;
  }
  consumers_sync();
  SP_STAMP(4);

  // ---- phase 2: y_c[t, :] = sum_h a[t, h] * W2[h, :] ----
  const int tid = threadIdx.x;
  const int n_vec = (p.N + VE - 1) / VE;
  // column pairs (e, e + 1) updated by packed FFMA2 with a[t, h] broadcast (per
  // accumulator the same fma sequence as scalar FFMAs)
  float2 acc2[NV][VE / 2][TT];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VE / 2; ++e)
#pragma unroll
      for (int t = 0; t < TT; ++t) acc2[v][e][t] = make_float2(0.f, 0.f);
  for (int d = 0; d < n_dn; ++d) {
    const int s = n_up + d;
    const int slot = s % NST;
    mbar_wait(&full[slot], (s / NST) & 1);
    const int rows_s = min(fp.rs_down, n_local - d * fp.rs_down);
    const unsigned char* st = ring + size_t(slot) * fp.stage_bytes;
    for (int j = 0; j < rows_s; ++j) {
      const int lr = d * fp.rs_down + j;
      float at[TT];
#pragma unroll
      for (int t = 0; t < TT; ++t) at[t] = a_loc[lr * TT + t];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int vec = tid + v * kConsumers * 32;
        if (vec < n_vec) {
          const uint4 w = *reinterpret_cast<const uint4*>(st + size_t(j) * row2 + size_t(vec) * 16);
          float wf[VE];
          unpack<WT>(w, wf);
#pragma unroll
          for (int e = 0; e < VE / 2; ++e)
#pragma unroll
            for (int t = 0; t < TT; ++t)
              acc2[v][e][t] = __ffma2_rn(make_float2(at[t], at[t]), make_float2(wf[2 * e], wf[2 * e + 1]),
                                         acc2[v][e][t]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  SP_STAMP(5);
  // write this CTA's partial slice (a CTA with no rows writes zeros)
  float* out = p.part + (p.slice0 + cta) * p.slice_stride;
#pragma unroll
  for (int t = 0; t < TT; ++t) {
    if (t >= p.T) break;
    float* orow = out + int64_t(p.t0 + t) * p.N;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int vec = tid + v * kConsumers * 32;
      if (vec >= n_vec) continue;
      const int n0 = vec * VE;
      if (n0 + VE <= p.N && (p.N & 3) == 0) {
#pragma unroll
        for (int e = 0; e < VE; e += 4)
          *reinterpret_cast<float4*>(orow + n0 + e) =
              make_float4(acc2[v][e / 2][t].x, acc2[v][e / 2][t].y, acc2[v][e / 2 + 1][t].x, acc2[v][e / 2 + 1][t].y);
      } else {
#pragma unroll
        for (int e = 0; e < VE; ++e)
          if (n0 + e < p.N) orow[n0 + e] = (e & 1) ? acc2[v][e / 2][t].y : acc2[v][e / 2][t].x;
      }
    }
  }
  SP_STAMP(6);
  if (p.kspan1) {
    consumers_sync();
    if (threadIdx.x == 0) atomicMax(p.kspan1, global_ns());
  }
}

// ---- finalize: slice reduction + CC partial + MoE gates + cast, one launch -------------
//   y[t, n] = sum over entries (c, i, gate) of token t (host-built CSR, in call order)
//             of gate * (sum_s part_c[s, i, n] + y_cc_c[i, n])
// Block = (32 output columns as 8 float4 lanes) x 32 slice groups, one output
// token per blockIdx.y: N/32 blocks per token, so a decode step's few hundred
// partial slices are read by ~128 CTAs instead of 32.  Every sum runs in a
// fixed order -> deterministic.
constexpr int kMaxCalls = 32;
constexpr int kFinLanes = 8;    // float4 column lanes per block
constexpr int kFinGroups = 32;  // slice groups per block
struct FinalCall {
  const float* part;     // [S][T_e][N] partial slices
  int S;
  const float* y_cc;     // [T_e, N] or null; rows >= n_cc are absent
  int n_cc;
  int T_e;
};
struct FinalArgs {
  FinalCall c[kMaxCalls];
  const int* entry_start;  // device [T + 1]
  const int* entry_call;   // device [entries]
  const int* entry_row;    // device [entries]
  const float* entry_gate; // device [entries]
  int T;
  int N;
  void* out;    // [T, N] in odtype
  int odtype;
};

__global__ void __launch_bounds__(kFinLanes * kFinGroups) finalize_kernel(FinalArgs p) {
  __shared__ float4 red[kFinGroups][kFinLanes];
  const int lane = threadIdx.x % kFinLanes, grp = threadIdx.x / kFinLanes;
  const int n = (blockIdx.x * kFinLanes + lane) * 4;
  const int t = blockIdx.y;
  const bool live = n < p.N;  // N % 4 == 0 on this path
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int e = p.entry_start[t]; e < p.entry_start[t + 1]; ++e) {
    const FinalCall& fc = p.c[p.entry_call[e]];
    const int i = p.entry_row[e];
    float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
    if (live) {
      const int64_t stride = int64_t(fc.T_e) * p.N;
      const float* base = fc.part + int64_t(i) * p.N + n;
      int s = grp;
      for (; s + kFinGroups < fc.S; s += 2 * kFinGroups) {
        const float4 a = __ldcg(reinterpret_cast<const float4*>(base + int64_t(s) * stride));
        const float4 b = __ldcg(reinterpret_cast<const float4*>(base + int64_t(s + kFinGroups) * stride));
        v0.x += a.x; v0.y += a.y; v0.z += a.z; v0.w += a.w;
        v1.x += b.x; v1.y += b.y; v1.z += b.z; v1.w += b.w;
      }
      for (; s < fc.S; s += kFinGroups) {
        const float4 a = __ldcg(reinterpret_cast<const float4*>(base + int64_t(s) * stride));
        v0.x += a.x; v0.y += a.y; v0.z += a.z; v0.w += a.w;
      }
    }
    red[grp][lane] = make_float4(v0.x + v1.x, v0.y + v1.y, v0.z + v1.z, v0.w + v1.w);
    __syncthreads();
    if (grp == 0 && live) {
      float4 tot = red[0][lane];
#pragma unroll 8
      for (int g = 1; g < kFinGroups; ++g) {
        const float4 r = red[g][lane];
        tot.x += r.x; tot.y += r.y; tot.z += r.z; tot.w += r.w;
      }
      if (fc.y_cc && i < fc.n_cc) {
        const float4 c = *reinterpret_cast<const float4*>(fc.y_cc + int64_t(i) * p.N + n);
        tot.x += c.x; tot.y += c.y; tot.z += c.z; tot.w += c.w;
      }
      const float gate = p.entry_gate[e];
      acc.x += gate * tot.x; acc.y += gate * tot.y; acc.z += gate * tot.z; acc.w += gate * tot.w;
    }
    __syncthreads();
  }
  if (grp == 0 && live) {
    if (p.odtype == 1) {
      __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(p.out) + int64_t(t) * p.N + n);
      o[0] = __floats2bfloat162_rn(acc.x, acc.y);
      o[1] = __floats2bfloat162_rn(acc.z, acc.w);
    } else {
      *reinterpret_cast<float4*>(static_cast<float*>(p.out) + int64_t(t) * p.N + n) = acc;
    }
  }
}

// Same contract for many tokens with few slices (prefill: a handful of split-K
// slices per call, hundreds of tokens): one thread per 4 output columns of one
// token, the slices summed sequentially in slice order -- every thread busy and
// every load a coalesced float4 (the slice-group layout above would leave 31 of
// its 32 groups idle).
// Sum each call's S partial slices into its slice 0 (grid.y = call).  Enqueued
// on the device stream right after a call's last GPU block, so the many-slice
// reduction of a decode step (one slice per GG-group CTA, per CG chunk CTA)
// runs while the host CC block is still busy; the finalize that waits for the
// CC partial then reads one slice per call.  Slices summed in kFinGroups
// strided groups, groups in order: deterministic.
__global__ void __launch_bounds__(kFinLanes * kFinGroups) reduce_slices_kernel(FinalArgs p) {
  __shared__ float4 red[kFinGroups][kFinLanes];
  const FinalCall& fc = p.c[blockIdx.y];
  const int64_t count = int64_t(fc.T_e) * p.N;  // floats per slice
  if (fc.S <= 1 || int64_t(blockIdx.x) * kFinLanes * 4 >= count) return;
  const int lane = threadIdx.x % kFinLanes, grp = threadIdx.x / kFinLanes;
  const int64_t col = (int64_t(blockIdx.x) * kFinLanes + lane) * 4;
  const bool live = col < count;  // N % 4 == 0 on this path
  float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
  if (live) {
    int s = grp;
    for (; s + kFinGroups < fc.S; s += 2 * kFinGroups) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(fc.part + int64_t(s) * count + col));
      const float4 b = __ldcg(reinterpret_cast<const float4*>(fc.part + int64_t(s + kFinGroups) * count + col));
      v0.x += a.x; v0.y += a.y; v0.z += a.z; v0.w += a.w;
      v1.x += b.x; v1.y += b.y; v1.z += b.z; v1.w += b.w;
    }
    for (; s < fc.S; s += kFinGroups) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(fc.part + int64_t(s) * count + col));
      v0.x += a.x; v0.y += a.y; v0.z += a.z; v0.w += a.w;
    }
  }
  red[grp][lane] = make_float4(v0.x + v1.x, v0.y + v1.y, v0.z + v1.z, v0.w + v1.w);
  __syncthreads();
  if (grp == 0 && live) {
    float4 tot = red[0][lane];
#pragma unroll 8
    for (int g = 1; g < kFinGroups; ++g) {
      const float4 r = red[g][lane];
      tot.x += r.x; tot.y += r.y; tot.z += r.z; tot.w += r.w;
    }
    *reinterpret_cast<float4*>(const_cast<float*>(fc.part) + col) = tot;  // the workspace is writable
  }
}

constexpr int kFinRowsThreads = 128;
__global__ void __launch_bounds__(kFinRowsThreads) finalize_rows_kernel(FinalArgs p) {
  const int t = blockIdx.y;
  const int n = (blockIdx.x * kFinRowsThreads + threadIdx.x) * 4;
  if (n >= p.N) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int e0 = p.entry_start[t], e1 = p.entry_start[t + 1];
  // the CC partials may sit in mapped host memory (a PCIe round trip each):
  // issue the first few entries' loads together, before any slice is summed
  constexpr int kPre = 4;
  float4 cpre[kPre];
#pragma unroll
  for (int q = 0; q < kPre; ++q) {
    cpre[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e0 + q < e1) {
      const FinalCall& fc = p.c[p.entry_call[e0 + q]];
      const int i = p.entry_row[e0 + q];
      if (fc.y_cc && i < fc.n_cc) cpre[q] = *reinterpret_cast<const float4*>(fc.y_cc + int64_t(i) * p.N + n);
    }
  }
  for (int e = e0; e < e1; ++e) {
    const FinalCall& fc = p.c[p.entry_call[e]];
    const int i = p.entry_row[e];
    const int64_t stride = int64_t(fc.T_e) * p.N;
    const float* base = fc.part + int64_t(i) * p.N + n;
    const bool cc = fc.y_cc && i < fc.n_cc;
    float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e - e0 < kPre) {
#pragma unroll
      for (int q = 0; q < kPre; ++q)
        if (q == e - e0) c = cpre[q];
    } else if (cc) {
      c = *reinterpret_cast<const float4*>(fc.y_cc + int64_t(i) * p.N + n);
    }
    float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
    // 8 slice loads in flight per thread, summed in slice order
    int s = 0;
    for (; s + 8 <= fc.S; s += 8) {
      float4 a[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = __ldcg(reinterpret_cast<const float4*>(base + int64_t(s + j) * stride));
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        tot.x += a[j].x; tot.y += a[j].y; tot.z += a[j].z; tot.w += a[j].w;
      }
    }
    for (; s < fc.S; ++s) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(base + int64_t(s) * stride));
      tot.x += a.x; tot.y += a.y; tot.z += a.z; tot.w += a.w;
    }
    if (cc) {
      tot.x += c.x; tot.y += c.y; tot.z += c.z; tot.w += c.w;
    }
    const float gate = p.entry_gate[e];
    acc.x += gate * tot.x; acc.y += gate * tot.y; acc.z += gate * tot.z; acc.w += gate * tot.w;
  }
  if (p.odtype == 1) {
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(p.out) + int64_t(t) * p.N + n);
    o[0] = __floats2bfloat162_rn(acc.x, acc.y);
    o[1] = __floats2bfloat162_rn(acc.z, acc.w);
  } else {
    *reinterpret_cast<float4*>(static_cast<float*>(p.out) + int64_t(t) * p.N + n) = acc;
  }
}

// Same contract for N % 4 != 0 (small test shapes): one thread per output element.
__global__ void __launch_bounds__(256) finalize_scalar_kernel(FinalArgs p) {
  const int t = blockIdx.y;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < p.N; n += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int e = p.entry_start[t]; e < p.entry_start[t + 1]; ++e) {
      const FinalCall& fc = p.c[p.entry_call[e]];
      const int i = p.entry_row[e];
      float tot = 0.f;
      for (int s = 0; s < fc.S; ++s) tot += fc.part[(int64_t(s) * fc.T_e + i) * p.N + n];
      if (fc.y_cc && i < fc.n_cc) tot += fc.y_cc[int64_t(i) * p.N + n];
      acc += p.entry_gate[e] * tot;
    }
    if (p.odtype == 1)
      static_cast<__nv_bfloat16*>(p.out)[int64_t(t) * p.N + n] = __float2bfloat16_rn(acc);
    else
      static_cast<float*>(p.out)[int64_t(t) * p.N + n] = acc;
  }
}

}  // namespace sp
