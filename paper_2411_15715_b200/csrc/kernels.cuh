// kernels.cuh -- sm_100a kernels of the sliced FFN path.
//
// Every GPU-side product of the path is a "row dot": out[t, r] = epi(<W[r, :K], x[t, :K]>)
// with W stored row-major, rows padded to a multiple of 64 elements (zero
// padding), so each hidden column of the reference's W1 / W3 (slicing_kernel.py:
// 75-76, columns) and each output column of W2 restricted to a row block
// (slicing_kernel.py:77, rows) is one contiguous, 128-byte aligned row.  The same
// kernel serves
//   * the up-projection  a[t, h] = act(<W1t[h], x[t]>) [* <W3t[h], x[t]>]   (K = M)
//   * the down-projection y[t, n] (+)= <W2t[n, block], a[t, block]>          (K = |block|)
// for the GG block (weights resident in HBM) and for every streamed CG chunk
// (weights in the staging ring).  The activation of the reference
// (slicing_kernel.py:33-38) is fused into the up-projection epilogue.
//
// Decode GEMV design (HBM-bound, ~1 flop per weight byte):
//   * persistent grid: #SMs x resident CTAs, contiguous row ranges per CTA;
//   * x (the T activations) staged once per CTA in shared memory as fp32;
//   * 128-bit streaming loads (ld.global.nc.L1::no_allocate) of the weights;
//   * split-K across WPR warps of a CTA for long rows + warp-shuffle
//     reductions, a double-buffered smem combine across the WPR warps;
//   * fp32 accumulation throughout.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kRowGroup = 2;        // rows a warp works on together (ILP)
constexpr int kPadElems = 64;       // row padding of every packed matrix
constexpr int kMaxTileFloats = 16384;  // x tile: TT * KT floats <= 64 KB

enum Mode : int { kUp = 0, kUpGated = 1, kDown = 2 };

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

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 16 weight bytes -> fp32 lanes
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

__device__ __forceinline__ float act_fn(int act, float z) {
  if (act == 1) return z / (1.0f + expf(-z));                       // SiLU
  if (act == 2) return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));  // GELU (erf)
  return z;
}

__device__ __forceinline__ float bf16_to_f(uint16_t b) { return __uint_as_float(uint32_t(b) << 16); }

struct RowDotArgs {
  const void* w0;      // rows [0, rows) of length ldw elements
  const void* w1;      // second matrix (gated up-projection) or nullptr
  int64_t ldw;         // row stride (elements), multiple of kPadElems
  int rows;
  int K;               // valid reduction length <= ldw
  // activations: x_row(t) = src + (ids ? ids[t0 + t] : t0 + t) * ldx + xcol0
  const void* x;
  int xdtype;          // 0 f32, 1 bf16
  int64_t ldx;
  int64_t xcol0;
  const int32_t* ids;  // device, may be null
  int t0;              // first token (row of the call) this launch covers
  int T;               // tokens this launch covers (<= TT)
  // output: out[(t0 + t) * ldo + ocol0 + r]
  float* out;
  int64_t ldo;
  int64_t ocol0;
  int accumulate;      // kDown: add into out instead of overwrite
  int act;
  int kt;              // x tile length (multiple of 256, <= kMaxTileFloats / TT)
};

// Shared memory: xs[TT][kt] | red[2][kWarps][kRowGroup*G][TT] | acc[rows_per_cta][G][TT]
template <typename WT, int TT, int MODE, int WPR>
__global__ void __launch_bounds__(kThreads) rowdot_kernel(RowDotArgs p) {
  constexpr int VE = VecTraits<WT>::kElems;
  constexpr int G = (MODE == kUpGated) ? 2 : 1;
  constexpr int SUBROWS = kWarps / WPR;         // rows processed concurrently by the CTA
  constexpr int GROUP = SUBROWS * kRowGroup;    // rows per group step
  extern __shared__ __align__(16) float smem[];
  float* xs = smem;
  float* red = xs + TT * p.kt;
  float* acc = red + 2 * kWarps * kRowGroup * G * TT;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = warp / WPR, part = warp % WPR;
  const int64_t r_begin = (int64_t)p.rows * blockIdx.x / gridDim.x;
  const int64_t r_end = (int64_t)p.rows * (blockIdx.x + 1) / gridDim.x;
  const int n_local = int(r_end - r_begin);
  if (n_local <= 0) return;
  for (int i = threadIdx.x; i < n_local * G * TT; i += kThreads) acc[i] = 0.f;

  const char* wbase[G];
  wbase[0] = static_cast<const char*>(p.w0);
  if constexpr (G == 2) wbase[1] = static_cast<const char*>(p.w1);
  int red_buf = 0;

  for (int k0 = 0; k0 < p.K; k0 += p.kt) {
    const int kt_valid = min(p.kt, p.K - k0);
    __syncthreads();
    // ---- stage x[:, k0 : k0 + kt] as fp32 (zero beyond K and beyond T) ----
    for (int i = threadIdx.x; i < TT * p.kt; i += kThreads) {
      const int t = i / p.kt, k = i - t * p.kt;
      float v = 0.f;
      if (t < p.T && k < kt_valid) {
        const int64_t row = p.ids ? p.ids[p.t0 + t] : int64_t(p.t0 + t);
        const int64_t off = row * p.ldx + p.xcol0 + k0 + k;
        v = p.xdtype == 1 ? bf16_to_f(static_cast<const uint16_t*>(p.x)[off])
                          : static_cast<const float*>(p.x)[off];
      }
      xs[t * p.kt + xs_pos<WT>(k, p.kt)] = v;
    }
    __syncthreads();

    // this warp's k-slice of the tile, rounded to whole vectors
    const int per_part = ((kt_valid + WPR - 1) / WPR + VE - 1) / VE * VE;
    const int kb = part * per_part;
    const int ke = min(kt_valid, kb + per_part);

    for (int g0 = 0; g0 < n_local; g0 += GROUP) {
      float s[kRowGroup][G][TT];
#pragma unroll
      for (int j = 0; j < kRowGroup; ++j)
#pragma unroll
        for (int m = 0; m < G; ++m)
#pragma unroll
          for (int t = 0; t < TT; ++t) s[j][m][t] = 0.f;

      int64_t rows_j[kRowGroup];
      bool live[kRowGroup];
#pragma unroll
      for (int j = 0; j < kRowGroup; ++j) {
        const int lr = g0 + sub * kRowGroup + j;
        live[j] = lr < n_local;
        rows_j[j] = r_begin + (live[j] ? lr : 0);
      }

#pragma unroll 2
      for (int k = kb + lane * VE; k < ke; k += 32 * VE) {
        uint4 wv[kRowGroup][G];
#pragma unroll
        for (int j = 0; j < kRowGroup; ++j)
#pragma unroll
          for (int m = 0; m < G; ++m) {
            const char* ptr = wbase[m] + (rows_j[j] * p.ldw + k0 + k) * sizeof(WT);
            wv[j][m] = live[j] ? ld_stream(ptr) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          float xv[VE];
          const float* xrow = xs + t * p.kt;
          const int pos = xs_pos<WT>(k, p.kt);
          const float4 a = *reinterpret_cast<const float4*>(xrow + pos);
          xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
          if constexpr (VE == 8) {
            const float4 b = *reinterpret_cast<const float4*>(xrow + pos + (p.kt >> 1));
            xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
          }
#pragma unroll
          for (int j = 0; j < kRowGroup; ++j)
#pragma unroll
            for (int m = 0; m < G; ++m) {
              float wf[VE];
              unpack<WT>(wv[j][m], wf);
#pragma unroll
              for (int e = 0; e < VE; ++e) s[j][m][t] = fmaf(wf[e], xv[e], s[j][m][t]);
            }
        }
      }
      // warp reduction
#pragma unroll
      for (int j = 0; j < kRowGroup; ++j)
#pragma unroll
        for (int m = 0; m < G; ++m)
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            float v = s[j][m][t];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            s[j][m][t] = v;
          }
      if constexpr (WPR == 1) {
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < kRowGroup; ++j)
            if (live[j]) {
              const int lr = g0 + sub * kRowGroup + j;
#pragma unroll
              for (int m = 0; m < G; ++m)
#pragma unroll
                for (int t = 0; t < TT; ++t) acc[(lr * G + m) * TT + t] += s[j][m][t];
            }
        }
      } else {
        float* rb = red + red_buf * (kWarps * kRowGroup * G * TT);
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < kRowGroup; ++j)
#pragma unroll
            for (int m = 0; m < G; ++m)
#pragma unroll
              for (int t = 0; t < TT; ++t) rb[((warp * kRowGroup + j) * G + m) * TT + t] = s[j][m][t];
        }
        __syncthreads();
        // combine the WPR partial sums of every (row, matrix, token)
        for (int i = threadIdx.x; i < SUBROWS * kRowGroup * G * TT; i += kThreads) {
          const int t = i % TT, m = (i / TT) % G, j = (i / (TT * G)) % kRowGroup,
                    sr = i / (TT * G * kRowGroup);
          const int lr = g0 + sr * kRowGroup + j;
          if (lr < n_local) {
            float v = 0.f;
#pragma unroll
            for (int q = 0; q < WPR; ++q) v += rb[(((sr * WPR + q) * kRowGroup + j) * G + m) * TT + t];
            acc[(lr * G + m) * TT + t] += v;
          }
        }
        red_buf ^= 1;
      }
    }
  }
  __syncthreads();
  // ---- epilogue ----
  for (int i = threadIdx.x; i < n_local * TT; i += kThreads) {
    const int lr = i / TT, t = i - lr * TT;
    if (t >= p.T) continue;
    float* o = p.out + int64_t(p.t0 + t) * p.ldo + p.ocol0 + r_begin + lr;
    if constexpr (MODE == kDown) {
      const float v = acc[lr * TT + t];
      *o = p.accumulate ? *o + v : v;
    } else if constexpr (MODE == kUp) {
      *o = act_fn(p.act, acc[lr * TT + t]);
    } else {
      *o = act_fn(p.act, acc[(lr * 2 + 0) * TT + t]) * acc[(lr * 2 + 1) * TT + t];
    }
  }
}

// ---- merge: y[t] = sum_c sum_{i: ids_c[i]=t} gate_c[i] * (y_gpu_c[i] + y_cc_c[i]) -------
constexpr int kMaxMergeCalls = 32;
struct MergeCall {
  const float* y_gpu;    // [T_e, N]
  const float* y_cc;     // [T_e, N] or null; rows >= n_cc are absent
  const int32_t* ids;    // device [T_e] or null (identity)
  const float* gates;    // device [T_e] or null (1.0)
  int T_e;
  int n_cc;
};
struct MergeArgs {
  MergeCall c[kMaxMergeCalls];
  int n_calls;
  int T;
  int64_t N;
  float* acc;   // [T, N] fp32 scratch (also the output when odtype == f32)
  void* out;    // [T, N] in odtype
  int odtype;
};

__global__ void __launch_bounds__(256) merge_kernel(MergeArgs p) {
  for (int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; n < p.N;
       n += int64_t(gridDim.x) * blockDim.x) {
    for (int t = 0; t < p.T; ++t) p.acc[t * p.N + n] = 0.f;
    for (int c = 0; c < p.n_calls; ++c) {
      const MergeCall& mc = p.c[c];
      for (int i = 0; i < mc.T_e; ++i) {
        const int t = mc.ids ? mc.ids[i] : i;
        float v = mc.y_gpu[int64_t(i) * p.N + n];
        if (mc.y_cc && i < mc.n_cc) v += mc.y_cc[int64_t(i) * p.N + n];
        const float g = mc.gates ? mc.gates[i] : 1.0f;
        p.acc[t * p.N + n] += g * v;
      }
    }
    if (p.odtype == 1) {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out);
      for (int t = 0; t < p.T; ++t) o[t * p.N + n] = __float2bfloat16_rn(p.acc[t * p.N + n]);
    } else if (p.out != p.acc) {
      float* o = static_cast<float*>(p.out);
      for (int t = 0; t < p.T; ++t) o[t * p.N + n] = p.acc[t * p.N + n];
    }
  }
}

}  // namespace sp
