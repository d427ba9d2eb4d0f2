// gemm_tc.cuh -- tcgen05 / TMEM / TMA GEMM for the prefill (many-token) path, sm_100a.
//
// Prefill is a real contraction: T tokens against every weight row, ~2*T
// flop per weight byte.  Per block of hidden units (GG block or streamed chunk)
// the path runs two GEMMs on the 5th-gen tensor cores:
//   up   : a[T, R]  = act(x[T, M] . W1t[R, M]^T) * (x . W3t^T)     (SwiGLU epilogue, bf16 out)
//   down : y[T, N] += a[T, R] . W2[R, N]                            (fp32 accumulate)
// D[BM x BN] = A[BM x K] . B[BN x K]^T with A = tokens (UMMA M = 128), B = the
// weights (K-major W1t/W3t rows for up, MN-major W2 rows for down), bf16
// operands, fp32 accumulators in TMEM.
//
// Warp roles (192 threads, one CTA per output tile):
//   warp 0      TMA producer: one lane issues cp.async.bulk.tensor 2D loads
//               (128B swizzle) of A and B k-blocks into an S-deep smem ring
//   warp 1      TMEM allocator + MMA issuer: one lane issues tcgen05.mma
//               (kind::f16, cta_group::1, M=128, N=BN, K=16) and commits each
//               stage back to the producer through an mbarrier
//   warps 2..5  epilogue: tcgen05.ld 32x32b rows of the accumulator(s), fused
//               activation / gate / accumulate, stores
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace sp {
namespace tc {

constexpr int BM = 128;  // tokens per tile (UMMA M)
constexpr int BK = 64;   // k per stage: one 128-byte swizzle atom of bf16
constexpr int UK = 16;   // UMMA K for 16-bit inputs
constexpr int kThreads = 192;

enum Mode : int { kUpGated = 0, kUpPlain = 1, kDownAcc = 2 };

struct GemmArgs {
  int m_valid;      // valid token rows
  int n_valid;      // valid B rows (hidden units for up, output columns for down)
  int k;            // contraction length
  int mode;
  int act;
  // up epilogue: a_out[(m0 + r) * lda + a_col0 + n]  (bf16)
  __nv_bfloat16* a_out;
  int64_t lda;
  int64_t a_col0;
  // down epilogue: y[(m0 + r) * ldy + n] (+)= acc  (fp32)
  float* y;
  int64_t ldy;
  int accumulate;
  int stages;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor, 128-byte swizzle, Blackwell version bits.
__device__ __forceinline__ uint64_t umma_desc(const void* smem, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((smem_u32(smem) & 0x3FFFF) >> 4);          // start address   [0, 14)
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;           // leading offset  [16, 30)
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;           // stride offset   [32, 46)
  d |= uint64_t(1) << 46;                                   // version = 1 (sm100)
  d |= uint64_t(2) << 61;                                   // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, A K-major.
__host__ __device__ constexpr uint32_t umma_idesc(int m, int n, bool b_mn_major) {
  return (1u << 4)                          // D format f32
         | (1u << 7)                        // A format bf16
         | (1u << 10)                       // B format bf16
         | (uint32_t(b_mn_major) << 16)     // B major
         | (uint32_t(n >> 3) << 17)         // N / 8
         | (uint32_t(m >> 4) << 24);        // M / 16
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN, int NB>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                const __grid_constant__ CUtensorMap tmB1, GemmArgs g) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE = A_BYTES + NB * B_BYTES;
  constexpr int TMEM_COLS = (NB * BN) <= 32 ? 32 : (NB * BN) <= 64 ? 64 : (NB * BN) <= 128 ? 128 : (NB * BN) <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzled tiles
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * STAGE);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int nkb = (g.k + BK - 1) / BK;
  const bool b_mn = g.mode == kDownAcc;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB0)) : "memory");
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

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        unsigned char* st = smem + size_t(s) * STAGE;
        mbar_expect_tx(&full[s], STAGE);
        tma_load_2d(st, &tmA, &full[s], kb * BK, m0);
        if (!b_mn) {
          tma_load_2d(st + A_BYTES, &tmB0, &full[s], kb * BK, n0);
          if constexpr (NB == 2) tma_load_2d(st + A_BYTES + B_BYTES, &tmB1, &full[s], kb * BK, n0);
        } else {
          // MN-major B: boxes of 64 columns x BK rows, one per 64-column group
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(st + A_BYTES + j * (BK * 128), &tmB0, &full[s], n0 + j * 64, kb * BK);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = umma_idesc(BM, BN, b_mn);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const unsigned char* st = smem + size_t(s) * STAGE;
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          const uint64_t a = umma_desc(st + kk * 32, 16, 1024);
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const unsigned char* bt = st + A_BYTES + b * B_BYTES;
            const uint64_t bd = b_mn ? umma_desc(bt + kk * UK * 128, BK * 128, 1024)  // k rows of 128 B
                                     : umma_desc(bt + kk * 32, 16, 1024);
            umma_bf16(tmem + uint32_t(b * BN), a, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
        }
        umma_commit(&empty[s]);
        if (kb == nkb - 1) umma_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: warps 2..5 cover TMEM lanes 32*(warp%4) ----------------
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int m = m0 + row;
    const uint32_t lane_addr = tmem + (uint32_t(quarter * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r0[16], r1[16];
      tmem_ld16(lane_addr + uint32_t(c), r0);
      if constexpr (NB == 2) tmem_ld16(lane_addr + uint32_t(BN + c), r1);
      if (m >= g.m_valid) continue;
      if (g.mode == kDownAcc) {
        float* yr = g.y + int64_t(m) * g.ldy + n0 + c;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          if (n0 + c + e < g.n_valid) {
            const float v = __uint_as_float(r0[e]);
            yr[e] = g.accumulate ? yr[e] + v : v;
          }
        }
      } else {
        __nv_bfloat16* ar = g.a_out + int64_t(m) * g.lda + g.a_col0 + n0 + c;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          if (n0 + c + e < g.n_valid) {
            float v = act_fn(g.act, __uint_as_float(r0[e]));
            if constexpr (NB == 2) v *= __uint_as_float(r1[e]);
            ar[e] = __float2bfloat16_rn(v);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

// gather x rows (any dtype) into a contiguous bf16 [T_pad, ldx] buffer
__global__ void gather_rows_bf16_kernel(const void* x, int xdtype, int64_t ldx_in, const int32_t* ids, int t0,
                                        int T, int M, __nv_bfloat16* out, int64_t ldo) {
  const int t = blockIdx.y;
  if (t >= T) return;
  const int64_t row = ids ? ids[t0 + t] : int64_t(t0 + t);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < M; k += gridDim.x * blockDim.x) {
    const float v = xdtype == 1 ? bf16_to_f(static_cast<const uint16_t*>(x)[row * ldx_in + k])
                                : static_cast<const float*>(x)[row * ldx_in + k];
    out[int64_t(t) * ldo + k] = __float2bfloat16_rn(v);
  }
}

}  // namespace tc
}  // namespace sp
