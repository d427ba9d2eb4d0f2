// gemm_tc.cuh -- tcgen05 / TMEM / TMA GEMMs for the prefill (many-token) path, sm_100a.
//
// Prefill is a real contraction: T tokens against every weight row.  Per block
// of hidden units (GG block or streamed chunk) the path runs two GEMMs on the
// 5th-gen tensor cores, with the WEIGHTS as the 128-row UMMA M operand and the
// tokens as N (<= 256), so each weight byte is streamed once per token tile:
//   up   : D[h, t] = W1t[h, :] . x[t, :]  (and W3t)  -> a[t, h] = act(D1) * D3   (bf16)
//   down : D[n, t] = W2[:, n] . a[t, :]               -> y[t, n] += D             (fp32)
// A operands: W1t / W3t rows are K-major; W2 ([h, n], n contiguous) is MN-major.
// B operands (x, a: [t, k] row-major) are K-major.  bf16 in, fp32 accumulate in TMEM.
//
// Parallelism: a block has few 128-row tiles (56 for 7168 hidden units, 32
// output-column tiles for N = 4096), so K is split over KS CTAs to put ~one CTA
// on every SM.  Each split writes an fp32 partial tile; the LAST CTA of a tile
// (atomic ticket) sums the KS partials in split order -- deterministic -- and
// runs the epilogue (SwiGLU + bf16 store for up, accumulate into the call's
// output slice for down), then re-arms the ticket.
//
// Warp roles (192 threads):
//   warp 0      TMA producer: one lane issues cp.async.bulk.tensor 2D loads
//               (128B swizzle) into an S-deep smem ring
//   warp 1      TMEM allocator + MMA issuer: one lane issues tcgen05.mma
//               (kind::f16, cta_group::1, M = 128, N = NT, K = 16), commits
//               stages back to the producer through mbarriers
//   warps 2..5  epilogue: tcgen05.ld 32x32b (TMEM lane = weight row), fused
//               epilogue or partial write + split fix-up
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace sp {
namespace tc {

constexpr int BM = 128;  // weight rows per tile (UMMA M)
constexpr int BK = 64;   // k per stage: one 128-byte swizzle atom of bf16
constexpr int UK = 16;   // UMMA K for 16-bit inputs
constexpr int kThreads = 192;

enum Mode : int { kUpGated = 0, kUpPlain = 1, kDown = 2 };

struct GemmArgs {
  int mode;
  int act;
  int rows;         // weight rows (hidden units for up, output columns N for down)
  int T;            // valid tokens
  int k;            // contraction length
  int m_tiles, t_tiles, ks;
  int stages;
  // up epilogue: a[t * lda + h]  (bf16)
  __nv_bfloat16* a_out;
  int64_t lda;
  // down epilogue: y[t * ldy + n] += acc  (fp32, the call's tensor-core slice), or with
  // split_slices: split q STORES its partial into y + q * y_split_stride (one output
  // slice per split; finalize_kernel sums the slices in order -- no fix-up pass)
  float* y;
  int64_t ldy;
  int split_slices;
  int64_t y_split_stride;
  // up with ks > 1: split q stores fp32 pre-activations z[q][a][t][h] (ld = zld) and
  // swiglu_reduce_kernel finishes (sum in split order, act, gate, bf16)
  float* z;
  int64_t zld;
  // split-K partials [tile][ks][NA][128][NT] fp32 and tickets [tile]
  float* partial;
  int* tickets;
  int dbg_no_mma;  // probe: stream the operands but issue no MMA (SP_TC_DBG_NOMMA)
  // trace: atomicMin of every CTA's start / atomicMax of every CTA's end
  // (%globaltimer ns) over the block's chain, or null
  unsigned long long* kspan0;
  unsigned long long* kspan1;
};

// Programmatic dependent launch (PDL).  The prefill chain gather -> up GEMM ->
// (swiglu_reduce) -> down GEMM is launched with programmatic stream
// serialization: each kernel lets its successor launch early and the successor
// streams the operands that do not depend on its predecessor (the weights)
// before it waits.  Launched without the attribute, both are no-ops.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


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

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, B K-major.
__host__ __device__ constexpr uint32_t umma_idesc(int m, int n, bool a_mn_major) {
  return (1u << 4)                          // D format f32
         | (1u << 7)                        // A format bf16
         | (1u << 10)                       // B format bf16
         | (uint32_t(a_mn_major) << 15)     // A major
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

__device__ __forceinline__ void epilogue_sync() {
  asm volatile("bar.sync 2, 128;" ::: "memory");
}

// NT: tokens per tile (UMMA N, multiple of 16, <= 256).  NA A-tiles share one B tile,
// each with its own TMEM accumulator: up -> W1t and W3t rows of the same 128
// hidden units (NA = 2 gated); down -> NA consecutive 128-column sub-tiles of W2
// (one fetch of `a` per k-block feeds NA MMAs; W2 rows are read NA*256 bytes at a time).
template <int NT, int NA, bool DOWN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                const __grid_constant__ CUtensorMap tmB, const GemmArgs g) {
  constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  constexpr int B_BYTES = NT * BK * 2;
  constexpr int STAGE = NA * A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = (NA * NT) <= 32 ? 32 : (NA * NT) <= 64 ? 64 : (NA * NT) <= 128 ? 128
                            : (NA * NT) <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * STAGE);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (g.kspan0 && threadIdx.x == 0) atomicMin(g.kspan0, global_ns());
  // blockIdx -> (token tile, row tile, split)
  const int ks_id = blockIdx.x % g.ks;
  const int tile = blockIdx.x / g.ks;  // = mt * t_tiles + tt
  // a row tile's token tiles run on adjacent CTAs: the second reads the weight
  // tile from L2 while the first streams it from HBM (T = 512: 254 -> 248 us)
  const int mt = tile / g.t_tiles, tt = tile % g.t_tiles;
  const int m0 = mt * BM * (DOWN ? NA : 1), t0 = tt * NT;
  const int nkb = (g.k + BK - 1) / BK;
  const int kb0 = nkb * ks_id / g.ks, kb1 = nkb * (ks_id + 1) / g.ks;
  constexpr bool a_mn = DOWN;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
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

  const int nk = kb1 - kb0;
  grid_dep_launch();  // the successor may start its weight stream on the SMs this grid leaves idle
  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      auto load_a = [&](int i) {
        const int kb = kb0 + i, s = i % S;
        unsigned char* st = smem + size_t(s) * STAGE;
        if constexpr (!DOWN) {
          tma_load_2d(st, &tmA0, &full[s], kb * BK, m0);
          if constexpr (NA == 2) tma_load_2d(st + A_BYTES, &tmA1, &full[s], kb * BK, m0);
        } else {
          // MN-major A (W2 [k rows][n]): per sub-tile two 64-column boxes of BK rows
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            tma_load_2d(st + a * A_BYTES, &tmA0, &full[s], m0 + a * BM, kb * BK);
            tma_load_2d(st + a * A_BYTES + BK * 128, &tmA0, &full[s], m0 + a * BM + 64, kb * BK);
          }
        }
      };
      auto load_b = [&](int i) {
        const int kb = kb0 + i, s = i % S;
        tma_load_2d(smem + size_t(s) * STAGE + NA * A_BYTES, &tmB, &full[s], kb * BK, t0);
      };
      // the first S stages' weights do not depend on the predecessor kernel:
      // issue them before waiting for it, then the dependent x / a tiles
      const int pre = nk < S ? nk : S;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], STAGE);
        load_a(i);
      }
      grid_dep_wait();
      for (int i = 0; i < pre; ++i) load_b(i);
      for (int i = pre; i < nk; ++i) {
        const int s = i % S;
        mbar_wait(&empty[s], ((i / S) - 1) & 1);
        mbar_expect_tx(&full[s], STAGE);
        load_a(i);
        load_b(i);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = umma_idesc(BM, NT, a_mn);
    for (int i = 0; i < nk; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const unsigned char* st = smem + size_t(s) * STAGE;
        if (!g.dbg_no_mma) {
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t b = umma_desc(st + NA * A_BYTES + kk * 32, 16, 1024);
#pragma unroll
            for (int a = 0; a < NA; ++a) {
              const uint64_t ad = a_mn ? umma_desc(st + a * A_BYTES + kk * UK * 128, BK * 128, 1024)
                                       : umma_desc(st + a * A_BYTES + kk * 32, 16, 1024);
              umma_bf16(tmem + uint32_t(a * NT), ad, b, idesc, (i > 0 || kk > 0) ? 1u : 0u);
            }
          }
        }
        umma_commit(&empty[s]);  // the probe still hands every stage back
        if (i == nk - 1) umma_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: warps 2..5 own TMEM lanes 32*(warp%4) ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // weight row inside the tile
    const int m = m0 + row;
    const uint32_t lane_addr = tmem + (uint32_t(quarter * 32) << 16);
    const int et = threadIdx.x - 64;      // 0..127
    float* part = g.partial + (size_t(tile) * g.ks + ks_id) * NA * NT * BM;
    grid_dep_wait();  // outputs are written only once the predecessor grid is complete
    if (kb1 > kb0) {
      mbar_wait(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (!DOWN && g.ks > 1) {
#pragma unroll 1
      for (int c = 0; c < NT; c += 16) {
        uint32_t r[NA][16];
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          if (kb1 > kb0) {
            tmem_ld16(lane_addr + uint32_t(a * NT + c), r[a]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) r[a][e] = 0u;
          }
        }
        if (m >= g.rows) continue;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int t = t0 + c + e;
          if (t >= g.T) break;
#pragma unroll
          for (int a = 0; a < NA; ++a)
            g.z[((int64_t(ks_id) * NA + a) * g.T + t) * g.zld + m] = __uint_as_float(r[a][e]);
        }
      }
    } else if (DOWN && g.split_slices) {
      float* ys = g.y + int64_t(ks_id) * g.y_split_stride;
#pragma unroll 1
      for (int c = 0; c < NT; c += 16) {
        uint32_t r[NA][16];
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          if (kb1 > kb0) {
            tmem_ld16(lane_addr + uint32_t(a * NT + c), r[a]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) r[a][e] = 0u;
          }
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int t = t0 + c + e;
          if (t >= g.T) break;
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            const int mm = m + a * BM;
            if (mm < g.rows) ys[int64_t(t) * g.ldy + mm] = __uint_as_float(r[a][e]);
          }
        }
      }
    } else if (g.ks == 1) {
      // direct epilogue from TMEM
#pragma unroll 1
      for (int c = 0; c < NT; c += 16) {
        uint32_t r[NA][16];
#pragma unroll
        for (int a = 0; a < NA; ++a) tmem_ld16(lane_addr + uint32_t(a * NT + c), r[a]);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int t = t0 + c + e;
          if (t >= g.T) break;
          if constexpr (DOWN) {
#pragma unroll
            for (int a = 0; a < NA; ++a) {
              const int mm = m + a * BM;
              if (mm < g.rows) g.y[int64_t(t) * g.ldy + mm] += __uint_as_float(r[a][e]);
            }
          } else {
            if (m >= g.rows) continue;
            float v = act_fn(g.act, __uint_as_float(r[0][e]));
            if constexpr (NA == 2) v *= __uint_as_float(r[1][e]);
            g.a_out[int64_t(t) * g.lda + m] = __float2bfloat16_rn(v);
          }
        }
      }
    } else {
      // split-K: partial [NA][128 rows][NT] (a row's tokens contiguous -> float4), then the
      // last split of the tile sums the KS partials in split order and runs the epilogue
      float* prow = part + size_t(row) * NT;
#pragma unroll 1
      for (int c = 0; c < NT; c += 16) {
        uint32_t r[16];
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          if (kb1 > kb0) {
            tmem_ld16(lane_addr + uint32_t(a * NT + c), r);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) r[e] = 0u;
          }
          float4* dst = reinterpret_cast<float4*>(prow + size_t(a) * BM * NT + c);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            dst[e] = make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                 __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]));
        }
      }
      __threadfence();
      epilogue_sync();
      if (et == 0) {
        const int ticket = atomicAdd(&g.tickets[tile], 1);
        *last_flag = ticket == g.ks - 1;
        if (ticket == g.ks - 1) g.tickets[tile] = 0;  // re-arm for the next launch
      }
      epilogue_sync();
      if (*last_flag) {
        __threadfence();
        const float* base = g.partial + size_t(tile) * g.ks * NA * NT * BM + size_t(row) * NT;
#pragma unroll 1
        for (int c = 0; c < NT && t0 + c < g.T; c += 16) {
          float4 acc[NA][4];
#pragma unroll
          for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[a][e] = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int q = 0; q < g.ks; ++q) {
            float4 v[NA][4];
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
              for (int e = 0; e < 4; ++e)
                v[a][e] = __ldcg(reinterpret_cast<const float4*>(base + (size_t(q) * NA + a) * BM * NT + c) + e);
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                acc[a][e].x += v[a][e].x;
                acc[a][e].y += v[a][e].y;
                acc[a][e].z += v[a][e].z;
                acc[a][e].w += v[a][e].w;
              }
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int t = t0 + c + e;
            if (t >= g.T) break;
            if constexpr (DOWN) {
#pragma unroll
              for (int a = 0; a < NA; ++a) {
                const int mm = m + a * BM;
                if (mm < g.rows) g.y[int64_t(t) * g.ldy + mm] += reinterpret_cast<const float*>(&acc[a][0])[e];
              }
            } else {
              if (m >= g.rows) continue;
              float o = act_fn(g.act, reinterpret_cast<const float*>(&acc[0][0])[e]);
              if constexpr (NA == 2) o *= reinterpret_cast<const float*>(&acc[NA - 1][0])[e];
              g.a_out[int64_t(t) * g.lda + m] = __float2bfloat16_rn(o);
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (g.kspan1 && threadIdx.x == 0) atomicMax(g.kspan1, global_ns());
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

// ---- up GEMM on CTA pairs (tcgen05 cta_group::2) ------------------------------
//
// The up GEMM is operand-delivery bound: with the MMAs switched off it runs as
// long as with them (T = 512: 167 vs 152 us), each SM taking in ~55 GB/s of
// weight + x tiles.  A CTA pair (cluster of 2 on one TPC) issues one
// M = 256 MMA: rank r holds weight rows m0 + 128 r (its own TMEM accumulators)
// and HALF of the x tile (tokens t0 + r * NT/2); the tensor cores read the
// peer's half over the pair.  Per k-block each SM then loads 32 KB of W1/W3
// and NT/2 token rows instead of NT: 48 KB instead of 64 at NT = 256.
// Rank 0 issues the MMAs; both ranks' TMA loads complete on rank 0's full
// barrier (cta_group::2 form), the MMA commits arrive on both ranks' empty
// barriers and accumulator barrier (multicast), and each rank runs its own
// epilogue over its 128 rows exactly as gemm_kernel does.

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (own smem) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

// grid: 2 * pairs * ks CTAs, cluster (2, 1, 1); pair p -> (tile pair, split) like gemm_kernel
template <int NT, int NA>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_up_pair_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                        const __grid_constant__ CUtensorMap tmB, const GemmArgs g) {
  constexpr int HALF = NT / 2;          // token rows of x this rank loads
  constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  constexpr int B_BYTES = HALF * BK * 2;
  constexpr int STAGE = NA * A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = (NA * NT) <= 32 ? 32 : (NA * NT) <= 64 ? 64 : (NA * NT) <= 128 ? 128
                            : (NA * NT) <= 256 ? 256 : 512;
  static_assert(HALF % 8 == 0, "x half-tile must be whole 8-row swizzle atoms");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * STAGE);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (g.kspan0 && threadIdx.x == 0) atomicMin(g.kspan0, global_ns());
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int ks_id = pair % g.ks;
  const int tp = pair / g.ks;  // = mt_pair * t_tiles + tt
  const int mt = tp / g.t_tiles, tt = tp % g.t_tiles;
  const int m0 = (mt * 2 + int(rank)) * BM, t0 = tt * NT;
  const int nkb = (g.k + BK - 1) / BK;
  const int kb0 = nkb * ks_id / g.ks, kb1 = nkb * (ks_id + 1) / g.ks;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both ranks' barriers initialised before any TMA signals rank 0
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int nk = kb1 - kb0;
  grid_dep_launch();
  if (warp == 0) {
    // ---------------- TMA producer (both ranks) ----------------
    if (lane == 0) {
      auto load_a = [&](int i) {
        const int kb = kb0 + i, s = i % S;
        unsigned char* st = smem + size_t(s) * STAGE;
        const uint32_t lbar = map_to_rank(&full[s], 0);
        tma_load_2d_pair(st, &tmA0, lbar, kb * BK, m0);
        if constexpr (NA == 2) tma_load_2d_pair(st + A_BYTES, &tmA1, lbar, kb * BK, m0);
      };
      auto load_b = [&](int i) {
        const int kb = kb0 + i, s = i % S;
        tma_load_2d_pair(smem + size_t(s) * STAGE + NA * A_BYTES, &tmB, map_to_rank(&full[s], 0), kb * BK,
                         t0 + int(rank) * HALF);
      };
      const int pre = nk < S ? nk : S;
      for (int i = 0; i < pre; ++i) {
        if (rank == 0) mbar_expect_tx(&full[i], 2 * STAGE);
        load_a(i);
      }
      grid_dep_wait();
      for (int i = 0; i < pre; ++i) load_b(i);
      for (int i = pre; i < nk; ++i) {
        const int s = i % S;
        mbar_wait(&empty[s], ((i / S) - 1) & 1);
        if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE);
        load_a(i);
        load_b(i);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (rank 0 only) ----------------
    if (rank == 0) {
      const uint32_t idesc = umma_idesc(2 * BM, NT, false);
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const unsigned char* st = smem + size_t(s) * STAGE;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t b = umma_desc(st + NA * A_BYTES + kk * 32, 16, 1024);
#pragma unroll
            for (int a = 0; a < NA; ++a)
              umma_bf16_pair(tmem + uint32_t(a * NT), umma_desc(st + a * A_BYTES + kk * 32, 16, 1024), b, idesc,
                             (i > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit_pair(&empty[s]);
          if (i == nk - 1) umma_commit_pair(tmem_full);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5, this rank's 128 rows ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int m = m0 + row;
    const uint32_t lane_addr = tmem + (uint32_t(quarter * 32) << 16);
    grid_dep_wait();
    if (kb1 > kb0) {
      mbar_wait(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
#pragma unroll 1
    for (int c = 0; c < NT; c += 16) {
      uint32_t r[NA][16];
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        if (kb1 > kb0) {
          tmem_ld16(lane_addr + uint32_t(a * NT + c), r[a]);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) r[a][e] = 0u;
        }
      }
      if (m >= g.rows) continue;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int t = t0 + c + e;
        if (t >= g.T) break;
        if (g.ks > 1) {
#pragma unroll
          for (int a = 0; a < NA; ++a)
            g.z[((int64_t(ks_id) * NA + a) * g.T + t) * g.zld + m] = __uint_as_float(r[a][e]);
        } else {
          float v = act_fn(g.act, __uint_as_float(r[0][e]));
          if constexpr (NA == 2) v *= __uint_as_float(r[1][e]);
          g.a_out[int64_t(t) * g.lda + m] = __float2bfloat16_rn(v);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // the peer's MMAs / barrier traffic are over before either rank frees or exits
  if (g.kspan1 && threadIdx.x == 0) atomicMax(g.kspan1, global_ns());
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

// a[t, h] = act(sum_q z[q][0][t][h]) [* sum_q z[q][1][t][h]], splits summed in order
__global__ void swiglu_reduce_kernel(const float* __restrict__ z, int ks, int na, int T, int R, int64_t zld,
                                     int act, __nv_bfloat16* __restrict__ a_out, int64_t lda) {
  grid_dep_launch();
  grid_dep_wait();  // z comes from the up GEMM
  const int t = blockIdx.y;
  const int h = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (h >= R) return;
  const int64_t plane = int64_t(T) * zld;
  float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
  for (int q = 0; q < ks; ++q) {
    const float* base = z + (int64_t(q) * na * T + t) * zld + h;
    const float4 v0 = __ldcg(reinterpret_cast<const float4*>(base));
    s0.x += v0.x; s0.y += v0.y; s0.z += v0.z; s0.w += v0.w;
    if (na == 2) {
      const float4 v1 = __ldcg(reinterpret_cast<const float4*>(base + plane));
      s1.x += v1.x; s1.y += v1.y; s1.z += v1.z; s1.w += v1.w;
    }
  }
  float o[4] = {act_fn(act, s0.x), act_fn(act, s0.y), act_fn(act, s0.z), act_fn(act, s0.w)};
  if (na == 2) {
    o[0] *= s1.x; o[1] *= s1.y; o[2] *= s1.z; o[3] *= s1.w;
  }
  __nv_bfloat16* dst = a_out + int64_t(t) * lda + h;
  for (int e = 0; e < 4 && h + e < R; ++e) dst[e] = __float2bfloat16_rn(o[e]);
}

// gather x rows (any dtype) into a contiguous bf16 [T, ldo] buffer; `vec`: 8 elements
// per thread with 16-byte (bf16) / 2 x 16-byte (f32) loads (rows 16-byte aligned)
__global__ void gather_rows_bf16_kernel(const void* x, int xdtype, int64_t ldx_in, const int32_t* ids, int t0,
                                        int T, int M, __nv_bfloat16* out, int64_t ldo, int vec,
                                        unsigned long long* kspan0) {
  grid_dep_launch();  // the up GEMM starts streaming its weights meanwhile
  if (kspan0 && threadIdx.x == 0) atomicMin(kspan0, global_ns());
  const int t = blockIdx.y;
  if (t >= T) return;
  const int64_t row = ids ? ids[t0 + t] : int64_t(t0 + t);
  if (vec) {
    for (int k = (blockIdx.x * blockDim.x + threadIdx.x) * 8; k < M; k += gridDim.x * blockDim.x * 8) {
      uint4 o;
      if (xdtype == 1) {
        o = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + row * ldx_in + k);
      } else {
        const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(x) + row * ldx_in + k);
        const float4 a = src[0], b = src[1];
        __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x, b.y), p3 = __floats2bfloat162_rn(b.z, b.w);
        o.x = *reinterpret_cast<uint32_t*>(&p0);
        o.y = *reinterpret_cast<uint32_t*>(&p1);
        o.z = *reinterpret_cast<uint32_t*>(&p2);
        o.w = *reinterpret_cast<uint32_t*>(&p3);
      }
      *reinterpret_cast<uint4*>(out + int64_t(t) * ldo + k) = o;
    }
    return;
  }
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < M; k += gridDim.x * blockDim.x) {
    const float v = xdtype == 1 ? bf16_to_f(static_cast<const uint16_t*>(x)[row * ldx_in + k])
                                : static_cast<const float*>(x)[row * ldx_in + k];
    out[int64_t(t) * ldo + k] = __float2bfloat16_rn(v);
  }
}

}  // namespace tc
}  // namespace sp
