// Operand-delivery probe: how fast can 148 CTAs stream a [R, 4096] bf16 weight
// matrix (row stride 8 KB) from HBM into shared memory, by delivery method?
// No math: a consumer warp waits each stage and hands it back.  This isolates
// the up GEMM's A-operand pattern (128 B from each of 128 rows per k-block)
// from the tensor cores.
//
//   V0  2-D TMA box {64 el, 128 rows}, SWIZZLE_128B       (gemm_kernel's A tile, 16 KB)
//   V1  4-D TMA box {64, 8 rows, 4 atoms, 16 groups}, SW128 (128 rows x 512 B/row, 64 KB,
//       smem [group][atom][row][128 B] -- a UMMA K-major SW128 layout with SBO = 4 KB)
//   V2  1-D cp.async.bulk, 32 KB contiguous                (ffn_block_kernel's pattern)
//   V3  2-D TMA box {256 el, 32 rows}, no swizzle           (32 rows x 512 B, 16 KB)
//   V4  3-D TMA box {64, 128 rows, 2 atoms}, SW128          (128 rows x 256 B, 32 KB)
//   V5  4-D TMA box {64, 8, 2, 16}, SW128                   (128 rows x 256 B, [group][atom][row])
//   V6  3-D TMA box {64, 4 atoms, 128 rows}, SW128           (128 rows x 512 B, smem [row][atom])
//   V7  V0 on TWO row tiles per stage from distant regions    (the up GEMM's W1t + W3t pair, 32 KB)
//   V8  V0 on two ADJACENT row tiles per stage                (256 consecutive rows, 32 KB)
//
// Each CTA owns row tiles of 128 rows (tile c, c + grid, ...) and walks k inside a
// tile; in-flight bytes per CTA are ~192 KB for every variant.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <algorithm>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

constexpr int K = 4096;
constexpr int ROWS_PER_TILE = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// L2 flush without dirty lines: read a buffer larger than L2 (a memset would leave
// ~100 MB of dirty lines whose write-back competes with the measured reads)
__global__ void read_flush(const int4* __restrict__ p, size_t n, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const int4 v = __ldcs(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x7fffffff) *sink = 1;
}

struct Args {
  int variant, stage_bytes, stages, tiles;
  const char* base;  // for V2
};

__device__ unsigned long long g_t0 = ~0ull, g_t1 = 0;

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, Args a) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(&g_t0, t);
  }
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(a.stages) * a.stage_bytes);
  uint64_t* empty = full + a.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // k-steps per tile
  const int kstep_el = (a.variant == 0 || a.variant >= 7) ? 64 : (a.variant == 1 || a.variant == 3 || a.variant == 6) ? 256
                       : a.variant == 2 ? 0 : 128;
  int steps_per_tile;
  if (a.variant == 2) steps_per_tile = ROWS_PER_TILE * K * 2 / a.stage_bytes;
  else if (a.variant == 3) steps_per_tile = (K / kstep_el) * (ROWS_PER_TILE / 32);
  else steps_per_tile = K / kstep_el;
  const int my_tiles = (a.tiles - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
  const int n = my_tiles * steps_per_tile;
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int s = i % a.stages;
        if (i >= a.stages) mbar_wait(&empty[s], ((i / a.stages) - 1) & 1);
        const int tile = int(blockIdx.x) + (i / steps_per_tile) * int(gridDim.x);
        const int j = i % steps_per_tile;
        const int r0 = tile * ROWS_PER_TILE;
        unsigned char* st = smem + size_t(s) * a.stage_bytes;
        mbar_expect_tx(&full[s], a.stage_bytes);
        switch (a.variant) {
          case 0: tma2(st, &tm, &full[s], j * 64, r0); break;
          case 1: tma4(st, &tm, &full[s], 0, 0, j * 4, r0 / 8); break;
          case 2: bulk(st, a.base + size_t(r0) * K * 2 + size_t(j) * a.stage_bytes, a.stage_bytes, &full[s]); break;
          case 3: tma2(st, &tm, &full[s], (j % (K / 256)) * 256, r0 + (j / (K / 256)) * 32); break;
          case 4: tma3(st, &tm, &full[s], 0, r0, j * 2); break;
          case 5: tma4(st, &tm, &full[s], 0, 0, j * 2, r0 / 8); break;
          case 6: tma3(st, &tm, &full[s], 0, j * 4, r0); break;
          case 7:  // tile pair (r0 in the first half, r0 + half in the second)
            tma2(st, &tm, &full[s], j * 64, r0);
            tma2(st + 16384, &tm, &full[s], j * 64, r0 + a.tiles * ROWS_PER_TILE);
            break;
          case 8:
            tma2(st, &tm, &full[s], j * 64, 2 * r0);
            tma2(st + 16384, &tm, &full[s], j * 64, 2 * r0 + 128);
            break;
        }
      }
    }
  } else {
    for (int i = 0; i < n; ++i) {
      const int s = i % a.stages;
      mbar_wait(&full[s], (i / a.stages) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (lane == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(&g_t1, t);
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static bool make_map(int v, CUtensorMap* m, void* base, int64_t R) {
  auto f = enc();
  const uint64_t rs = uint64_t(K) * 2;
  CUresult r;
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (v == 0) {
    cuuint64_t d[2] = {cuuint64_t(K), cuuint64_t(R)};
    cuuint64_t st[1] = {rs};
    cuuint32_t b[2] = {64, 128};
    r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (v == 1 || v == 5) {
    const int atoms = v == 1 ? 4 : 2;
    cuuint64_t d[4] = {64, 8, cuuint64_t(K / 64), cuuint64_t(R / 8)};
    cuuint64_t st[3] = {rs, 128, rs * 8};
    cuuint32_t b[4] = {64, 8, cuuint32_t(atoms), 16};
    r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (v == 3) {
    cuuint64_t d[2] = {cuuint64_t(K), cuuint64_t(R)};
    cuuint64_t st[1] = {rs};
    cuuint32_t b[2] = {256, 32};
    r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (v == 4) {
    cuuint64_t d[3] = {64, cuuint64_t(R), cuuint64_t(K / 64)};
    cuuint64_t st[2] = {rs, 128};
    cuuint32_t b[3] = {64, 128, 2};
    r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (v == 7 || v == 8) {
    return make_map(0, m, base, R);
  } else if (v == 6) {
    cuuint64_t d[3] = {64, cuuint64_t(K / 64), cuuint64_t(R)};
    cuuint64_t st[2] = {128, rs};
    cuuint32_t b[3] = {64, 4, 128};
    r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    return true;
  }
  if (r != CUDA_SUCCESS) printf("variant %d: tensor map encode failed (%d)\n", v, int(r));
  return r == CUDA_SUCCESS;
}

int main(int argc, char** argv) {
  const int64_t RMAX = 148 * 128 * 3;  // 444 MB of bf16 weights, > L2
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* w;
  CK(cudaMalloc(&w, size_t(RMAX) * K * 2));
  CK(cudaMemset(w, 1, size_t(RMAX) * K * 2));
  void* flush;
  CK(cudaMalloc(&flush, size_t(256) << 20));
  CK(cudaMemset(flush, 0, size_t(256) << 20));
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  const int stage_bytes[9] = {16384, 65536, 32768, 16384, 32768, 32768, 65536, 32768, 32768};
  const char* names[9] = {"V0 tma2d 128rx128B sw128", "V1 tma4d 128rx512B sw128", "V2 bulk1d 32KB contiguous",
                          "V3 tma2d 32rx512B noswz", "V4 tma3d 128rx256B sw128", "V5 tma4d 128rx256B sw128",
                          "V6 tma3d 128rx512B [row][atom]", "V7 tma2d x2 distant tiles", "V8 tma2d x2 adjacent tiles"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid : {sms, 112}) {
    // whole tiles per CTA: every CTA streams the same bytes (no tail)
    const int64_t R = int64_t(grid) * 128 * (RMAX / (int64_t(grid) * 128));
    const size_t bytes = size_t(R) * K * 2;
    for (int v = 0; v < 9; ++v) {
      CUtensorMap tm{};
      if (!make_map(v, &tm, w, R)) continue;
      Args a{v, stage_bytes[v], std::min(12, (200 * 1024) / stage_bytes[v]),
             int(R / ROWS_PER_TILE) / (v >= 7 ? 2 : 1),
             static_cast<const char*>(w)};
      const size_t smem = size_t(a.stages) * a.stage_bytes + 1024 + 512;
      std::vector<float> ts, ds;
      for (int rep = 0; rep < 7; ++rep) {
        read_flush<<<sms * 4, 512>>>(static_cast<const int4*>(flush), (size_t(256) << 20) / 16,
                                     static_cast<int*>(flush));
        unsigned long long i0 = ~0ull, i1 = 0;
        cudaMemcpyToSymbol(g_t0, &i0, 8);
        cudaMemcpyToSymbol(g_t1, &i1, 8);
        cudaEventRecord(e0);
        stream_kernel<<<grid, 64, smem>>>(tm, a);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long t0, t1;
        cudaMemcpyFromSymbol(&t0, g_t0, 8);
        cudaMemcpyFromSymbol(&t1, g_t1, 8);
        if (rep > 0) {
          ts.push_back(ms);
          ds.push_back(float(t1 - t0) * 1e-6f);
        }
      }
      std::sort(ts.begin(), ts.end());
      std::sort(ds.begin(), ds.end());
      const float ms = ts[ts.size() / 2], dms = ds[ds.size() / 2];
      printf("grid %3d  %-30s stages %2d  %8.1f us  %7.0f GB/s   device span %8.1f us  %7.0f GB/s\n", grid, names[v],
             a.stages, ms * 1e3, bytes / (ms * 1e-3) / 1e9, dms * 1e3, bytes / (dms * 1e-3) / 1e9);
    }
  }
  return 0;
}
