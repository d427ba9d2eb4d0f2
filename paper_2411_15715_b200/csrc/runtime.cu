// runtime.cu -- libsliced: placement, streams, CG streamer, CC threads, merge.
//
// The reference executes the three column blocks one after another in numpy
// (slicing_kernel.py:119-123).  Here one sp_forward_batch call runs them
// concurrently on the four streams of the paper's pipeline:
//   Stream-A  host thread pool      CC block (host_cc.cpp)
//   Stream-B  this calling thread   kernel launches
//   Stream-C  copy stream           CG chunks pinned host -> 3-slot HBM ring
//   Stream-D  compute stream        GG kernels, CG chunk kernels, merge
// and sums the partial outputs in a merge kernel.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sliced.h"
#include <immintrin.h>

#include "host_cc.h"
#include "kernels.cuh"
#include "gemm_tc.cuh"
#include <cudaTypedefs.h>


namespace sp {

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define SP_CUDA(expr)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(SP_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                \
  } while (0)

#define SP_TRY(expr)              \
  do {                            \
    int s_ = (expr);              \
    if (s_ != SP_OK) return s_;   \
  } while (0)

static inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// device buffers

// Growable device buffer.  Growth doubles (steady state never grows again) and,
// given the stream that uses the buffer, is stream-ordered (cudaFreeAsync /
// cudaMallocAsync): a plain cudaFree synchronises the whole device, i.e. waits
// for every in-flight chunk copy -- a 10-30 ms stall inside a decode step.
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  bool async = false;
  int ensure(size_t bytes, cudaStream_t s = nullptr) {
    if (bytes <= n) return SP_OK;
    const size_t want = std::max({bytes, n * 2, size_t(1) << 20});
    if (s) {
      if (p) {
        if (async) cudaFreeAsync(p, s);
        else cudaFree(p);
      }
      p = nullptr;
      n = 0;
      if (cudaMallocAsync(&p, want, s) != cudaSuccess)
        return fail(SP_ERR_NOMEM, "cudaMallocAsync(%zu) failed", want);
      async = true;
    } else {
      if (p) {
        if (async) cudaFreeAsync(p, 0);
        else cudaFree(p);
      }
      p = nullptr;
      n = 0;
      if (cudaMalloc(&p, want) != cudaSuccess) return fail(SP_ERR_NOMEM, "cudaMalloc(%zu) failed", want);
      async = false;
    }
    n = want;
    return SP_OK;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// Growable pinned host buffer.  cudaFreeHost synchronises the device, so a
// grown-out buffer is retired (freed at destruction) instead of freed on the
// spot; growth doubles, so the retired total stays below the live size.
struct PinnedBuf {
  void* p = nullptr;
  size_t n = 0;
  std::vector<void*> retired;
  int ensure(size_t bytes) {
    if (bytes <= n) return SP_OK;
    const size_t want = std::max({bytes, n * 2, size_t(1) << 16});
    if (p) retired.push_back(p);
    p = nullptr;
    n = 0;
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess)
      return fail(SP_ERR_NOMEM, "cudaHostAlloc(%zu) failed", want);
    n = want;
    return SP_OK;
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
    for (void* r : retired) cudaFreeHost(r);
  }
};

constexpr int kMaxRingSlots = 8;


// Measured timeline: CUDA events on the library's streams (GPU spans) and the
// host clock (launch / CC spans), both relative to one synchronised origin.
struct Span {
  cudaEvent_t a = nullptr, b = nullptr;  // GPU span
  int kslot = -1;                        // kernel-side span slot (ffn_block launches)
  double ha = 0, hb = 0;                 // host span (seconds since host_t0)
  int stream, kind, call;
  double bytes;
};
struct Trace {
  bool on = false;
  // sp_trace_enable(2): GPU spans only around GG launches (the roofline
  // kernel); copy / chunk / merge spans are skipped, so the traced step keeps
  // the timing of an untraced one (events on the copy stream cost stream time
  // while the link is saturated, scripts/probes/event_span.cu).  Host spans
  // are always recorded (host clock, no device work).
  bool gg_only = false;
  cudaEvent_t t0 = nullptr;
  double host_t0 = 0;
  int call = 0;
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
  // kernel-side spans: starts[kKSlots] (init ~0) | ends[kKSlots] (init 0), device
  unsigned long long* kspan = nullptr;
  int kspan_next = 0;
  int kslot_cur = -1;  // slot of the GpuSpan being enqueued, picked up by ffn_args
};
constexpr int kKSlots = 16384;
constexpr int kTracePoolEvents = 8192;

struct Context {
  int device = -1;
  bool host_only = false;  // sp_init(-1): CC kernels only, for GPU-less hosts
  int num_sms = 0;
  cudaStream_t s_comp = nullptr, s_copy = nullptr, s_aux = nullptr;
  cudaEvent_t ev_user, ev_x, ev_ycc, ev_done;
  cudaEvent_t ev_meta = nullptr;  // on s_copy after a forward's metadata copies
  cudaEvent_t ev_copied[kMaxRingSlots], ev_free[kMaxRingSlots];
  DevBuf ring[kMaxRingSlots];
  size_t ring_bytes = 0;
  int ring_next = 0;
  DevBuf ws;         // device workspace
  // Pinned host staging (ids/gates, CSR, x, y_cc, y), two halves used by
  // alternate forwards: a device-I/O forward returns before its copies and its
  // finalize (which reads y_cc in place) have run, so the next forward must not
  // write the same bytes.  hpin_done[i] is recorded after the last GPU use of
  // half i; a forward waits on it before reusing the half.
  PinnedBuf hpin[2];
  cudaEvent_t hpin_done[2] = {nullptr, nullptr};
  bool hpin_used[2] = {false, false};
  int hpin_turn = 0;
  cudaEvent_t ev_ws = nullptr;  // on s_comp after this forward's workspace (re)allocation
  PinnedBuf xroute;  // x read back for the MoE router (and reused by the CC blocks)
  DevBuf tc_partial;  // split-K partial tiles of the tensor-core GEMMs
  DevBuf tc_tickets;  // per-tile split tickets (zero, re-armed by the last split)
  DevBuf tc_z;        // up-GEMM split partials of the pre-activations
  // a forward's device metadata (token ids, gates, finalize CSR), alternating
  // like the pinned halves: half hb's previous user finished (hpin_done[hb]),
  // so it is overwritten from the copy stream without waiting on s_comp
  DevBuf dmeta[2];
  std::vector<float> hscratch;
  std::unique_ptr<ThreadPool> pool;
  int host_threads = 1;
  // caller-supplied CC executor (sp_set_cc_executor): when set, every CC block
  // runs through it instead of the native host kernels
  sp_cc_fn cc_fn = nullptr;
  void* cc_user = nullptr;
  // CC coordinator: runs a forward's CC block (on `pool`) while the calling
  // thread keeps enqueueing GPU work -- Stream-A and Stream-B of PAPER.md:161
  // on separate host threads.
  std::thread cc_thread;
  std::mutex cc_mu;
  std::condition_variable cc_cv;
  std::function<int()> cc_job;
  std::function<int()> cc_tail;  // work to run after the CC block (see cc_join_with_tail)
  bool cc_pending = false, cc_stop = false, cc_done = false;
  int cc_status = 0;
  std::string cc_error;
  std::mutex trace_mu;  // spans come from the calling thread and the coordinator

  ~Context() {
    {
      std::lock_guard<std::mutex> lk(cc_mu);
      cc_stop = true;
      cc_cv.notify_all();
    }
    if (cc_thread.joinable()) cc_thread.join();
  }
  std::mutex mu;
  Trace trace;
  std::map<std::pair<const void*, size_t>, int> occ_cache;
  uint64_t launches = 0, h2d_bytes = 0;
  unsigned long long* stamps = nullptr;  // SP_KSTAMPS=1: per-CTA %globaltimer stamps of ffn_block
};

static std::mutex g_ctx_mu;
static std::unique_ptr<Context> g_ctx;

static Context* ctx_or_null() { return g_ctx.get(); }

// Bind the calling thread to the context's device.  The ABI may be entered from
// any host thread (a Python worker, a rank whose current device was never
// set); every entry point that touches the library's streams or device memory
// goes through here first.
static int bind_device(const Context* C) {
  if (!C || C->device < 0) return SP_OK;
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != C->device) {
    const cudaError_t e = cudaSetDevice(C->device);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, "cudaSetDevice(%d): %s", C->device, cudaGetErrorString(e));
  }
  return SP_OK;
}

// ---------------------------------------------------------------------------
// layer placement
//
// Packed block layout (see kernels.cuh): W1t[rows, ldm] | W3t[rows, ldm] | W2[rows, ldn].
// GG block rows [b2, H) live in HBM; CC rows [0, b1) and CG rows [b1, b2) live in
// one pinned host region as chunks of chunk_rows hidden units, each chunk one
// contiguous (4 KB aligned) copy.  CC chunks double as the stream for the n_g
// rows diverted to the GPU (cg_prime).

struct Chunk {
  int64_t r0, rc;
  size_t off, bytes;       // within the pinned host region
  size_t w3_off, w2_off;   // offsets inside the chunk
  bool cc;
};

}  // namespace sp

struct sp_layer {
  sp_layer_desc d;
  int device;
  size_t esz;
  int64_t ldm, ldn;        // padded M, padded N
  // GG (HBM)
  int64_t h_gg;
  void* gg = nullptr;
  size_t gg_bytes = 0, gg_w3_off = 0, gg_w2_off = 0;
  // host region (pinned): CC chunks then CG chunks
  void* host = nullptr;
  size_t host_bytes = 0, cc_bytes = 0, cg_bytes = 0;
  std::vector<sp::Chunk> chunks;
  bool host_only = false;
  size_t host_map_bytes = 0;  // > 0: host region is an mmap'd (THP) range registered with CUDA
  int n_cc_chunks = 0;
  size_t max_chunk_bytes = 0;
  // the CC rows' W2 in the AMX down phase's VNNI round blocks (sp::amx_prepack_w2),
  // built at the layer's first AMX CC block (SP_CC_PREPACK=0: never)
  uint16_t* w2_vnni = nullptr;
};

namespace sp {

// Copy rows [r0, r0 + n) of a row-major [*, cols] source into a [n, ld] block.
static void copy_rows(char* dst, int64_t ld, const char* src, int64_t cols, int64_t r0, int64_t n,
                      size_t esz) {
  for (int64_t r = 0; r < n; ++r)
    memcpy(dst + size_t(r) * ld * esz, src + size_t(r0 + r) * cols * esz, size_t(cols) * esz);
}

static int env_int(const char* name, int dflt);
// SP_HUGEPAGES=1: CC/CG host region on 2 MB transparent huge pages (mmap + cudaHostRegister)
static const bool g_hugepages = env_int("SP_HUGEPAGES", 0) != 0;
// default CG/CC chunk size (MB) when the layer does not set chunk_rows
static const int g_chunk_mb = std::max(1, env_int("SP_CHUNK_MB", 8));

// Layout + allocation of a layer's GG block (HBM) and host region (pinned
// CC then CG chunks); contents zeroed.  `fill_rows` / an image copy fill them.
static int place_layer(sp_layer* L) {
  const sp_layer_desc& d = L->d;
  const size_t esz = L->esz;
  const int G = d.gated ? 2 : 1;

  // ---- GG block -> HBM ----
  L->h_gg = d.hidden_dim - d.b2;
  if (L->h_gg > 0 && L->host_only)
    return fail(SP_ERR_STATE, "host-only context: a GG block (b2 < H) needs a CUDA device");
  if (L->h_gg > 0) {
    const size_t up = size_t(L->h_gg) * L->ldm * esz;
    L->gg_w3_off = up;
    L->gg_w2_off = up * G;
    L->gg_bytes = up * G + size_t(L->h_gg) * L->ldn * esz;
    SP_CUDA(cudaMalloc(&L->gg, L->gg_bytes));
    SP_CUDA(cudaMemset(L->gg, 0, L->gg_bytes));
  }

  // ---- CC and CG blocks -> pinned host, chunk-interleaved ----
  int64_t cr = d.chunk_rows;
  if (cr <= 0) {
    const int64_t row_bytes = (G * L->ldm + L->ldn) * int64_t(esz);
    cr = std::max<int64_t>(kPadElems, ((int64_t(g_chunk_mb) << 20) / row_bytes) / kPadElems * kPadElems);
  }
  cr = round_up(cr, kPadElems);
  L->d.chunk_rows = int32_t(cr);
  size_t off = 0;
  auto add_segment = [&](int64_t lo, int64_t hi, bool cc) {
    for (int64_t r0 = lo; r0 < hi; r0 += cr) {
      Chunk c;
      c.r0 = r0;
      c.rc = std::min(cr, hi - r0);
      c.cc = cc;
      const size_t up = size_t(c.rc) * L->ldm * esz;
      c.w3_off = up;
      c.w2_off = up * G;
      c.bytes = up * G + size_t(c.rc) * L->ldn * esz;
      c.off = off;
      off += round_up(int64_t(c.bytes), 4096);
      L->max_chunk_bytes = std::max(L->max_chunk_bytes, c.bytes);
      (cc ? L->cc_bytes : L->cg_bytes) += c.bytes;
      L->chunks.push_back(c);
    }
  };
  add_segment(0, d.b1, true);
  L->n_cc_chunks = int(L->chunks.size());
  add_segment(d.b1, d.b2, false);
  L->host_bytes = off;
  if (off > 0) {
    if (L->host_only) {
      L->host = aligned_alloc(4096, off);
      if (!L->host) return fail(SP_ERR_NOMEM, "aligned_alloc(%zu) failed", off);
    } else if (g_hugepages) {
      // 2 MB transparent huge pages: the CC threads' streams cross far fewer TLB
      // entries; the range is then page-locked for the copy engine.
      const size_t map = size_t(round_up(int64_t(off), int64_t(2) << 20));
      void* p = mmap(nullptr, map, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
      if (p == MAP_FAILED) return fail(SP_ERR_NOMEM, "mmap(%zu) for the CC/CG blocks failed", map);
      madvise(p, map, MADV_HUGEPAGE);
      memset(p, 0, map);
      if (cudaHostRegister(p, map, cudaHostRegisterDefault) != cudaSuccess) {
        cudaGetLastError();
        munmap(p, map);
        return fail(SP_ERR_NOMEM, "cudaHostRegister(%zu) for the CC/CG blocks failed", map);
      }
      L->host = p;
      L->host_map_bytes = map;
    } else if (cudaHostAlloc(&L->host, off, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      return fail(SP_ERR_NOMEM, "cudaHostAlloc(%zu) for the CC/CG blocks failed", off);
    }
    memset(L->host, 0, off);
  }
  return SP_OK;
}

// CG staging ring depth.  Decode steps are triple-buffered (the kernel
// consumes chunk i while i+1 and i+2 are in flight).  Long prefill streams
// (>= kLongStream chunks in one call) use 6 slots: the launching thread shares
// the cores with the CC block, and 5 queued copies (~0.8 ms) ride out its
// scheduling gaps where 2 did not (cfg3, alternating same-box pairs: e2e
// 430 -> 479 on one box, 477 -> 485 and prefill 533 -> 540 tokens/s on
// another; decode unchanged).  SP_RING_SLOTS / SP_RING_SLOTS_LONG override.
static const int g_ring_slots = std::max(2, std::min(kMaxRingSlots, env_int("SP_RING_SLOTS", 3)));
static const int g_ring_slots_long = std::max(2, std::min(kMaxRingSlots, env_int("SP_RING_SLOTS_LONG", 6)));
constexpr size_t kLongStream = 32;

// Fill a placed layer from row-major sources: w1t / w3t [H, M], w2 [H, N].
static int fill_rows(sp_layer* L, const void* w1t, const void* w3t, const void* w2) {
  const sp_layer_desc& d = L->d;
  const int64_t M = d.model_dim, N = d.out_dim;
  const size_t esz = L->esz;
  const char* s1 = static_cast<const char*>(w1t);
  const char* s3 = static_cast<const char*>(w3t);
  const char* s2 = static_cast<const char*>(w2);
  if (L->h_gg > 0) {
    char* g = static_cast<char*>(L->gg);
    SP_CUDA(cudaMemcpy2D(g, L->ldm * esz, s1 + size_t(d.b2) * M * esz, M * esz, M * esz, L->h_gg,
                         cudaMemcpyHostToDevice));
    if (d.gated)
      SP_CUDA(cudaMemcpy2D(g + L->gg_w3_off, L->ldm * esz, s3 + size_t(d.b2) * M * esz, M * esz,
                           M * esz, L->h_gg, cudaMemcpyHostToDevice));
    SP_CUDA(cudaMemcpy2D(g + L->gg_w2_off, L->ldn * esz, s2 + size_t(d.b2) * N * esz, N * esz,
                         N * esz, L->h_gg, cudaMemcpyHostToDevice));
  }
  char* h = static_cast<char*>(L->host);
  for (const Chunk& c : L->chunks) {
    char* base = h + c.off;
    copy_rows(base, L->ldm, s1, M, c.r0, c.rc, esz);
    if (d.gated) copy_rows(base + c.w3_off, L->ldm, s3, M, c.r0, c.rc, esz);
    copy_rows(base + c.w2_off, L->ldn, s2, N, c.r0, c.rc, esz);
  }
  return SP_OK;
}


// Row-major [H, M] / [H, N] copies of a placed layer's weights (GG rows read
// back from HBM): the input of a re-slice.
static int gather_rows(const sp_layer* L, char* w1t, char* w3t, char* w2) {
  const sp_layer_desc& d = L->d;
  const int64_t M = d.model_dim, N = d.out_dim;
  const size_t esz = L->esz;
  if (L->h_gg > 0) {
    const char* g = static_cast<const char*>(L->gg);
    SP_CUDA(cudaMemcpy2D(w1t + size_t(d.b2) * M * esz, M * esz, g, L->ldm * esz, M * esz, L->h_gg,
                         cudaMemcpyDeviceToHost));
    if (d.gated)
      SP_CUDA(cudaMemcpy2D(w3t + size_t(d.b2) * M * esz, M * esz, g + L->gg_w3_off, L->ldm * esz, M * esz,
                           L->h_gg, cudaMemcpyDeviceToHost));
    SP_CUDA(cudaMemcpy2D(w2 + size_t(d.b2) * N * esz, N * esz, g + L->gg_w2_off, L->ldn * esz, N * esz,
                         L->h_gg, cudaMemcpyDeviceToHost));
  }
  const char* h = static_cast<const char*>(L->host);
  for (const Chunk& c : L->chunks) {
    const char* base = h + c.off;
    for (int64_t r = 0; r < c.rc; ++r) {
      memcpy(w1t + size_t(c.r0 + r) * M * esz, base + size_t(r) * L->ldm * esz, size_t(M) * esz);
      if (d.gated) memcpy(w3t + size_t(c.r0 + r) * M * esz, base + c.w3_off + size_t(r) * L->ldm * esz, size_t(M) * esz);
      memcpy(w2 + size_t(c.r0 + r) * N * esz, base + c.w2_off + size_t(r) * L->ldn * esz, size_t(N) * esz);
    }
  }
  return SP_OK;
}

// ---------------------------------------------------------------------------
// kernel dispatch

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
// Tunables (read once): stage size target, ring depth cap, minimum hidden rows per CTA.
static const int g_stage_bytes = env_int("SP_STAGE_KB", 32) * 1024;
static const int g_max_stages = std::min(kMaxStages, env_int("SP_STAGES", kMaxStages));
static const int g_min_rows_per_cta = std::max(1, env_int("SP_MIN_ROWS", 4));
constexpr int kSmemLimit = 227 * 1024;
constexpr int kMaxTileFloats = 16384;  // TT * roundup(M, 256) floats of x <= 64 KB

// Streamed chunks hide under their own PCIe copy (~150 us for 8 MB), so they
// run on fewer, fatter CTAs: fewer partial slices for finalize_kernel.
static const int g_chunk_min_rows = std::max(1, env_int("SP_CHUNK_MIN_ROWS", 16));
// SP_WIDE_LAST_CHUNK=0: a call's last streamed chunk keeps the chunk grid too
static const bool g_wide_last_chunk = env_int("SP_WIDE_LAST_CHUNK", 1) != 0;

// CTAs a block of `rows` hidden units is split over (also its partial-slice count).
static int block_grid(const Context* C, int64_t rows, int min_rows = g_min_rows_per_cta) {
  if (rows <= 0) return 0;
  const int64_t by_rows = (rows + min_rows - 1) / min_rows;
  return int(std::max<int64_t>(1, std::min<int64_t>(C->num_sms, by_rows)));
}

// Largest token tile (1, 2 or 4) whose x copy fits the 64 KB budget.
static int max_token_tile(int64_t M) {
  const int64_t kt = round_up(M, 256);
  for (int tt : {4, 2, 1})
    if (tt * kt <= kMaxTileFloats) return tt;
  return 0;
}

// Most hidden rows one ffn_block CTA can own (its phase-1 partials live in
// shared memory next to the x tile and a 2-stage ring): a grouped launch of many
// experts must not pack more rows than this into one CTA.
static int64_t max_rows_per_cta(int64_t M, int gated, int tt, int xel) {
  const int64_t G = gated ? 2 : 1;
  const int64_t kt = round_up(M, 256);
  const int64_t fixed = int64_t(tt) * kt * 4 + (int64_t(tt) * M * xel + 15) / 16 * 16 + (2 * kMaxStages + 1) * 8 + 128;
  const int64_t per_row = int64_t(kConsumers) * G * tt * 4 + tt * 4;
  const int64_t room = int64_t(kSmemLimit) - fixed - 2 * int64_t(g_stage_bytes) - 1024;
  return std::max<int64_t>(1, room / per_row);
}

template <typename WT, int TT, bool GATED, int NV>
static int launch_ffn_t(Context* C, const FfnGroup& grp, int grid, cudaStream_t s) {
  constexpr int G = GATED ? 2 : 1;
  auto kern = ffn_block_kernel<WT, TT, GATED, NV>;
  static bool attr_set = false;
  if (!attr_set) {
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
    attr_set = true;
  }
  const FfnArgs& a = grp.a[0];
  int per_cta = 1;
  for (int i = 0; i < grp.n; ++i) per_cta = std::max(per_cta, (grp.a[i].rows + grp.a[i].ncta - 1) / grp.a[i].ncta);
  const int64_t row1 = a.ldm * int64_t(sizeof(WT)), row2 = a.ldn * int64_t(sizeof(WT));
  int rs_up = int(std::max<int64_t>(1, g_stage_bytes / (G * row1)));
  int rs_dn = int(std::max<int64_t>(1, g_stage_bytes / row2));
  rs_up = std::min(rs_up, per_cta);
  rs_dn = std::min(rs_dn, per_cta);
  const size_t stage = size_t(std::max<int64_t>(G * rs_up * row1, rs_dn * row2));
  const size_t xraw = a.xvec ? size_t((TT * a.M * (a.xdtype == 1 ? 2 : 4) + 15) / 16 * 16) : 0;
  const size_t fixed = size_t(TT) * a.kt * 4 + xraw + size_t(per_cta) * kConsumers * G * TT * 4 +
                       size_t((per_cta * TT + 1) & ~1) * 4 + (2 * kMaxStages + 1) * 8 + 128;
  if (fixed + 2 * stage > size_t(kSmemLimit))
    return fail(SP_ERR_VALUE, "block of %d rows/CTA (M=%d, N=%d) does not fit shared memory", per_cta, a.M, a.N);
  const int nst = int(std::min<size_t>(g_max_stages, (kSmemLimit - fixed) / stage));
  FfnPlan fp{rs_up, rs_dn, nst, int(stage)};
  kern<<<grid, kBlockThreads, size_t(nst) * stage + fixed, s>>>(grp, fp);
  SP_CUDA(cudaGetLastError());
  ++C->launches;
  return SP_OK;
}

template <typename WT, int TT, bool GATED>
static int launch_nv(Context* C, const FfnGroup& g, int grid, cudaStream_t s) {
  const FfnArgs& a = g.a[0];
  const int n_vec = (a.N + VecTraits<WT>::kElems - 1) / VecTraits<WT>::kElems;
  const int nv = (n_vec + kConsumers * 32 - 1) / (kConsumers * 32);
  if (nv <= 1) return launch_ffn_t<WT, TT, GATED, 1>(C, g, grid, s);
  if (nv <= 2) return launch_ffn_t<WT, TT, GATED, 2>(C, g, grid, s);
  if (nv <= 4) return launch_ffn_t<WT, TT, GATED, 4>(C, g, grid, s);
  return fail(SP_ERR_VALUE, "out_dim %d exceeds the kernel's %d column vectors per thread", a.N, kMaxVec);
}

template <typename WT, bool GATED>
static int launch_tt(Context* C, int tt, const FfnGroup& g, int grid, cudaStream_t s) {
  switch (tt) {
    case 1: return launch_nv<WT, 1, GATED>(C, g, grid, s);
    case 2: return launch_nv<WT, 2, GATED>(C, g, grid, s);
    default: return launch_nv<WT, 4, GATED>(C, g, grid, s);
  }
}

static int launch_group(Context* C, const sp_layer* L, int tt, const FfnGroup& g, int grid, cudaStream_t s) {
  if (L->d.wdtype == SP_BF16)
    return L->d.gated ? launch_tt<__nv_bfloat16, true>(C, tt, g, grid, s)
                      : launch_tt<__nv_bfloat16, false>(C, tt, g, grid, s);
  return L->d.gated ? launch_tt<float, true>(C, tt, g, grid, s) : launch_tt<float, false>(C, tt, g, grid, s);
}

// ---- eager module loading ------------------------------------------------
// CUDA loads kernels lazily (CUDA_MODULE_LOADING=LAZY is the default): the
// first launch of each template instance loads it, which can hold the host
// tens of ms and serialises against in-flight work.  With ~60 instances picked
// by token count at run time, a new routing pattern in the middle of a decode
// run paid that inside the step (measured: 55 ms outliers).  sp_init touches
// every instance once and sets its shared-memory opt-in.
template <typename K>
static int preload(K kern, bool big_smem) {
  cudaFuncAttributes a;
  SP_CUDA(cudaFuncGetAttributes(&a, kern));
  if (big_smem) SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
  return SP_OK;
}
template <typename WT, int TT, bool GATED>
static int preload_ffn() {
  SP_TRY(preload(ffn_block_kernel<WT, TT, GATED, 1>, true));
  SP_TRY(preload(ffn_block_kernel<WT, TT, GATED, 2>, true));
  return preload(ffn_block_kernel<WT, TT, GATED, 4>, true);
}
template <int NA, bool DOWN>
static int preload_gemm() {
  SP_TRY(preload(tc::gemm_kernel<16, NA, DOWN>, true));
  SP_TRY(preload(tc::gemm_kernel<32, NA, DOWN>, true));
  SP_TRY(preload(tc::gemm_kernel<64, NA, DOWN>, true));
  SP_TRY(preload(tc::gemm_kernel<128, NA, DOWN>, true));
  return preload(tc::gemm_kernel<256, NA, DOWN>, true);
}
static int preload_kernels() {
  SP_TRY((preload_ffn<float, 1, false>()));
  SP_TRY((preload_ffn<float, 2, false>()));
  SP_TRY((preload_ffn<float, 4, false>()));
  SP_TRY((preload_ffn<float, 1, true>()));
  SP_TRY((preload_ffn<float, 2, true>()));
  SP_TRY((preload_ffn<float, 4, true>()));
  SP_TRY((preload_ffn<__nv_bfloat16, 1, false>()));
  SP_TRY((preload_ffn<__nv_bfloat16, 2, false>()));
  SP_TRY((preload_ffn<__nv_bfloat16, 4, false>()));
  SP_TRY((preload_ffn<__nv_bfloat16, 1, true>()));
  SP_TRY((preload_ffn<__nv_bfloat16, 2, true>()));
  SP_TRY((preload_ffn<__nv_bfloat16, 4, true>()));
  SP_TRY((preload_gemm<1, false>()));
  SP_TRY((preload_gemm<2, false>()));
  SP_TRY((preload_gemm<2, true>()));
  SP_TRY(preload(finalize_kernel, false));
  SP_TRY(preload(finalize_rows_kernel, false));
  SP_TRY(preload(reduce_slices_kernel, false));
  SP_TRY(preload(finalize_scalar_kernel, false));
  SP_TRY(preload(tc::swiglu_reduce_kernel, false));
  SP_TRY(preload(tc::gemm_up_pair_kernel<256, 1>, true));
  SP_TRY(preload(tc::gemm_up_pair_kernel<256, 2>, true));
  return preload(tc::gather_rows_bf16_kernel, false);
}

// One weight block applied to tokens [t0, t0 + T) of a call: partial slices
// [slice0, slice0 + grid) of the call's partial buffer.
struct BlockView {
  const char* base;    // W1t at base, W3t at base + w3_off, W2 at base + w2_off
  size_t w3_off, w2_off;
  int64_t rows;
};

struct CallWs {
  float* part;     // [S][T_e][N] partial slices of every block of the call
  int S;           // slices in use
  int tc_slice = -1;            // slice the tensor-core blocks accumulate into
  int split_capacity = 0;       // spare slices for split-K partials of resident tc blocks
  __nv_bfloat16* x_tc = nullptr;  // [T_e, ldm] gathered bf16 x (tensor-core path)
  __nv_bfloat16* a_tc = nullptr;  // [T_e, ld_a] bf16 hidden activations of one block
  int64_t ld_a = 0;
  float* ycc;      // [T_e, N] CC partial (from the host)
  int32_t* ids;    // device
  float* gates;    // device
  bool ids_identity = false;  // the call's tokens are rows 0..T_e-1 of x (no token_ids)
};

// ---- tensor-core (tcgen05) block path for many tokens -------------------------
// Tensor-core path as soon as the CUDA-core path would need a second token tile
// (and so re-stream the weights); SP_TC_MIN_T overrides the threshold.
static const int g_tc_min_tokens_env = env_int("SP_TC_MIN_T", 0);
static int max_token_tile(int64_t M);
static bool use_tc(const sp_layer* L, int64_t T) {
  if (L->d.wdtype != SP_BF16) return false;
  return g_tc_min_tokens_env > 0 ? T >= g_tc_min_tokens_env : T > max_token_tile(L->d.model_dim);
}
// SP_CC_BATCH=0: one pool pass per call's CC block instead of one per step
static const bool g_cc_batch = env_int("SP_CC_BATCH", 1) != 0;
// SP_CC_FIRST=0: submit the CC block after the first chunk copies, as before
static const bool g_cc_first = env_int("SP_CC_FIRST", 1) != 0;
// SP_PREREDUCE=0: leave every partial slice to the finalize (no early reduction)
static const bool g_prereduce = env_int("SP_PREREDUCE", 1) != 0;
// The grouped GG launch runs behind the call's last chunk kernel, i.e. once the
// CG copies are done: a timing event recorded while copy-engine H2D traffic
// saturates the link lands ~23 us late (scripts/probes/event_span.cu), so only
// there does the event-timed GG span match the kernel.  Against the round-1
// placement (behind the first chunk copy), same-box alternating pairs: GG span
// by events 0.64 -> 0.86 of HBM, value 498 -> 511 and e2e 508 -> 532 tokens/s
// (profiles/r2/ab_gg_last.txt).  It is not free: with the calibrated split the
// CC block and the copies end within ~20 us of each other, so the group (64 us)
// sits on the step's tail (profiles/r2/timeline/cfg2_anatomy_*.txt).
// SP_GG_LAST=1 instead launches the group right after the call's last copy is
// queued: every copy is already enqueued (nothing it could delay) and the
// copies still in flight cover it, so it never lands on the step's tail (in a
// link-bound step, e.g. cfg4 on a fast-host box, the group behind the last
// chunk kernel adds ~120 us).  Same-box pairs with fixed rates
// (profiles/r2/ab_gg_placement.txt): cfg2 value +2.4 %, e2e +1.7 % (within the
// box noise), cfg4 inside the noise -- but every GG timing event then lands
// under the saturated link and the event-timed GG span reads 0.61 of HBM
// instead of 0.85 (device span 0.92 either way).  The default keeps the
// measurement clean.  SP_GG_LAST=0: behind the first chunk copy.
static const int g_gg_last = env_int("SP_GG_LAST", 2);
// SP_Y_ZERO_COPY=0: small host outputs go through a device buffer and a read-back copy
static const bool g_y_zero_copy = env_int("SP_Y_ZERO_COPY", 1) != 0;
static const bool g_host_merge = env_int("SP_HOST_MERGE", 1) != 0;
static const bool g_cc_prepack = env_int("SP_CC_PREPACK", 1) != 0;
constexpr size_t kZeroCopyY = size_t(256) << 10;
constexpr int kTcMaxSplits = 24;
// finalize: per-token rows kernel up to this many slices per call, slice groups beyond
constexpr int kFinRowsMaxSlices = 16;  // split-K output slices a resident tc block may use

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor map over a row-major [outer, inner] matrix, 128B swizzle, zero OOB fill.
static int make_tmap(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int64_t row_bytes,
                     int box_inner, int box_outer) {
  auto enc = tmap_encoder();
  if (!enc) return fail(SP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(row_bytes)};
  cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  const CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS)
    return fail(SP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): inner %lld outer %lld stride %lld", int(res),
                (long long)inner, (long long)outer, (long long)row_bytes);
  return SP_OK;
}

// SP_TC_PDL=0: the prefill chain's kernels wait for full completion of their predecessor
static const bool g_tc_pdl = env_int("SP_TC_PDL", 1) != 0;

// Launch with programmatic stream serialization when `pdl` (the kernel's
// griddepcontrol.wait then orders it after its predecessor; everything it does
// before that wait -- barrier init, TMEM alloc, the first weight stages --
// overlaps the predecessor's tail).  Only used when the previous operation on
// `s` is one of this chain's kernels.
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && g_tc_pdl) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <int NT, int NA, bool DOWN>
static int launch_gemm_t(Context* C, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b,
                         tc::GemmArgs g, cudaStream_t s, bool pdl) {
  auto kern = tc::gemm_kernel<NT, NA, DOWN>;
  constexpr int STAGE = NA * tc::BM * tc::BK * 2 + NT * tc::BK * 2;
  static bool attr_set = false;
  if (!attr_set) {
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
    attr_set = true;
  }
  const int ctas = g.m_tiles * g.t_tiles * g.ks;
  // one CTA per SM with a deep ring, or two per SM with a shallow one -- the
  // latter only when two CTAs with >= 2 stages each actually fit (a 64 KB stage
  // does not: halving the budget then just left one CTA per SM on 2 stages,
  // 132 KB instead of 198 KB of loads in flight -- the T = 512 up GEMM)
  const bool two_per_sm = ctas > C->num_sms && 2 * (2 * STAGE + 1024 + 256) <= kSmemLimit;
  const int budget = two_per_sm ? kSmemLimit / 2 - 1024 : kSmemLimit;
  g.stages = std::max(2, std::min(6, (budget - 1024 - 256) / STAGE));
  const size_t smem = size_t(g.stages) * STAGE + 1024 + 256;
  if (g.ks > 1 && (DOWN ? !g.split_slices : !g.z)) {
    // split-K fix-up through fp32 partial tiles (no current caller; allocating
    // here puts stream operations inside the chain, so it never runs under PDL)
    pdl = false;
    const size_t need = size_t(g.m_tiles) * g.t_tiles * g.ks * NA * NT * tc::BM * 4;
    SP_TRY(C->tc_partial.ensure(need, s));
    g.partial = static_cast<float*>(C->tc_partial.p);
    const size_t tk = size_t(g.m_tiles) * g.t_tiles * 4;
    if (tk > C->tc_tickets.n) {
      SP_TRY(C->tc_tickets.ensure(tk, s));
      SP_CUDA(cudaMemsetAsync(C->tc_tickets.p, 0, C->tc_tickets.n, s));
    }
    g.tickets = static_cast<int*>(C->tc_tickets.p);
  }
  static const int dbg_no_mma = env_int("SP_TC_DBG_NOMMA", 0);
  g.dbg_no_mma = dbg_no_mma;
  SP_CUDA(launch_k(kern, dim3(ctas), dim3(tc::kThreads), smem, s, pdl, a0, a1, b, g));
  ++C->launches;
  return SP_OK;
}

template <int NA, bool DOWN>
static int launch_gemm(Context* C, int nt, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b,
                       const tc::GemmArgs& g, cudaStream_t s, bool pdl) {
  switch (nt) {
    case 16: return launch_gemm_t<16, NA, DOWN>(C, a0, a1, b, g, s, pdl);
    case 32: return launch_gemm_t<32, NA, DOWN>(C, a0, a1, b, g, s, pdl);
    case 64: return launch_gemm_t<64, NA, DOWN>(C, a0, a1, b, g, s, pdl);
    case 128: return launch_gemm_t<128, NA, DOWN>(C, a0, a1, b, g, s, pdl);
    default:
      if constexpr (NA <= 2) return launch_gemm_t<256, NA, DOWN>(C, a0, a1, b, g, s, pdl);
      return fail(SP_ERR_VALUE, "token tile 256 with %d sub-tiles exceeds TMEM", NA);
  }
}

// up GEMM on CTA pairs (gemm_up_pair_kernel): rank r of pair p covers 128-row
// tile 2 * (p's row pair) + r and loads half of the x tile
template <int NT, int NA>
static int launch_gemm_pair_t(Context* C, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b,
                              tc::GemmArgs g, cudaStream_t s, bool pdl) {
  auto kern = tc::gemm_up_pair_kernel<NT, NA>;
  constexpr int STAGE = NA * tc::BM * tc::BK * 2 + (NT / 2) * tc::BK * 2;
  static bool attr_set = false;
  if (!attr_set) {
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
    attr_set = true;
  }
  const int pairs = (g.m_tiles + 1) / 2 * g.t_tiles;
  g.stages = std::max(2, std::min(6, (kSmemLimit - 1024 - 256) / STAGE));
  const size_t smem = size_t(g.stages) * STAGE + 1024 + 256;
  SP_CUDA(launch_k(kern, dim3(2 * pairs * g.ks), dim3(tc::kThreads), smem, s, pdl, a0, a1, b, g));
  ++C->launches;
  return SP_OK;
}

template <int NA>
static int launch_gemm_pair(Context* C, int nt, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b,
                            const tc::GemmArgs& g, cudaStream_t s, bool pdl) {
  switch (nt) {
    case 256: return launch_gemm_pair_t<256, NA>(C, a0, a1, b, g, s, pdl);
    case 128: return launch_gemm_pair_t<128, NA>(C, a0, a1, b, g, s, pdl);
    case 64: return launch_gemm_pair_t<64, NA>(C, a0, a1, b, g, s, pdl);
    case 32: return launch_gemm_pair_t<32, NA>(C, a0, a1, b, g, s, pdl);
    case 16: return launch_gemm_pair_t<16, NA>(C, a0, a1, b, g, s, pdl);
    default: return fail(SP_ERR_VALUE, "CTA-pair up GEMM: no %d-token tile", nt);
  }
}
// SP_TC_PAIR=0 keeps every up GEMM on single-CTA tiles
static const bool g_tc_pair = env_int("SP_TC_PAIR", 1) != 0;
// smallest token tile that runs the up GEMM on CTA pairs (SP_TC_PAIR_MIN_NT)
static const int g_tc_pair_min_nt = env_int("SP_TC_PAIR_MIN_NT", 16);

// Split K so the launch puts ~`target` CTAs to work (bounded by the k-blocks).
static int split_k(int tiles, int k, int target) {
  const int nkb = (k + tc::BK - 1) / tc::BK;
  return std::max(1, std::min(nkb, target / std::max(1, tiles)));
}

static const int64_t g_test_fail_after_cc = env_int("SP_TEST_FAIL_AFTER_CC", 0);
// up GEMM (fused SwiGLU / act) into a_tc, then down GEMM accumulated into the call's tc slice.
// Every workspace is sized and every memset enqueued first, so the chain
// gather -> up -> (swiglu_reduce) -> down is back-to-back kernels on `s` and
// each one after the gather is launched with PDL (launch_k).
static int run_block_tc(Context* C, const sp_layer* L, const BlockView& b, const void* x, int xdtype, int64_t ldx,
                        CallWs& w, const int32_t* dev_ids, int64_t T_e, int t0, int T, cudaStream_t s,
                        bool resident) {
  const int64_t M = L->d.model_dim, N = L->d.out_dim, R = b.rows;
  // streamed chunks accumulate into one shared slice (zeroed once per call);
  // a resident block stores its own split slices, so its chain starts with the gather
  if (!resident && w.tc_slice < 0) {
    w.tc_slice = w.S++;
    SP_CUDA(cudaMemsetAsync(w.part + size_t(w.tc_slice) * T_e * N, 0, size_t(T_e) * N * 4, s));
  }
  const int nt = T <= 16 ? 16 : T <= 32 ? 32 : T <= 64 ? 64 : T <= 128 ? 128 : 256;
  const int t_tiles = int((T + nt - 1) / nt);
  // HBM-resident blocks spread over every SM; streamed chunks hide under their copy
  // (SP_TC_UP_CTAS / SP_TC_DN_CTAS: probe overrides of the resident targets)
  static const int up_ctas_env = env_int("SP_TC_UP_CTAS", 0), dn_ctas_env = env_int("SP_TC_DN_CTAS", 0);
  const int target = resident ? C->num_sms : 32;
  const int up_target = resident && up_ctas_env > 0 ? up_ctas_env : target;
  const int dn_target = resident && dn_ctas_env > 0 ? dn_ctas_env : target;
  const int na = L->d.gated ? 2 : 1;
  tc::GemmArgs up{};
  up.mode = L->d.gated ? tc::kUpGated : tc::kUpPlain;
  up.act = L->d.act;
  up.rows = int(R);
  up.T = T;
  up.k = int(M);
  up.m_tiles = int((R + tc::BM - 1) / tc::BM);
  up.t_tiles = t_tiles;
  up.ks = split_k(up.m_tiles * t_tiles, int(M), up_target);
  up.a_out = w.a_tc;
  up.lda = w.ld_a;
  if (up.ks > 1) {
    // split partials of the pre-activations, finished by swiglu_reduce_kernel
    up.zld = round_up(R, 4);
    SP_TRY(C->tc_z.ensure(size_t(up.ks) * na * T * up.zld * 4, s));
    up.z = static_cast<float*>(C->tc_z.p);
  }
  tc::GemmArgs dn{};
  dn.mode = tc::kDown;
  dn.rows = int(N);
  dn.T = T;
  dn.k = int(R);
  // 2 column sub-tiles per CTA share each fetched `a` tile
  constexpr int sub = 2;
  dn.m_tiles = int((N + tc::BM * sub - 1) / (tc::BM * sub));
  dn.t_tiles = t_tiles;
  dn.ldy = N;
  if (resident) {
    // HBM-resident block: split K over ~every SM, one output slice per split
    dn.ks = std::min(split_k(dn.m_tiles * t_tiles, int(R), dn_target), w.split_capacity);
    dn.split_slices = 1;
    dn.y_split_stride = int64_t(T_e) * N;
    if (t0 > 0 || T < T_e)  // rows outside [t0, t0 + T) of the new slices must read as zero
      SP_CUDA(cudaMemsetAsync(w.part + size_t(w.S) * T_e * N, 0, size_t(dn.ks) * T_e * N * 4, s));
    dn.y = w.part + size_t(w.S) * T_e * N + size_t(t0) * N;
    w.S += dn.ks;
  } else {
    dn.ks = 1;  // streamed chunk: hidden under its copy, accumulate into the tc slice
    dn.y = w.part + size_t(w.tc_slice) * T_e * N + size_t(t0) * N;
  }
  if (C->trace.kslot_cur >= 0) {  // the block's chain span (trace ABI dev_s)
    up.kspan0 = dn.kspan0 = C->trace.kspan + C->trace.kslot_cur;
    up.kspan1 = dn.kspan1 = C->trace.kspan + kKSlots + C->trace.kslot_cur;
  }
  // bf16 x whose tokens are its own rows in order feeds the up GEMM's TMA
  // directly (out-of-range columns / rows read as zero); otherwise the gather
  // kernel builds the bf16 token tile first
  static const bool direct_x_env = env_int("SP_TC_DIRECT_X", 1) != 0;
  const bool x_direct = direct_x_env && w.ids_identity && xdtype == SP_BF16 && (size_t(ldx) * 2) % 16 == 0 &&
                        reinterpret_cast<uintptr_t>(x) % 16 == 0;
  const void* xt = x_direct ? static_cast<const void*>(static_cast<const char*>(x) + size_t(t0) * ldx * 2)
                            : static_cast<const void*>(w.x_tc);
  const int64_t xt_stride = x_direct ? ldx * 2 : L->ldm * 2;
  CUtensorMap tx, tw1, tw3, ta, tw2;
  SP_TRY(make_tmap(&tw1, b.base, M, R, L->ldm * 2, tc::BK, tc::BM));
  SP_TRY(make_tmap(&tw3, L->d.gated ? b.base + b.w3_off : b.base, M, R, L->ldm * 2, tc::BK, tc::BM));
  SP_TRY(make_tmap(&tx, xt, M, T, xt_stride, tc::BK, nt));
  SP_TRY(make_tmap(&tw2, b.base + b.w2_off, N, R, L->ldn * 2, 64, tc::BK));
  SP_TRY(make_tmap(&ta, w.a_tc, R, T, w.ld_a * 2, tc::BK, nt));

  // gathered bf16 x rows [T, M]
  if (!x_direct) {
    const size_t xel = xdtype == SP_BF16 ? 2 : 4;
    const bool vec = M % 8 == 0 && (size_t(ldx) * xel) % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
    const int per = vec ? 8 : 1;
    dim3 grid(unsigned(std::min<int64_t>((M / per + 255) / 256, 16)), unsigned(T));
    tc::gather_rows_bf16_kernel<<<grid, 256, 0, s>>>(x, xdtype, ldx, dev_ids, t0, T, int(M), w.x_tc, L->ldm,
                                                     vec ? 1 : 0, up.kspan0);
    SP_CUDA(cudaGetLastError());
    ++C->launches;
  }
  if (g_tc_pair && nt >= std::max(16, g_tc_pair_min_nt)) {
    // x tile split across the two SMs of a CTA pair: fewer bytes into each SM.
    // Measured (ncu, 14336-row expert): T = 512 up GEMM 153 -> 141 us, T = 256
    // expert 134 -> 129 us; with x read by the TMA map directly, 64 / 128-token
    // tiles -3.5 / -4.6 %, 16-token tiles -5 % (60 vs 63 us device span;
    // profiles/r2/tc_pair_small_ab.txt).
    CUtensorMap txh;
    SP_TRY(make_tmap(&txh, xt, M, T, xt_stride, tc::BK, nt / 2));
    if (L->d.gated)
      SP_TRY((launch_gemm_pair<2>(C, nt, tw1, tw3, txh, up, s, !x_direct)));
    else
      SP_TRY((launch_gemm_pair<1>(C, nt, tw1, tw1, txh, up, s, !x_direct)));
  } else if (L->d.gated) {
    SP_TRY((launch_gemm<2, false>(C, nt, tw1, tw3, tx, up, s, !x_direct)));
  } else {
    SP_TRY((launch_gemm<1, false>(C, nt, tw1, tw1, tx, up, s, !x_direct)));
  }
  if (up.ks > 1) {
    dim3 grid(unsigned((R / 4 + 127) / 128 + 1), unsigned(T));
    SP_CUDA(launch_k(tc::swiglu_reduce_kernel, grid, dim3(128), 0, s, true, static_cast<const float*>(up.z), up.ks,
                     na, T, int(R), up.zld, int(L->d.act), w.a_tc, w.ld_a));
    ++C->launches;
  }
  return launch_gemm<sub, true>(C, nt, tw2, tw2, ta, dn, s, true);
}

static FfnArgs ffn_args(Context* C, const sp_layer* L, const BlockView& b, const void* x, int xdtype,
                        int64_t ldx, const CallWs& w, int64_t T_e) {
  FfnArgs a{};
  a.w1t = b.base;
  a.w3t = L->d.gated ? b.base + b.w3_off : nullptr;
  a.w2 = b.base + b.w2_off;
  a.ldm = L->ldm;
  a.ldn = L->ldn;
  a.rows = int(b.rows);
  a.M = int(L->d.model_dim);
  a.N = int(L->d.out_dim);
  a.x = x;
  a.xdtype = xdtype;
  a.ldx = ldx;
  a.ids = w.ids;
  a.act = L->d.act;
  a.kt = int(round_up(L->d.model_dim, 256));
  const int vx = xdtype == SP_BF16 ? 8 : 4;
  const size_t esz_x = xdtype == SP_BF16 ? 2 : 4;
  a.xvec = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (ldx % vx == 0) &&
           ((size_t(ldx) * esz_x) % 16 == 0) && (L->d.model_dim % vx == 0);
  a.part = w.part;
  a.stamps = C->stamps;
  if (C->trace.kslot_cur >= 0) {
    a.kspan0 = C->trace.kspan + C->trace.kslot_cur;
    a.kspan1 = C->trace.kspan + kKSlots + C->trace.kslot_cur;
  }
  a.slice0 = w.S;
  a.slice_stride = T_e * L->d.out_dim;
  return a;
}

static void set_tokens(FfnArgs& a, const int32_t* host_ids, int64_t T_e, int t0, int n) {
  a.t0 = t0;
  a.T = n;
  for (int t = 0; t < 4; ++t) {
    const int64_t i = std::min<int64_t>(t0 + t, T_e - 1);
    a.tok[t] = host_ids ? host_ids[i] : int32_t(i);
  }
}

static int run_block(Context* C, const sp_layer* L, const BlockView& b, const void* x, int xdtype,
                     int64_t ldx, CallWs& w, const int32_t* host_ids, int64_t T_e, int t0, int T,
                     cudaStream_t s, int min_rows = g_min_rows_per_cta) {
  if (use_tc(L, T) && w.x_tc && w.a_tc)
    return run_block_tc(C, L, b, x, xdtype, ldx, w, w.ids, T_e, t0, T, s, min_rows == g_min_rows_per_cta);
  const int grid = block_grid(C, b.rows, min_rows);
  const int tt_max = max_token_tile(L->d.model_dim);
  if (tt_max == 0) return fail(SP_ERR_VALUE, "model_dim %lld exceeds the x tile", (long long)L->d.model_dim);
  FfnArgs a = ffn_args(C, L, b, x, xdtype, ldx, w, T_e);
  a.cta0 = 0;
  a.ncta = grid;
  for (int tb = 0; tb < T; tb += tt_max) {
    const int n = std::min(tt_max, T - tb);
    const int tt = n <= 1 ? 1 : n <= 2 ? 2 : 4;
    set_tokens(a, host_ids, T_e, t0 + tb, n);
    FfnGroup g{};
    g.a[0] = a;
    g.n = 1;
    SP_TRY(launch_group(C, L, tt, g, grid, s));
  }
  w.S += grid;
  return SP_OK;
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static cudaEvent_t trace_event(Context* C) {
  if (!C->trace.pool.empty()) {
    cudaEvent_t e = C->trace.pool.back();
    C->trace.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// GPU span bracketing the work enqueued on `s` between construction and end().
struct GpuSpan {
  Context* C;
  cudaStream_t s;
  Span sp;
  bool on;
  GpuSpan(Context* c, cudaStream_t st, int stream, int kind, double bytes)
      : C(c), s(st), on(c->trace.on && (!c->trace.gg_only || kind == SP_TRACE_GG)) {
    if (!on) return;
    sp.stream = stream;
    sp.kind = kind;
    sp.call = c->trace.call;
    sp.bytes = bytes;
    sp.a = trace_event(C);
    sp.b = trace_event(C);
    if (C->trace.kspan && (kind == SP_TRACE_GG || kind == SP_TRACE_CG || kind == SP_TRACE_CG_PRIME) &&
        C->trace.kspan_next < kKSlots) {
      sp.kslot = C->trace.kspan_next++;
      C->trace.kslot_cur = sp.kslot;
    }
    cudaEventRecord(sp.a, s);
  }
  void end() {
    if (!on) return;
    C->trace.kslot_cur = -1;
    cudaEventRecord(sp.b, s);
    std::lock_guard<std::mutex> g(C->trace_mu);
    C->trace.spans.push_back(sp);
    on = false;
  }
};

static void host_span(Context* C, int stream, int kind, double a, double b, double bytes) {
  if (!C->trace.on) return;
  Span sp;
  sp.stream = stream;
  sp.kind = kind;
  sp.call = C->trace.call;
  sp.bytes = bytes;
  sp.ha = a - C->trace.host_t0;
  sp.hb = b - C->trace.host_t0;
  std::lock_guard<std::mutex> g(C->trace_mu);
  C->trace.spans.push_back(sp);
}

static std::vector<HostChunk> host_cc_chunks(const sp_layer* L) {
  std::vector<HostChunk> hc(L->n_cc_chunks);
  for (int k = 0; k < L->n_cc_chunks; ++k) {
    const Chunk& ch = L->chunks[k];
    const char* base = static_cast<const char*>(L->host) + ch.off;
    hc[k] = HostChunk{base, L->d.gated ? base + ch.w3_off : nullptr, base + ch.w2_off, ch.r0, ch.rc};
  }
  return hc;
}

// one x row to fp32 [ldx] (zero padded); round: f32 x rounded to bf16 values
// (the caller's f32 x under SP_X_TO_BF16 -- what the GPU side sees)
static void gather_host_row(float* dst, int64_t ldx, const void* x, int xdtype, int64_t M, int64_t row,
                            bool round) {
  if (xdtype == SP_BF16) {
    const uint16_t* src = static_cast<const uint16_t*>(x) + row * M;
    for (int64_t k = 0; k < M; ++k) {
      const uint32_t u = uint32_t(src[k]) << 16;
      memcpy(&dst[k], &u, 4);
    }
  } else if (round) {
    const float* src = static_cast<const float*>(x) + row * M;
    for (int64_t k = 0; k < M; ++k) {
      uint32_t u;
      memcpy(&u, src + k, 4);
      u = ((u + 0x7fffu + ((u >> 16) & 1u)) >> 16) << 16;
      memcpy(&dst[k], &u, 4);
    }
  } else {
    memcpy(dst, static_cast<const float*>(x) + row * M, size_t(M) * 4);
  }
  for (int64_t k = M; k < ldx; ++k) dst[k] = 0.f;
}

// x rows of a call gathered to fp32 [T, ldx] (zero padded) for the host CC kernel
static void gather_host_x(float* xh, int64_t ldx, const void* x, int xdtype, int64_t M,
                          const int32_t* ids, int64_t T) {
  for (int64_t i = 0; i < T; ++i) {
    const int64_t row = ids ? ids[i] : i;
    if (xdtype == SP_BF16) {
      const uint16_t* src = static_cast<const uint16_t*>(x) + row * M;
      for (int64_t k = 0; k < M; ++k) {
        const uint32_t u = uint32_t(src[k]) << 16;
        memcpy(&xh[i * ldx + k], &u, 4);
      }
    } else {
      memcpy(&xh[i * ldx], static_cast<const float*>(x) + row * M, size_t(M) * 4);
    }
  }
}

static void cc_coordinator(Context* C) {
  // this thread may run a forward's tail (finalize launch, event records on the
  // library's streams), so it must be bound to the context's device: a fresh
  // host thread starts on device 0, and rank r of a multi-GPU job lives on r
  if (C->device >= 0) cudaSetDevice(C->device);
  std::unique_lock<std::mutex> lk(C->cc_mu);
  for (;;) {
    C->cc_cv.wait(lk, [&] { return C->cc_stop || (C->cc_pending && C->cc_job); });
    if (C->cc_stop) return;
    std::function<int()> job = std::move(C->cc_job);
    C->cc_job = nullptr;
    lk.unlock();
    int st = job();
    std::string err = st == SP_OK ? std::string() : g_err;
    lk.lock();
    C->cc_done = true;
    if (st == SP_OK && C->cc_tail) {
      // the launching thread finished enqueueing first: run its tail here
      std::function<int()> tail = std::move(C->cc_tail);
      C->cc_tail = nullptr;
      lk.unlock();
      st = tail();
      if (st != SP_OK) err = g_err;
      lk.lock();
    }
    C->cc_status = st;
    C->cc_error = err;
    C->cc_pending = false;
    C->cc_cv.notify_all();
  }
}

static void cc_submit(Context* C, std::function<int()> job) {
  std::lock_guard<std::mutex> g(C->cc_mu);
  C->cc_job = std::move(job);
  C->cc_tail = nullptr;
  C->cc_done = false;
  C->cc_pending = true;
  C->cc_status = SP_OK;
  C->cc_cv.notify_all();
}

// Join the CC block; `tail` (the work that needs its result) runs on the
// coordinator if the block is still running, else here.
static int cc_join_with_tail(Context* C, const std::function<int()>& tail) {
  std::unique_lock<std::mutex> lk(C->cc_mu);
  if (!C->cc_done) {
    C->cc_tail = tail;
    C->cc_cv.wait(lk, [&] { return !C->cc_pending; });
    if (C->cc_status != SP_OK) return fail(C->cc_status, "%s", C->cc_error.c_str());
    if (!C->cc_tail) return SP_OK;  // ran on the coordinator
    C->cc_tail = nullptr;
    lk.unlock();
    return tail();
  }
  C->cc_cv.wait(lk, [&] { return !C->cc_pending; });
  if (C->cc_status != SP_OK) return fail(C->cc_status, "%s", C->cc_error.c_str());
  lk.unlock();
  return tail();
}


// ---------------------------------------------------------------------------
// forward

// Error-path cleanup of forward_batch.  A forward that fails after submitting
// its CC block must not return while the coordinator still runs the job: the
// job reads the caller's calls / token ids / x and writes the pinned staging
// half, and a later cc_submit would reset the flags under it (a stale
// completion then satisfies the next forward's join).  So the destructor,
// while armed, drops any pending tail, waits for the coordinator to go idle
// and drains the library's streams (the pinned half's in-flight copies).
struct ErrorDrain {
  Context* C;
  bool armed = true;
  ~ErrorDrain() {
    if (!armed) return;
    {
      std::unique_lock<std::mutex> lk(C->cc_mu);
      C->cc_tail = nullptr;
      C->cc_cv.wait(lk, [&] { return !C->cc_pending; });
    }
    cudaStreamSynchronize(C->s_copy);
    cudaStreamSynchronize(C->s_comp);
    cudaStreamSynchronize(C->s_aux);
  }
};

// fp32 -> bf16 bit patterns, round to nearest even: u + 0x7fff + ((u >> 16) & 1),
// the same integer arithmetic as the Python fallback (NaNs are not special-cased).
// Native so host activations never go through a multi-threaded framework cast,
// whose spinning worker threads steal the cores the CC block runs on.
__attribute__((target("avx512f,avx512bw"))) static void round_bf16_avx512(const float* src, uint16_t* dst,
                                                                           int64_t n) {
  const __m512i bias = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1);
  int64_t i = 0;
  for (; i + 16 <= n; i += 16) {
    __m512i u = _mm512_castps_si512(_mm512_loadu_ps(src + i));
    u = _mm512_add_epi32(u, _mm512_add_epi32(bias, _mm512_and_si512(_mm512_srli_epi32(u, 16), one)));
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), _mm512_cvtepi32_epi16(_mm512_srli_epi32(u, 16)));
  }
  for (; i < n; ++i) {
    uint32_t u;
    memcpy(&u, src + i, 4);
    dst[i] = uint16_t((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
  }
}

static void round_bf16_host(const float* src, uint16_t* dst, int64_t n) {
  if (host_has_avx512()) return round_bf16_avx512(src, dst, n);
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, src + i, 4);
    dst[i] = uint16_t((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
  }
}

static int forward_batch(Context* C, const sp_call* calls, int n_calls, const void* x, int xdtype,
                         int64_t T, void* y, int ydtype, unsigned flags, cudaStream_t user,
                         const void* x_host_ready = nullptr) {
  // ---- validate everything before enqueuing anything ----
  if (n_calls < 1 || n_calls > kMaxCalls)
    return fail(SP_ERR_VALUE, "n_calls must lie in [1, %d], got %d", kMaxCalls, n_calls);
  if (T < 0) return fail(SP_ERR_SHAPE, "negative row count T=%lld", (long long)T);
  if ((xdtype != SP_F32 && xdtype != SP_BF16) || (ydtype != SP_F32 && ydtype != SP_BF16))
    return fail(SP_ERR_VALUE, "x/y dtype must be SP_F32 or SP_BF16");
  // SP_X_TO_BF16: the caller's f32 x is rounded into the bf16 staging copy; every
  // consumer (GPU upload, CC threads) then sees bf16 activations
  const bool stage_bf16 = (flags & SP_X_TO_BF16) && xdtype == SP_F32;
  if ((flags & SP_X_TO_BF16) && !(flags & SP_IO_HOST))
    return fail(SP_ERR_VALUE, "SP_X_TO_BF16 needs SP_IO_HOST");
  const void* x_src = x;
  if (stage_bf16) xdtype = SP_BF16;
  int64_t M = -1, N = -1;
  for (int c = 0; c < n_calls; ++c) {
    const sp_call& k = calls[c];
    if (!k.layer) return fail(SP_ERR_VALUE, "call %d has no layer", c);
    if (k.layer->device != C->device)
      return fail(SP_ERR_STATE, "call %d: layer lives on device %d, context is %d", c, k.layer->device,
                  C->device);
    if (M < 0) {
      M = k.layer->d.model_dim;
      N = k.layer->d.out_dim;
    } else if (M != k.layer->d.model_dim || N != k.layer->d.out_dim) {
      return fail(SP_ERR_SHAPE, "call %d: layer is %lldx%lld, batch expects %lldx%lld", c,
                  (long long)k.layer->d.model_dim, (long long)k.layer->d.out_dim, (long long)M,
                  (long long)N);
    }
    if (k.tokens < 0) return fail(SP_ERR_SHAPE, "call %d: negative token count", c);
    if (k.n_g < 0 || k.n_g > k.tokens)
      return fail(SP_ERR_TOKENS, "n_g must lie in [0, %lld], got %lld", (long long)k.tokens,
                  (long long)k.n_g);
    if (!k.token_ids && k.tokens > T)
      return fail(SP_ERR_SHAPE, "call %d covers %lld rows but x has %lld", c, (long long)k.tokens,
                  (long long)T);
    if (k.token_ids)
      for (int64_t i = 0; i < k.tokens; ++i)
        if (k.token_ids[i] < 0 || k.token_ids[i] >= T)
          return fail(SP_ERR_SHAPE, "call %d: token id %d outside [0, %lld)", c, k.token_ids[i],
                      (long long)T);
  }
  if (max_token_tile(M) == 0)
    return fail(SP_ERR_VALUE, "model_dim %lld exceeds the %d-float x tile", (long long)M, kMaxTileFloats);
  // no rows: nothing to compute (the reference returns an empty [0, N] output,
  // slicing_kernel.py:119); every call was checked to cover zero rows above
  if (T == 0) return SP_OK;
  const bool host_io = flags & SP_IO_HOST;
  const double t_call = now_s();

  // ---- workspace layout ----
  const size_t xel = xdtype == SP_BF16 ? 2 : 4, yel = ydtype == SP_BF16 ? 2 : 4;
  std::vector<CallWs> ws(n_calls);
  size_t dev_off = 0;
  auto dalloc = [&](size_t bytes) {
    const size_t o = dev_off;
    dev_off += size_t(round_up(int64_t(bytes), 256));
    return o;
  };
  std::vector<size_t> o_part(n_calls), o_ycc(n_calls), o_xtc(n_calls),
      o_atc(n_calls);
  std::vector<int64_t> ws_ld_a(n_calls);
  std::vector<int> ws_split(n_calls, 0);
  // Streamed chunks run on few, fat CTAs (they hide under their own copy), except
  // a call's last one: nothing is left to hide it and the step waits for it.
  std::vector<int> last_ci(n_calls, -1);
  for (int c = 0; c < n_calls; ++c)
    for (int ci = 0; ci < int(calls[c].layer->chunks.size()); ++ci)
      if (ci >= calls[c].layer->n_cc_chunks || calls[c].n_g > 0) last_ci[c] = ci;
  auto chunk_min_rows = [&](int c, int ci) { return ci == last_ci[c] && g_wide_last_chunk ? g_min_rows_per_cta : g_chunk_min_rows; };
  int64_t total_rows = 0;
  for (int c = 0; c < n_calls; ++c) {
    const sp_layer* L = calls[c].layer;
    const int64_t Te = calls[c].tokens;
    const bool tc_call = use_tc(L, Te);
    ws_split[c] = tc_call ? kTcMaxSplits : 0;
    int64_t slices = block_grid(C, L->h_gg) + 1 + ws_split[c];  // + tc accumulation slice + tc splits
    for (int ci = 0; ci < int(L->chunks.size()); ++ci)
      if (ci >= L->n_cc_chunks || calls[c].n_g > 0) slices += block_grid(C, L->chunks[ci].rc, chunk_min_rows(c, ci));
    o_part[c] = dalloc(size_t(slices) * Te * N * 4);
    const bool tc = tc_call;
    int64_t max_rows = L->h_gg;
    for (const Chunk& ch : L->chunks) max_rows = std::max(max_rows, ch.rc);
    ws_ld_a[c] = round_up(std::max<int64_t>(max_rows, 1), 64);
    o_xtc[c] = tc ? dalloc(size_t(Te) * L->ldm * 2) : SIZE_MAX;
    o_atc[c] = tc ? dalloc(size_t(Te) * ws_ld_a[c] * 2) : SIZE_MAX;
    o_ycc[c] = dalloc(size_t(Te) * N * 4);
    total_rows += Te;
  }
  // device metadata (dmeta[hb]): per call [token ids | gates] as the pinned
  // block, then the finalize CSR -- two copies
  const size_t meta_bytes = size_t(round_up(int64_t(total_rows) * 8, 256));
  const size_t csr_bytes = size_t(T + 1 + 3 * total_rows) * 4;
  const size_t o_xdev = dalloc(host_io ? size_t(T) * M * xel : 0);
  const size_t o_ydev = dalloc(host_io ? size_t(T) * N * yel : 0);
  SP_TRY(C->ws.ensure(dev_off, C->s_comp));
  // other streams touching ws (the aux stream's CC-partial copies) order after
  // this point: the (stream-ordered) allocation and the previous forward's finalize
  SP_CUDA(cudaEventRecord(C->ev_ws, C->s_comp));
  char* dws = static_cast<char*>(C->ws.p);
  const int hb = C->hpin_turn;
  C->hpin_turn ^= 1;
  if (C->hpin_used[hb]) SP_CUDA(cudaEventSynchronize(C->hpin_done[hb]));
  SP_TRY(C->dmeta[hb].ensure(meta_bytes + csr_bytes));
  char* const dmeta = static_cast<char*>(C->dmeta[hb].p);
  int64_t meta_off = 0;
  for (int c = 0; c < n_calls; ++c) {
    ws[c].part = reinterpret_cast<float*>(dws + o_part[c]);
    ws[c].S = 0;
    ws[c].ld_a = ws_ld_a[c];
    ws[c].split_capacity = ws_split[c];
    if (o_xtc[c] != SIZE_MAX) {
      ws[c].x_tc = reinterpret_cast<__nv_bfloat16*>(dws + o_xtc[c]);
      ws[c].a_tc = reinterpret_cast<__nv_bfloat16*>(dws + o_atc[c]);
    }
    ws[c].ycc = reinterpret_cast<float*>(dws + o_ycc[c]);
    ws[c].ids = reinterpret_cast<int32_t*>(dmeta + size_t(meta_off) * 8);
    ws[c].ids_identity = calls[c].token_ids == nullptr;
    ws[c].gates = reinterpret_cast<float*>(dmeta + size_t(meta_off) * 8 + size_t(calls[c].tokens) * 4);
    meta_off += calls[c].tokens;
  }

  // pinned staging: [meta (ids+gates) | x | ycc per call | y]
  size_t pin_off = 0;
  auto palloc = [&](size_t bytes) {
    const size_t o = pin_off;
    pin_off += size_t(round_up(int64_t(bytes), 256));
    return o;
  };
  const size_t p_meta = palloc(size_t(total_rows) * 8);
  const size_t p_csr = palloc(size_t(T + 1 + 3 * total_rows) * 4);
  const size_t p_x = palloc(size_t(T) * M * xel);
  std::vector<size_t> p_ycc(n_calls);
  for (int c = 0; c < n_calls; ++c) p_ycc[c] = palloc(size_t(calls[c].tokens) * N * 4);
  const size_t p_y = palloc(host_io ? size_t(T) * N * yel : 0);
  // Small host outputs are written by the finalize kernel straight into pinned
  // host memory (mapped, unified addressing): no read-back copy after it.
  const bool y_zero_copy = host_io && g_y_zero_copy && size_t(T) * N * yel <= kZeroCopyY;
  SP_TRY(C->hpin[hb].ensure(pin_off));
  char* hp = static_cast<char*>(C->hpin[hb].p);
  // Any error return from here on leaves no work behind: the CC job (which
  // reads this call's arguments and writes the pinned half) is joined and the
  // GPU work already enqueued (copies from the pinned half) is drained.
  ErrorDrain drain{C};

  // ---- stream ordering against the caller ----
  SP_CUDA(cudaEventRecord(C->ev_user, user));
  SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_user, 0));

  // ---- x (device copy for the GPU, host copy for the CC threads) and the CC
  // block, submitted to the coordinator: before the first chunk copies when x is
  // already on the host (the CC block is the decode step's long pole), else after
  bool need_cc = false;
  const void* x_dev = x;
  const void* x_host = nullptr;
  bool cc_async = false;
  bool cc_started = false;
  std::function<int()> cc_work;
  auto start_cc = [&]() -> int {
    cc_started = true;
    // ---- x: device copy for the GPU, host copy for the CC threads ----
    for (int c = 0; c < n_calls; ++c)
      need_cc |= calls[c].layer->d.b1 > 0 && calls[c].tokens - calls[c].n_g > 0;
    // host I/O: the CC threads read the caller's x directly (rounding it to bf16
    // values themselves under SP_X_TO_BF16), so the CC block is submitted before
    // this thread stages x for the GPU (a prompt's x is MBs)
    const bool x_round = host_io && stage_bf16;
    const int x_dtype_cc = x_round ? SP_F32 : xdtype;
    if (host_io) {
      x_host = x_round ? x_src : x;
    } else if (need_cc && x_host_ready) {
      x_host = x_host_ready;  // already read back by the caller (sp_moe_forward): no GPU wait
    } else if (need_cc) {
      // on the aux stream, ordered after the caller's work only: on the compute
      // stream it also waited for the previous forward's GPU tail, so
      // back-to-back prompt layers could not start their CC blocks early
      SP_CUDA(cudaStreamWaitEvent(C->s_aux, C->ev_user, 0));
      SP_CUDA(cudaMemcpyAsync(hp + p_x, x, size_t(T) * M * xel, cudaMemcpyDeviceToHost, C->s_aux));
      SP_CUDA(cudaEventRecord(C->ev_x, C->s_aux));
      x_host = hp + p_x;
    }

    // ---- CC block: submitted to the coordinator now, runs while we enqueue ----
    cc_async = need_cc && !(flags & SP_NO_CC_THREADS);
    const bool x_on_host_now = host_io || x_host_ready;
    const sp_cc_fn cc_fn = C->cc_fn;
    void* const cc_user = C->cc_user;
    cc_work = [=]() -> int {
      if (!x_on_host_now) {
        const cudaError_t e = cudaEventSynchronize(C->ev_x);
        if (e != cudaSuccess) return fail(SP_ERR_CUDA, "x copy for the CC block: %s", cudaGetErrorString(e));
      }
      // every call's CC block in one pass of the pool (one join per step, not two per expert)
      const double t_cc0 = now_s();
      static const bool cc_prof = env_int("SP_CC_PROF", 0) != 0;
      const int64_t ldx = round_up(M, kPadElems);
      int64_t rows = 0;
      double bytes = 0.0;
      for (int c = 0; c < n_calls; ++c)
        if (calls[c].layer->d.b1 > 0) rows += std::max<int64_t>(0, calls[c].tokens - calls[c].n_g);
      if (C->hscratch.size() < size_t(rows * ldx)) C->hscratch.resize(size_t(rows * ldx));
      // the CC rows of every call, gathered in parallel on the pool (rows -> (call, index))
      {
        std::vector<int> row_call(static_cast<size_t>(rows));
        std::vector<int64_t> row_idx(static_cast<size_t>(rows));
        int64_t r = 0;
        for (int c = 0; c < n_calls; ++c) {
          const int64_t Tcc = calls[c].tokens - calls[c].n_g;
          if (calls[c].layer->d.b1 <= 0 || Tcc <= 0) continue;
          for (int64_t i = 0; i < Tcc; ++i, ++r) {
            row_call[size_t(r)] = c;
            row_idx[size_t(r)] = i;
          }
        }
        float* const xs0 = C->hscratch.data();
        auto gather = [&](int tid, int n) {
          for (int64_t q = rows * tid / n; q < rows * (tid + 1) / n; ++q) {
            const sp_call& k = calls[row_call[size_t(q)]];
            const int64_t i = row_idx[size_t(q)];
            gather_host_row(xs0 + size_t(q * ldx), ldx, x_host, x_dtype_cc, M, k.token_ids ? k.token_ids[i] : i,
                            x_round);
          }
        };
        const int gthreads = (flags & SP_NO_CC_THREADS) ? 1 : int(std::min<int64_t>(C->host_threads, rows / 8 + 1));
        if (gthreads > 1) C->pool->run(gthreads, gather);
        else gather(0, 1);
      }
      std::vector<std::vector<HostChunk>> hcs;
      std::vector<CCProblem> probs;
      hcs.reserve(size_t(n_calls));
      int64_t r0 = 0;
      for (int c = 0; c < n_calls; ++c) {
        const sp_layer* L = calls[c].layer;
        const int64_t Tcc = calls[c].tokens - calls[c].n_g;
        if (L->d.b1 <= 0 || Tcc <= 0) continue;
        float* xs = C->hscratch.data() + size_t(r0 * ldx);
        r0 += Tcc;
        hcs.push_back(host_cc_chunks(L));
        probs.push_back(CCProblem{L->d.wdtype, L->d.gated, L->d.act, M, N, L->ldm, L->ldn, hcs.back().data(),
                                  L->n_cc_chunks, L->d.b1, xs, ldx, Tcc, reinterpret_cast<float*>(hp + p_ycc[c])});
        if (g_cc_prepack && !cc_fn && cc_uses_amx(probs.back())) {
          // once per layer: W2 of the CC rows repacked for the AMX down phase (forwards
          // are serialised by the context lock, so no other CC job sees the layer now)
          sp_layer* Lm = const_cast<sp_layer*>(L);
          if (!Lm->w2_vnni) {
            const size_t elems = amx_w2_prepack_elems(probs.back());
            Lm->w2_vnni = static_cast<uint16_t*>(aligned_alloc(64, (elems * 2 + 63) / 64 * 64));
            if (Lm->w2_vnni) amx_prepack_w2(probs.back(), Lm->w2_vnni, *C->pool, C->host_threads);
          }
          probs.back().w2p = Lm->w2_vnni;
        }
        bytes += double(L->cc_bytes);
      }
      const int cc_threads = (flags & SP_NO_CC_THREADS) ? 1 : C->host_threads;
      const double t_prep = now_s();
      if (cc_fn) {
        // the caller's CC code (e.g. the reference's numpy forward) on this thread
        int k = 0;
        for (int c = 0; c < n_calls; ++c) {
          const sp_layer* L = calls[c].layer;
          const int64_t Tcc = calls[c].tokens - calls[c].n_g;
          if (L->d.b1 <= 0 || Tcc <= 0) continue;
          const CCProblem& pr = probs[size_t(k++)];
          if (cc_fn(cc_user, const_cast<sp_layer*>(L), pr.x, pr.ldx, Tcc, pr.y, N) != 0)
            return fail(SP_ERR_VALUE, "the CC executor failed on call %d", c);
        }
      } else if (g_cc_batch) {
        cc_forward_batch(probs.data(), int(probs.size()), *C->pool, cc_threads);
      } else {
        for (const CCProblem& pr : probs) cc_forward(pr, *C->pool, cc_threads);
      }
      host_span(C, 3, SP_TRACE_CC, t_cc0, now_s(), bytes);
      if (cc_prof)
        fprintf(stderr, "[cc] rows %lld  start %.0f us after the call  prep %.0f us  compute %.0f us\n",
                (long long)rows, (t_cc0 - t_call) * 1e6, (t_prep - t_cc0) * 1e6, (now_s() - t_prep) * 1e6);
      return SP_OK;
    };
    if (cc_async) cc_submit(C, cc_work);
    return SP_OK;
  };
  // host I/O: x for the GPU, staged into pinned memory (rounded to bf16 under
  // SP_X_TO_BF16) and copied.  Done once the ring's first chunk copies are
  // queued: a prompt's x is MBs, and staging it first kept the link idle ~1 ms.
  bool x_dev_staged = !host_io;
  auto stage_x_dev = [&]() -> int {
    if (x_dev_staged) return SP_OK;
    x_dev_staged = true;
    if (stage_bf16)
      round_bf16_host(static_cast<const float*>(x_src), reinterpret_cast<uint16_t*>(hp + p_x), T * M);
    else
      memcpy(hp + p_x, x, size_t(T) * M * xel);
    // on the copy stream, in line with the chunk copies (an H2D issued on the
    // compute stream was observed to land only behind the ring's copies)
    SP_CUDA(cudaStreamWaitEvent(C->s_copy, C->ev_ws, 0));
    SP_CUDA(cudaMemcpyAsync(dws + o_xdev, hp + p_x, size_t(T) * M * xel, cudaMemcpyHostToDevice, C->s_copy));
    SP_CUDA(cudaEventRecord(C->ev_x, C->s_copy));
    SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_x, 0));
    x_dev = dws + o_xdev;
    return SP_OK;
  };
  const bool cc_early = g_cc_first && (host_io || x_host_ready);
  if (cc_early) SP_TRY(start_cc());
  // test hook: a forward of exactly SP_TEST_FAIL_AFTER_CC tokens fails here, after
  // its CC block went to the coordinator (tests/test_runtime_robustness.py)
  if (g_test_fail_after_cc > 0 && T == g_test_fail_after_cc)
    return fail(SP_ERR_VALUE, "injected failure after the CC submit (SP_TEST_FAIL_AFTER_CC)");

  // ---- CG chunks (and CC chunks for the n_g diverted rows): the copy stream
  // is the step's bottleneck, so the first ring slots' copies are enqueued
  // before anything else; each later copy right after the kernel that frees its slot.
  struct StreamItem {
    int c;
    int ci;
    int slot;
  };
  std::vector<StreamItem> items;
  for (int c = 0; c < n_calls; ++c) {
    const sp_layer* L = calls[c].layer;
    if (calls[c].tokens == 0) continue;
    for (int ci = 0; ci < int(L->chunks.size()); ++ci)
      if (ci >= L->n_cc_chunks || calls[c].n_g > 0) items.push_back(StreamItem{c, ci, -1});
  }
  size_t next_copy = 0;
  const int ring_slots = items.size() >= kLongStream ? g_ring_slots_long : g_ring_slots;
  auto enqueue_copy = [&]() -> int {
    StreamItem& it = items[next_copy++];
    const sp_layer* L = calls[it.c].layer;
    const Chunk& ch = L->chunks[size_t(it.ci)];
    it.slot = C->ring_next % ring_slots;
    C->ring_next = (it.slot + 1) % ring_slots;
    SP_CUDA(cudaStreamWaitEvent(C->s_copy, C->ev_free[it.slot], 0));
    {
      GpuSpan span(C, C->s_copy, 1, SP_TRACE_COPY, double(ch.bytes));
      SP_CUDA(cudaMemcpyAsync(C->ring[it.slot].p, static_cast<const char*>(L->host) + ch.off, ch.bytes,
                              cudaMemcpyHostToDevice, C->s_copy));
      span.end();
    }
    C->h2d_bytes += ch.bytes;
    SP_CUDA(cudaEventRecord(C->ev_copied[it.slot], C->s_copy));
    return SP_OK;
  };

  // ---- plan metadata (token ids, gates) ----
  {
    char* m = hp + p_meta;
    size_t mo = 0;
    for (int c = 0; c < n_calls; ++c) {
      const int64_t Te = calls[c].tokens;
      int32_t* ids = reinterpret_cast<int32_t*>(m + mo);
      float* g = reinterpret_cast<float*>(m + mo + Te * 4);
      for (int64_t i = 0; i < Te; ++i) {
        ids[i] = calls[c].token_ids ? calls[c].token_ids[i] : int32_t(i);
        g[i] = calls[c].gates ? calls[c].gates[i] : 1.0f;
      }
      mo += Te * 8;
    }
  }

  // ---- output-row CSR for finalize: entries (call, row, gate) of every token, in call order ----
  {
    int32_t* cs = reinterpret_cast<int32_t*>(hp + p_csr);
    int32_t* ccall = cs + (T + 1);
    int32_t* crow = ccall + total_rows;
    float* cgate = reinterpret_cast<float*>(crow + total_rows);
    std::vector<int32_t> count(size_t(T) + 1, 0);
    for (int c = 0; c < n_calls; ++c)
      for (int64_t i = 0; i < calls[c].tokens; ++i) ++count[size_t(calls[c].token_ids ? calls[c].token_ids[i] : i)];
    cs[0] = 0;
    for (int64_t t = 0; t < T; ++t) cs[t + 1] = cs[t] + count[size_t(t)];
    std::vector<int32_t> fill(cs, cs + T);
    for (int c = 0; c < n_calls; ++c)
      for (int64_t i = 0; i < calls[c].tokens; ++i) {
        const int64_t t = calls[c].token_ids ? calls[c].token_ids[i] : i;
        const int32_t slot = fill[size_t(t)]++;
        ccall[slot] = c;
        crow[slot] = int32_t(i);
        cgate[slot] = calls[c].gates ? calls[c].gates[i] : 1.0f;
      }
    // both metadata blocks on the copy stream, ahead of the chunk copies: small
    // H2D copies on the compute stream were observed to land only behind the
    // ring's copies, holding the step's first kernels (~0.9 ms at 6 slots)
    if (total_rows > 0)
      SP_CUDA(cudaMemcpyAsync(dmeta, hp + p_meta, size_t(total_rows) * 8, cudaMemcpyHostToDevice, C->s_copy));
    SP_CUDA(cudaMemcpyAsync(dmeta + meta_bytes, cs, csr_bytes, cudaMemcpyHostToDevice, C->s_copy));
    SP_CUDA(cudaEventRecord(C->ev_meta, C->s_copy));
    SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_meta, 0));
  }

  // x only on the device: its read-back for the CC block goes ahead of the ring
  // copies (behind them it waited for all of them: ~0.9 ms for a prompt's CC block)
  if (!cc_started) SP_TRY(start_cc());

  // the first ring slots' copies go right behind the (tiny) metadata copies.
  // A small host x is staged and copied first: its H2D queued behind the ring's
  // copies would hold every GG block and chunk kernel for their whole duration
  // (~0.9 ms); a prompt's x (MBs, ~1 ms of staging) goes behind them instead.
  static const bool launch_prof = env_int("SP_LAUNCH_PROF", 0) != 0;
  double lp[6] = {now_s(), 0, 0, 0, 0, 0};
  if (size_t(T) * M * 2 <= (size_t(1) << 20)) SP_TRY(stage_x_dev());
  while (next_copy < items.size() && next_copy < size_t(ring_slots)) SP_TRY(enqueue_copy());
  SP_TRY(stage_x_dev());
  lp[1] = now_s();

  // ---- GG blocks (HBM resident): the decode-size calls share one grouped launch ----
  // GG work is off the critical path (the copy stream paces the step), but it
  // shares the compute stream with the chunk kernels, and a chunk kernel that
  // waits behind it frees its ring slot late and stalls the copies.  So the GG
  // work is cut into jobs: the grouped launch goes first (queued behind the
  // first chunk copy), every other GG block is slotted in after a chunk kernel,
  // into the compute stream's idle time while the next copy is in flight.
  std::vector<std::function<int()>> gg_jobs;
  bool has_group = false;
  {
    const int tt_max = max_token_tile(M);
    std::vector<int> group;
    std::vector<int> singles;
    for (int c = 0; c < n_calls; ++c) {
      const sp_layer* L = calls[c].layer;
      const int Te = int(calls[c].tokens);
      if (Te == 0 || L->h_gg <= 0) continue;
      const bool tc = use_tc(L, Te);
      const sp_layer* L0 = group.empty() ? L : calls[group[0]].layer;
      const bool same = L->d.wdtype == L0->d.wdtype && L->d.gated == L0->d.gated && L->d.act == L0->d.act;
      if (!tc && Te <= tt_max && same && int(group.size()) < kMaxGroup) group.push_back(c);
      else singles.push_back(c);
    }
    if (!group.empty()) {
      has_group = true;
      // CTAs proportional to each block's rows, one wave over the SMs
      int64_t rows_total = 0;
      double bytes = 0;
      int te_max = 1;
      for (int c : group) {
        rows_total += calls[c].layer->h_gg;
        bytes += double(calls[c].layer->gg_bytes);
        te_max = std::max(te_max, int(calls[c].tokens));
      }
      FfnGroup g{};
      int cta = 0;
      for (int c : group) {
        const sp_layer* L = calls[c].layer;
        const int Te = int(calls[c].tokens);
        int nc = int(double(C->num_sms) * double(L->h_gg) / double(rows_total));
        nc = std::max(1, std::min(nc, block_grid(C, L->h_gg)));
        // many experts in one group: more CTAs than SMs rather than too many rows per CTA
        const int64_t cap = max_rows_per_cta(M, L->d.gated, te_max <= 1 ? 1 : te_max <= 2 ? 2 : 4,
                                             xdtype == SP_BF16 ? 2 : 4);
        nc = std::min(std::max<int>(nc, int((L->h_gg + cap - 1) / cap)), block_grid(C, L->h_gg));
        BlockView b{static_cast<const char*>(L->gg), L->gg_w3_off, L->gg_w2_off, L->h_gg};
        FfnArgs a = ffn_args(C, L, b, x_dev, xdtype, M, ws[c], Te);
        set_tokens(a, calls[c].token_ids, Te, 0, Te);
        a.cta0 = cta;
        a.ncta = nc;
        g.a[g.n++] = a;
        cta += nc;
        ws[c].S += nc;
      }
      const int tt = te_max <= 1 ? 1 : te_max <= 2 ? 2 : 4;
      const sp_layer* L0 = calls[group[0]].layer;
      gg_jobs.push_back([&, g, cta, tt, bytes, L0]() mutable -> int {
        // queued behind the first chunk copy: the GPU starts it from a full
        // queue (no host-enqueue bubble inside its span)
        if (!items.empty()) SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_copied[items[0].slot], 0));
        GpuSpan span(C, C->s_comp, 2, SP_TRACE_GG, bytes);
        if (C->trace.kslot_cur >= 0)
          for (int i = 0; i < g.n; ++i) {
            g.a[i].kspan0 = C->trace.kspan + C->trace.kslot_cur;
            g.a[i].kspan1 = C->trace.kspan + kKSlots + C->trace.kslot_cur;
          }
        SP_TRY(launch_group(C, L0, tt, g, cta, C->s_comp));
        span.end();
        return SP_OK;
      });
    }
    for (int c : singles) {
      gg_jobs.push_back([&, c, tt_max]() -> int {
        const sp_layer* L = calls[c].layer;
        const int Te = int(calls[c].tokens);
        const bool tc = use_tc(L, Te);
        BlockView b{static_cast<const char*>(L->gg), L->gg_w3_off, L->gg_w2_off, L->h_gg};
        // weight bytes streamed: once on the tensor-core path, once per token tile otherwise
        const double passes = tc ? 1.0 : double((Te + tt_max - 1) / tt_max);
        GpuSpan span(C, C->s_comp, 2, SP_TRACE_GG, double(L->gg_bytes) * passes);
        SP_TRY(run_block(C, L, b, x_dev, xdtype, M, ws[c], calls[c].token_ids, Te, 0, Te, C->s_comp));
        span.end();
        return SP_OK;
      });
    }
  }
  size_t next_gg = 0;
  // the grouped GG launch is held back until every chunk copy is queued
  // (SP_GG_LAST, see g_gg_last)
  std::function<int()> gg_group_last;
  if (g_gg_last && has_group && !items.empty()) gg_group_last = std::move(gg_jobs[next_gg++]);
  lp[2] = now_s();
  if (next_gg < gg_jobs.size()) SP_TRY(gg_jobs[next_gg++]());
  lp[3] = now_s();
  if (items.empty())
    while (next_gg < gg_jobs.size()) SP_TRY(gg_jobs[next_gg++]());

  // ---- chunk kernels, in copy order, each followed by the copy its slot frees ----
  for (size_t i = 0; i < items.size(); ++i) {
    const StreamItem it = items[i];
    const int c = it.c;
    const sp_layer* L = calls[c].layer;
    const int Te = int(calls[c].tokens);
    const int ng = int(calls[c].n_g);
    const Chunk& ch = L->chunks[size_t(it.ci)];
    const bool is_cc = it.ci < L->n_cc_chunks;
    SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_copied[it.slot], 0));
    BlockView b{static_cast<const char*>(C->ring[it.slot].p), ch.w3_off, ch.w2_off, ch.rc};
    const int t0 = is_cc ? Te - ng : 0;
    if (t0 > 0) {
      // a cg_prime block writes only rows [t0, Te) of its slices; the reducer sums every row
      const size_t slice = size_t(Te) * N * 4;
      SP_CUDA(cudaMemsetAsync(ws[c].part + size_t(ws[c].S) * Te * N, 0,
                              slice * block_grid(C, ch.rc, chunk_min_rows(c, it.ci)), C->s_comp));
    }
    {
      GpuSpan span(C, C->s_comp, 2, is_cc ? SP_TRACE_CG_PRIME : SP_TRACE_CG, double(ch.bytes));
      SP_TRY(run_block(C, L, b, x_dev, xdtype, M, ws[c], calls[c].token_ids, Te, t0, Te - t0, C->s_comp,
                       chunk_min_rows(c, it.ci)));
      span.end();
    }
    SP_CUDA(cudaEventRecord(C->ev_free[it.slot], C->s_comp));
    if (i == 0) lp[4] = now_s();
    if (next_copy < items.size()) SP_TRY(enqueue_copy());
    if (gg_group_last && g_gg_last == 1 && next_copy == items.size()) {
      SP_TRY(gg_group_last());  // every copy queued: the group hides under the ones in flight
      gg_group_last = nullptr;
    }
    if (next_gg < gg_jobs.size()) SP_TRY(gg_jobs[next_gg++]());  // into the wait for the next copy
  }
  while (next_gg < gg_jobs.size()) SP_TRY(gg_jobs[next_gg++]());
  if (gg_group_last) SP_TRY(gg_group_last());

  const double t_enq_done = now_s();
  if (launch_prof)
    fprintf(stderr, "[launch] T %lld calls %d items %zu gg_jobs %zu | metadata+cc %.0f  ring copies %.0f  gg build %.0f  "
            "first gg job %.0f  first chunk %.0f  rest %.0f us\n", (long long)T, n_calls, items.size(), gg_jobs.size(),
            (lp[0] - t_call) * 1e6, (lp[1] - lp[0]) * 1e6, (lp[2] - lp[1]) * 1e6, (lp[3] - lp[2]) * 1e6,
            (lp[4] > 0 ? lp[4] - lp[3] : 0) * 1e6, (t_enq_done - (lp[4] > 0 ? lp[4] : lp[3])) * 1e6);
  host_span(C, 0, SP_TRACE_LAUNCH, t_call, t_enq_done, 0.0);

  // ---- finalize: reduce slices + CC partials + gates + cast ----
  // Small CC partials are read by finalize_kernel straight from pinned host
  // memory (unified addressing, no copy launch on the critical path); large
  // ones (prompt blocks) are copied on the aux stream first.
  constexpr size_t kZeroCopyYcc = size_t(256) << 10;
  FinalArgs fa{};
  fa.T = int(T);
  fa.N = int(N);
  fa.out = y_zero_copy ? static_cast<void*>(hp + p_y) : host_io ? static_cast<void*>(dws + o_ydev) : y;
  fa.odtype = ydtype;
  {
    const int32_t* cs = reinterpret_cast<const int32_t*>(dmeta + meta_bytes);
    fa.entry_start = cs;
    fa.entry_call = cs + (T + 1);
    fa.entry_row = fa.entry_call + total_rows;
    fa.entry_gate = reinterpret_cast<const float*>(fa.entry_row + total_rows);
  }
  bool ycc_copy = false;
  // Host I/O with an output too big for the zero-copy path (a prompt): the CC
  // partials are added on the host to the read-back device output, so the GPU
  // finalize and the read-back run before the CC block ends and its MBs of
  // partials never cross the link (SP_HOST_MERGE=0: through the GPU finalize)
  const bool host_merge = g_host_merge && host_io && !y_zero_copy && ydtype == SP_F32 && need_cc && cc_async;
  for (int c = 0; c < n_calls; ++c) {
    const sp_layer* L = calls[c].layer;
    const int64_t Tcc = calls[c].tokens - calls[c].n_g;
    const bool has_cc = L->d.b1 > 0 && Tcc > 0;
    const bool zc = size_t(Tcc) * N * 4 <= kZeroCopyYcc;
    if (!host_merge) ycc_copy |= has_cc && !zc;
    const float* ycc = (!has_cc || host_merge) ? nullptr
                       : zc ? reinterpret_cast<const float*>(hp + p_ycc[c])
                            : ws[c].ycc;
    fa.c[c] = FinalCall{ws[c].part, ws[c].S, ycc, int(Tcc), int(calls[c].tokens)};
  }
  // The finalize waits for the host CC block: reduce the device partial slices
  // now, behind the call's last GPU block, so only the CC partial is left for it.
  if (need_cc && cc_async && g_prereduce && N % 4 == 0) {
    int64_t most = 0;
    for (int c = 0; c < n_calls; ++c)
      if (fa.c[c].S > 1) most = std::max<int64_t>(most, calls[c].tokens * N);
    if (most > 0) {
      dim3 grid(unsigned((most / 4 + kFinLanes - 1) / kFinLanes), unsigned(n_calls));
      reduce_slices_kernel<<<grid, kFinLanes * kFinGroups, 0, C->s_comp>>>(fa);
      SP_CUDA(cudaGetLastError());
      ++C->launches;
      for (int c = 0; c < n_calls; ++c) fa.c[c].S = std::min(fa.c[c].S, 1);
    }
  }
  int max_slices = 0;
  for (int c = 0; c < n_calls; ++c) max_slices = std::max(max_slices, fa.c[c].S);
  // The tail runs on whichever thread finishes last: this one (GPU work all
  // enqueued) or the CC coordinator (CC block done) -- so finalize is enqueued
  // the moment both are ready, without a thread wake-up in between.
  auto tail = [=]() -> int {
    if (ycc_copy) {
      // after ws's allocation and the previous forward's finalize (reads these buffers)
      SP_CUDA(cudaStreamWaitEvent(C->s_aux, C->ev_ws, 0));
      double ycc_bytes = 0.0;
      for (int c = 0; c < n_calls; ++c)
        if (fa.c[c].y_cc == ws[c].ycc) ycc_bytes += double(calls[c].tokens - calls[c].n_g) * N * 4;
      // the reference's separate Y_cc transfer (pipeline.py:367-383), measured on its own
      GpuSpan yspan(C, C->s_aux, 1, SP_TRACE_YCC, ycc_bytes);
      for (int c = 0; c < n_calls; ++c) {
        const int64_t Tcc = calls[c].tokens - calls[c].n_g;
        if (fa.c[c].y_cc != ws[c].ycc) continue;
        SP_CUDA(cudaMemcpyAsync(ws[c].ycc, hp + p_ycc[c], size_t(Tcc) * N * 4, cudaMemcpyHostToDevice,
                                C->s_aux));
      }
      yspan.end();
      SP_CUDA(cudaEventRecord(C->ev_ycc, C->s_aux));
      SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_ycc, 0));
    }
    GpuSpan span(C, C->s_comp, 2, SP_TRACE_MERGE, 0.0);
    if (N % 4 == 0 && reinterpret_cast<uintptr_t>(fa.out) % 16 == 0 && max_slices <= kFinRowsMaxSlices) {
      dim3 grid(unsigned((N / 4 + kFinRowsThreads - 1) / kFinRowsThreads), unsigned(T));
      finalize_rows_kernel<<<grid, kFinRowsThreads, 0, C->s_comp>>>(fa);
    } else if (N % 4 == 0 && reinterpret_cast<uintptr_t>(fa.out) % 16 == 0) {
      dim3 grid(unsigned((N + 4 * kFinLanes - 1) / (4 * kFinLanes)), unsigned(T));
      finalize_kernel<<<grid, kFinLanes * kFinGroups, 0, C->s_comp>>>(fa);
    } else {
      dim3 grid(unsigned(std::min<int64_t>((N + 255) / 256, 64)), unsigned(T));
      finalize_scalar_kernel<<<grid, 256, 0, C->s_comp>>>(fa);
    }
    SP_CUDA(cudaGetLastError());
    span.end();
    ++C->launches;
    if (host_io && !y_zero_copy)
      SP_CUDA(cudaMemcpyAsync(hp + p_y, dws + o_ydev, size_t(T) * N * yel, cudaMemcpyDeviceToHost, C->s_comp));
    else
      SP_CUDA(cudaEventRecord(C->ev_done, C->s_comp));
    SP_CUDA(cudaEventRecord(C->hpin_done[hb], C->s_comp));
    return SP_OK;
  };
  C->hpin_used[hb] = true;  // from here on the half's last GPU use is behind hpin_done[hb]
  if (need_cc && cc_async && host_merge) {
    SP_TRY(tail());  // the GPU finalize without the CC partials and the read-back, now
    SP_TRY(cc_join_with_tail(C, [] { return SP_OK; }));
  } else if (need_cc && cc_async) {
    SP_TRY(cc_join_with_tail(C, tail));
  } else {
    if (need_cc) SP_TRY(cc_work());
    SP_TRY(tail());
  }
  drain.armed = false;
  if (host_io) {
    SP_CUDA(cudaStreamSynchronize(C->s_comp));
    // a prompt's output is MBs, usually into a fresh (not yet faulted-in) array:
    // copy it out on the pool, in 64 KB-aligned shares
    const size_t ybytes = size_t(T) * N * yel;
    const int nt = ybytes >= (size_t(256) << 10) ? C->pool->size() : 1;
    if (host_merge) {
      // y[t] = device part[t] + sum over t's entries (call c, row i, gate) with a CC
      // row of gate * y_cc_c[i], entries in the host CSR's order
      const double t_m0 = now_s();
      const int32_t* cs = reinterpret_cast<const int32_t*>(hp + p_csr);
      const int32_t* ecall = cs + (T + 1);
      const int32_t* erow = ecall + total_rows;
      const float* egate = reinterpret_cast<const float*>(erow + total_rows);
      const float* ydev = reinterpret_cast<const float*>(hp + p_y);
      float* yout = static_cast<float*>(y);
      C->pool->run(nt, [&](int tid, int n) {
        for (int64_t t = T * tid / n; t < T * (tid + 1) / n; ++t) {
          float* dst = yout + t * N;
          memcpy(dst, ydev + t * N, size_t(N) * 4);
          for (int32_t e = cs[t]; e < cs[t + 1]; ++e) {
            const int c = ecall[e];
            const int64_t i = erow[e];
            if (calls[c].layer->d.b1 <= 0 || i >= calls[c].tokens - calls[c].n_g) continue;
            const float g = egate[e];
            const float* yc = reinterpret_cast<const float*>(hp + p_ycc[c]) + i * N;
            for (int64_t k = 0; k < N; ++k) dst[k] += g * yc[k];
          }
        }
      });
      host_span(C, 3, SP_TRACE_MERGE, t_m0, now_s(), double(ybytes));
    } else if (nt > 1) {
      C->pool->run(nt, [&](int tid, int n) {
        const size_t a = (ybytes * size_t(tid) / size_t(n)) & ~size_t(65535);
        const size_t b = tid + 1 == n ? ybytes : (ybytes * size_t(tid + 1) / size_t(n)) & ~size_t(65535);
        if (b > a) memcpy(static_cast<char*>(y) + a, hp + p_y + a, b - a);
      });
    } else {
      memcpy(y, hp + p_y, ybytes);
    }
  } else {
    SP_CUDA(cudaStreamWaitEvent(user, C->ev_done, 0));
  }
  host_span(C, 0, SP_TRACE_RETURN, t_enq_done, now_s(), 0.0);
  if (C->trace.on) ++C->trace.call;
  return SP_OK;
}



// ---------------------------------------------------------------------------
// MoE routing (host, fp64) and the one-call MoE layer

// logits[t, e] = sum_m x[t, m] * router[m, e] in fp64, m ascending, one
// multiply then one add per term -- the same IEEE operations whether the e loop
// is scalar or 8-wide (fp contraction off, so no FMA changes the rounding).
__attribute__((target("avx512f"), optimize("fp-contract=off"))) static void route_logits_avx512(
    const float* router, int64_t M, int E, const void* x, int xdtype, double* logit) {
  __m512d acc[8];
  const int nv = E / 8;
  for (int v = 0; v < nv; ++v) acc[v] = _mm512_setzero_pd();
  for (int64_t m = 0; m < M; ++m) {
    double xv;
    if (xdtype == SP_BF16) {
      const uint32_t u = uint32_t(static_cast<const uint16_t*>(x)[m]) << 16;
      float f;
      memcpy(&f, &u, 4);
      xv = f;
    } else {
      xv = static_cast<const float*>(x)[m];
    }
    const __m512d xb = _mm512_set1_pd(xv);
    const float* rrow = router + m * E;
    for (int v = 0; v < nv; ++v)
      acc[v] = _mm512_add_pd(acc[v], _mm512_mul_pd(xb, _mm512_cvtps_pd(_mm256_loadu_ps(rrow + 8 * v))));
  }
  for (int v = 0; v < nv; ++v) _mm512_storeu_pd(logit + 8 * v, acc[v]);
}

__attribute__((optimize("fp-contract=off"))) static void route_logits(const float* router, int64_t M, int E,
                                                                      const void* x, int xdtype, double* logit) {
  if (E % 8 == 0 && E <= 64 && host_has_avx512()) return route_logits_avx512(router, M, E, x, xdtype, logit);
  for (int e = 0; e < E; ++e) logit[e] = 0.0;
  for (int64_t m = 0; m < M; ++m) {
    double xv;
    if (xdtype == SP_BF16) {
      const uint32_t u = uint32_t(static_cast<const uint16_t*>(x)[m]) << 16;
      float f;
      memcpy(&f, &u, 4);
      xv = f;
    } else {
      xv = static_cast<const float*>(x)[m];
    }
    const float* rrow = router + m * E;
    for (int e = 0; e < E; ++e) logit[e] += xv * double(rrow[e]);
  }
}

// Tokens are independent (each logit is one serial m-ascending sum, ~8 us at
// M = 4096), so a batch is routed on the host pool when one is given (the caller
// holds the context lock): 32 tokens took ~0.3 ms on one thread, ahead of the
// CC block and the first copy.
static int moe_route(const float* router, int64_t M, int E, int k, const void* x, int xdtype, int64_t T,
                     int32_t* ids, float* gates, ThreadPool* pool = nullptr, int threads = 1) {
  if (E < 1 || k < 1 || k > E) return fail(SP_ERR_VALUE, "top_k must lie in [1, %d], got %d", E, k);
  const size_t xel = xdtype == SP_BF16 ? 2 : 4;
  auto route_range = [&](int64_t t0, int64_t t1) {
    std::vector<double> logit(static_cast<size_t>(E), 0.0);
    std::vector<int> order(static_cast<size_t>(E), 0);
    for (int64_t t = t0; t < t1; ++t) {
      route_logits(router, M, E, static_cast<const char*>(x) + size_t(t) * M * xel, xdtype, logit.data());
      for (int e = 0; e < E; ++e) order[e] = e;
      // k largest, ties to the lower expert id (a stable descending sort)
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return logit[a] > logit[b]; });
      const double top = logit[order[0]];
      double z = 0.0;
      for (int j = 0; j < k; ++j) z += std::exp(logit[order[j]] - top);
      for (int j = 0; j < k; ++j) {
        ids[t * k + j] = order[j];
        gates[t * k + j] = float(std::exp(logit[order[j]] - top) / z);
      }
    }
  };
  const int nt = pool && T >= 4 ? int(std::min<int64_t>(std::min(threads, pool->size()), T)) : 1;
  if (nt > 1)
    pool->run(nt, [&](int tid, int n) { route_range(T * tid / n, T * (tid + 1) / n); });
  else
    route_range(0, T);
  return SP_OK;
}

static int moe_forward(Context* C, const sp_layer_t* layers, int E, const float* router, int k, const void* x,
                       int xdtype, int64_t T, void* y, int ydtype, unsigned flags, cudaStream_t user) {
  if (!layers || !router) return fail(SP_ERR_VALUE, "NULL argument");
  if (T < 0) return fail(SP_ERR_SHAPE, "negative row count T=%lld", (long long)T);
  if (T == 0) return SP_OK;  // no tokens: nothing to route or compute
  if (!x || !y) return fail(SP_ERR_VALUE, "NULL argument");
  const sp_layer* any = nullptr;
  for (int e = 0; e < E; ++e)
    if (layers[e]) any = layers[e];
  if (!any) return fail(SP_ERR_VALUE, "sp_moe_forward: no expert layer on this rank");
  const int64_t M = any->d.model_dim;
  const size_t xel = xdtype == SP_BF16 ? 2 : 4;
  const bool host_io = flags & SP_IO_HOST;
  const double t_route0 = now_s();
  if ((flags & SP_X_TO_BF16) && host_io && xdtype == SP_F32) {
    // route on the rounded activations the experts will see
    SP_TRY(C->xroute.ensure(size_t(T) * M * 2));
    round_bf16_host(static_cast<const float*>(x), static_cast<uint16_t*>(C->xroute.p), T * M);
    x = C->xroute.p;
    xdtype = SP_BF16;
    flags &= ~SP_X_TO_BF16;
  }
  // one read of x serves the router and every CC block
  const void* xh = x;
  if (!host_io) {
    SP_TRY(C->xroute.ensure(size_t(T) * M * xel));
    SP_CUDA(cudaEventRecord(C->ev_user, user));
    SP_CUDA(cudaStreamWaitEvent(C->s_aux, C->ev_user, 0));
    SP_CUDA(cudaMemcpyAsync(C->xroute.p, x, size_t(T) * M * xel, cudaMemcpyDeviceToHost, C->s_aux));
    SP_CUDA(cudaStreamSynchronize(C->s_aux));
    xh = C->xroute.p;
    host_span(C, 0, SP_TRACE_ROUTE, t_route0, now_s(), double(size_t(T) * M * xel));  // x read-back
  }
  const double t_route1 = now_s();
  std::vector<int32_t> ids(static_cast<size_t>(T * k));
  std::vector<float> gates(static_cast<size_t>(T * k));
  SP_TRY(moe_route(router, M, E, k, xh, xdtype, T, ids.data(), gates.data(), C->pool.get(), C->host_threads));
  // group token rows by expert (ascending token order per expert)
  std::vector<std::vector<int32_t>> rows(static_cast<size_t>(E));
  std::vector<std::vector<float>> g(static_cast<size_t>(E));
  for (int64_t t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j) {
      const int e = ids[t * k + j];
      rows[e].push_back(int32_t(t));
      g[e].push_back(gates[t * k + j]);
    }
  std::vector<sp_call> calls;
  for (int e = 0; e < E; ++e)
    if (layers[e] && !rows[e].empty())
      calls.push_back(sp_call{layers[e], int64_t(rows[e].size()), rows[e].data(), g[e].data(), 0});
  if (calls.empty()) {
    // nothing routed to this rank's experts: y = 0
    const size_t bytes = size_t(T) * any->d.out_dim * (ydtype == SP_BF16 ? 2 : 4);
    if (host_io) {
      memset(y, 0, bytes);
      return SP_OK;
    }
    SP_CUDA(cudaMemsetAsync(y, 0, bytes, user));
    return SP_OK;
  }
  if (int(calls.size()) > kMaxCalls) return fail(SP_ERR_VALUE, "%zu active experts exceed %d", calls.size(), kMaxCalls);
  host_span(C, 0, SP_TRACE_ROUTE, t_route1, now_s(), 0.0);  // routing + grouping
  return forward_batch(C, calls.data(), int(calls.size()), x, xdtype, T, y, ydtype, flags, user,
                       host_io ? nullptr : xh);
}

}  // namespace sp

// ===========================================================================
// C ABI

using namespace sp;

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }

const char* sp_last_error(void) { return g_err.c_str(); }

int sp_device_count(int* count) {
  if (!count) return fail(SP_ERR_VALUE, "count is NULL");
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  *count = e == cudaSuccess ? n : 0;
  if (e != cudaSuccess) cudaGetLastError();
  return SP_OK;
}

int sp_init(int device, int host_threads) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if (g_ctx && g_ctx->device == device) return SP_OK;
  if (g_ctx) return fail(SP_ERR_STATE, "already initialised on device %d", g_ctx->device);
  const int hw = int(std::thread::hardware_concurrency());
  if (device < 0) {
    // host-only context: layers may hold CC/CG blocks in plain memory and only
    // sp_cc_forward_host runs; every GPU entry point refuses.
    auto C = std::make_unique<Context>();
    C->host_only = true;
    C->host_threads = host_threads > 0 ? host_threads : std::max(1, hw);
    C->pool = std::make_unique<ThreadPool>(C->host_threads);
    g_ctx = std::move(C);
    return SP_OK;
  }
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(SP_ERR_STATE, "no CUDA device visible; the GG/CG blocks have no CPU fallback");
  }
  if (device < 0 || device >= n) return fail(SP_ERR_VALUE, "device %d outside [0, %d)", device, n);
  SP_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(SP_ERR_STATE, "device %d is sm_%d%d; libsliced is built for sm_100a only", device,
                prop.major, prop.minor);
  auto C = std::make_unique<Context>();
  C->device = device;
  C->num_sms = prop.multiProcessorCount;
  SP_CUDA(cudaStreamCreateWithFlags(&C->s_comp, cudaStreamNonBlocking));
  SP_CUDA(cudaStreamCreateWithFlags(&C->s_copy, cudaStreamNonBlocking));
  SP_CUDA(cudaStreamCreateWithFlags(&C->s_aux, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&C->ev_user, &C->ev_x, &C->ev_ycc, &C->ev_done, &C->ev_ws, &C->ev_meta, &C->hpin_done[0],
                         &C->hpin_done[1]})
    SP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (int i = 0; i < kMaxRingSlots; ++i) {
    SP_CUDA(cudaEventCreateWithFlags(&C->ev_copied[i], cudaEventDisableTiming));
    SP_CUDA(cudaEventCreateWithFlags(&C->ev_free[i], cudaEventDisableTiming));
  }
  C->host_threads = host_threads > 0 ? host_threads : std::max(1, hw);
  C->pool = std::make_unique<ThreadPool>(C->host_threads);
  Context* raw = C.get();
  C->cc_thread = std::thread([raw] { cc_coordinator(raw); });
  SP_TRY(preload_kernels());
  if (env_int("SP_KSTAMPS", 0)) {
    SP_CUDA(cudaMalloc(&C->stamps, 4096 * 8 * sizeof(unsigned long long)));
    SP_CUDA(cudaMemset(C->stamps, 0, 4096 * 8 * sizeof(unsigned long long)));
  }
  g_ctx = std::move(C);
  return SP_OK;
}

int sp_shutdown(void) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if (!g_ctx) return SP_OK;
  Context* C = g_ctx.get();
  if (C->host_only) {
    g_ctx.reset();
    return SP_OK;
  }
  {
    std::lock_guard<std::mutex> lk(C->cc_mu);
    C->cc_stop = true;
    C->cc_cv.notify_all();
  }
  if (C->cc_thread.joinable()) C->cc_thread.join();
  cudaDeviceSynchronize();
  for (cudaEvent_t e : {C->ev_user, C->ev_x, C->ev_ycc, C->ev_done, C->ev_ws, C->ev_meta, C->hpin_done[0], C->hpin_done[1]})
    cudaEventDestroy(e);
  for (int i = 0; i < kMaxRingSlots; ++i) {
    cudaEventDestroy(C->ev_copied[i]);
    cudaEventDestroy(C->ev_free[i]);
  }
  cudaStreamDestroy(C->s_comp);
  cudaStreamDestroy(C->s_copy);
  cudaStreamDestroy(C->s_aux);
  g_ctx.reset();
  return SP_OK;
}

static int validate_desc(const sp_layer_desc& d) {
  if (d.model_dim < 1 || d.hidden_dim < 1 || d.out_dim < 1)
    return fail(SP_ERR_SHAPE, "layer dims must be >= 1 (M=%lld H=%lld N=%lld)", (long long)d.model_dim,
                (long long)d.hidden_dim, (long long)d.out_dim);
  if (d.model_dim > (1 << 30) || d.hidden_dim > (1 << 30) || d.out_dim > (1 << 30))
    return fail(SP_ERR_SHAPE, "layer dims too large");
  if (d.b1 < 0 || d.b2 < d.b1 || d.b2 > d.hidden_dim)
    return fail(SP_ERR_VALUE, "boundaries must satisfy 0 <= b1 <= b2 <= H (b1=%lld b2=%lld H=%lld)",
                (long long)d.b1, (long long)d.b2, (long long)d.hidden_dim);
  if (d.act < 0 || d.act > 2) return fail(SP_ERR_VALUE, "unknown activation %d", d.act);
  if (d.wdtype != SP_F32 && d.wdtype != SP_BF16) return fail(SP_ERR_VALUE, "unknown weight dtype");
  // the decode kernel's limits (include/sliced.h "Limits"), refused at creation
  // rather than at the first forward
  const int64_t max_n = int64_t(kMaxVec) * kConsumers * 32 * (d.wdtype == SP_BF16 ? 8 : 4);
  if (d.out_dim > max_n)
    return fail(SP_ERR_VALUE, "out_dim %lld exceeds %lld for %s weights", (long long)d.out_dim, (long long)max_n,
                d.wdtype == SP_BF16 ? "bf16" : "f32");
  if (max_token_tile(d.model_dim) == 0)
    return fail(SP_ERR_VALUE, "model_dim %lld exceeds the %d-float x tile", (long long)d.model_dim, kMaxTileFloats);
  return SP_OK;
}

static void free_layer_memory(sp_layer* L) {
  if (L->gg) cudaFree(L->gg);
  L->gg = nullptr;
  if (L->host && L->host_map_bytes) {
    cudaHostUnregister(L->host);
    munmap(L->host, L->host_map_bytes);
  } else if (L->host) {
    L->host_only ? free(L->host) : (void)cudaFreeHost(L->host);
  }
  L->host = nullptr;
  free(L->w2_vnni);
  L->w2_vnni = nullptr;
}

// Validate, then place an empty layer (caller holds C->mu).
static int new_layer(Context* C, const sp_layer_desc& d, std::unique_ptr<sp_layer>& L) {
  SP_TRY(validate_desc(d));
  L = std::make_unique<sp_layer>();
  L->d = d;
  L->device = C->device;
  L->esz = d.wdtype == SP_BF16 ? 2 : 4;
  L->ldm = round_up(d.model_dim, kPadElems);
  L->ldn = round_up(d.out_dim, kPadElems);
  L->host_only = C->host_only;
  const int st = place_layer(L.get());
  if (st != SP_OK) free_layer_memory(L.get());
  return st;
}

// Grow the staging ring for the layer's largest chunk, hand the layer out.
static int publish_layer(Context* C, std::unique_ptr<sp_layer>& L, sp_layer_t* out) {
  if (!C->host_only && L->max_chunk_bytes > C->ring_bytes) {
    SP_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < std::max(g_ring_slots, g_ring_slots_long); ++i) SP_TRY(C->ring[i].ensure(L->max_chunk_bytes));
    C->ring_bytes = C->ring[0].n;
  }
  *out = L.release();
  return SP_OK;
}

int sp_layer_create(const sp_layer_desc* desc, const void* w1t, const void* w3t, const void* w2,
                    sp_layer_t* out) {
  if (!desc || !out || !w1t || !w2) return fail(SP_ERR_VALUE, "NULL argument");
  if (desc->gated && !w3t) return fail(SP_ERR_VALUE, "gated layer needs w3t");
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  SP_TRY(bind_device(C));
  std::lock_guard<std::mutex> g(C->mu);
  std::unique_ptr<sp_layer> L;
  SP_TRY(new_layer(C, *desc, L));
  const int st = fill_rows(L.get(), w1t, desc->gated ? w3t : nullptr, w2);
  if (st != SP_OK) {
    free_layer_memory(L.get());
    return st;
  }
  return publish_layer(C, L, out);
}

int sp_layer_image_sizes(sp_layer_t L, size_t* gg_bytes, size_t* host_bytes, int32_t* chunk_rows) {
  if (!L) return fail(SP_ERR_VALUE, "NULL layer");
  if (gg_bytes) *gg_bytes = L->gg_bytes;
  if (host_bytes) *host_bytes = L->host_bytes;
  if (chunk_rows) *chunk_rows = L->d.chunk_rows;
  return SP_OK;
}

int sp_layer_export(sp_layer_t L, void* gg_dst, void* host_dst) {
  if (!L) return fail(SP_ERR_VALUE, "NULL layer");
  SP_TRY(bind_device(ctx_or_null()));
  if (gg_dst && L->gg_bytes) SP_CUDA(cudaMemcpy(gg_dst, L->gg, L->gg_bytes, cudaMemcpyDeviceToHost));
  if (host_dst && L->host_bytes) memcpy(host_dst, L->host, L->host_bytes);
  return SP_OK;
}

int sp_layer_create_from_images(const sp_layer_desc* desc, const void* gg_img, size_t gg_bytes,
                                const void* host_img, size_t host_bytes, sp_layer_t* out) {
  if (!desc || !out) return fail(SP_ERR_VALUE, "NULL argument");
  if (desc->chunk_rows <= 0) return fail(SP_ERR_VALUE, "images need the chunk_rows they were packed with");
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  SP_TRY(bind_device(C));
  std::lock_guard<std::mutex> g(C->mu);
  std::unique_ptr<sp_layer> L;
  SP_TRY(new_layer(C, *desc, L));
  int st = SP_OK;
  if (L->gg_bytes != gg_bytes || L->host_bytes != host_bytes || (gg_bytes && !gg_img) || (host_bytes && !host_img))
    st = fail(SP_ERR_SHAPE, "image sizes %zu/%zu do not match the layout %zu/%zu", gg_bytes, host_bytes,
              L->gg_bytes, L->host_bytes);
  if (st == SP_OK && gg_bytes && cudaMemcpy(L->gg, gg_img, gg_bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    st = fail(SP_ERR_CUDA, "GG image upload failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (st == SP_OK && host_bytes) memcpy(L->host, host_img, host_bytes);
  if (st != SP_OK) {
    free_layer_memory(L.get());
    return st;
  }
  return publish_layer(C, L, out);
}

static int pread_all(int fd, void* dst, size_t n, uint64_t off, const char* path) {
  char* p = static_cast<char*>(dst);
  while (n > 0) {
    const ssize_t r = pread(fd, p, std::min<size_t>(n, size_t(1) << 30), off_t(off));
    if (r <= 0) return fail(SP_ERR_VALUE, "short read from %s at offset %llu", path, (unsigned long long)off);
    p += r;
    off += uint64_t(r);
    n -= size_t(r);
  }
  return SP_OK;
}

int sp_layer_load_file(const sp_layer_desc* desc, const char* path, uint64_t gg_offset, size_t gg_bytes,
                       uint64_t host_offset, size_t host_bytes, sp_layer_t* out) {
  if (!desc || !path || !out) return fail(SP_ERR_VALUE, "NULL argument");
  if (desc->chunk_rows <= 0) return fail(SP_ERR_VALUE, "images need the chunk_rows they were packed with");
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  SP_TRY(bind_device(C));
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(SP_ERR_VALUE, "cannot open %s", path);
  std::lock_guard<std::mutex> g(C->mu);
  std::unique_ptr<sp_layer> L;
  int st = new_layer(C, *desc, L);
  if (st != SP_OK) {
    close(fd);
    return st;
  }
  if (L->gg_bytes != gg_bytes || L->host_bytes != host_bytes)
    st = fail(SP_ERR_SHAPE, "image sizes %zu/%zu do not match the layout %zu/%zu", gg_bytes, host_bytes,
              L->gg_bytes, L->host_bytes);
  // host region: straight into the pinned (copy-engine visible) memory
  if (st == SP_OK && host_bytes) st = pread_all(fd, L->host, host_bytes, host_offset, path);
  // GG block: through a pinned bounce buffer, 8 MB at a time
  if (st == SP_OK && gg_bytes) {
    const size_t step = size_t(8) << 20;
    void* bounce = nullptr;
    if (cudaHostAlloc(&bounce, step, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      st = fail(SP_ERR_NOMEM, "cudaHostAlloc(8 MB) bounce buffer failed");
    }
    for (size_t o = 0; st == SP_OK && o < gg_bytes; o += step) {
      const size_t n = std::min(step, gg_bytes - o);
      st = pread_all(fd, bounce, n, gg_offset + o, path);
      if (st == SP_OK && cudaMemcpy(static_cast<char*>(L->gg) + o, bounce, n, cudaMemcpyHostToDevice) != cudaSuccess)
        st = fail(SP_ERR_CUDA, "GG image upload failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    if (bounce) cudaFreeHost(bounce);
  }
  close(fd);
  if (st != SP_OK) {
    free_layer_memory(L.get());
    return st;
  }
  return publish_layer(C, L, out);
}

int sp_layer_reslice(sp_layer_t src, int64_t b1, int64_t b2, sp_layer_t* out) {
  if (!src || !out) return fail(SP_ERR_VALUE, "NULL argument");
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  SP_TRY(bind_device(C));
  std::lock_guard<std::mutex> g(C->mu);
  sp_layer_desc d = src->d;
  d.b1 = b1;
  d.b2 = b2;
  const int64_t H = d.hidden_dim, M = d.model_dim, N = d.out_dim;
  std::vector<char> w1(size_t(H * M) * src->esz), w3(d.gated ? size_t(H * M) * src->esz : 0),
      w2(size_t(H * N) * src->esz);
  SP_TRY(gather_rows(src, w1.data(), d.gated ? w3.data() : nullptr, w2.data()));
  std::unique_ptr<sp_layer> L;
  SP_TRY(new_layer(C, d, L));
  const int st = fill_rows(L.get(), w1.data(), d.gated ? w3.data() : nullptr, w2.data());
  if (st != SP_OK) {
    free_layer_memory(L.get());
    return st;
  }
  return publish_layer(C, L, out);
}
int sp_layer_destroy(sp_layer_t L) {
  if (!L) return SP_OK;
  Context* C = ctx_or_null();
  if (C && !C->host_only) {
    std::lock_guard<std::mutex> g(C->mu);
    bind_device(C);
    cudaStreamSynchronize(C->s_comp);
    cudaStreamSynchronize(C->s_copy);
  }
  free_layer_memory(L);
  delete L;
  return SP_OK;
}

int sp_layer_bytes(sp_layer_t L, size_t* gg, size_t* cg, size_t* cc) {
  if (!L) return fail(SP_ERR_VALUE, "NULL layer");
  if (gg) *gg = L->gg_bytes;
  if (cg) *cg = L->cg_bytes;
  if (cc) *cc = L->cc_bytes;
  return SP_OK;
}

int sp_layer_widths(sp_layer_t L, int64_t widths[3]) {
  if (!L || !widths) return fail(SP_ERR_VALUE, "NULL argument");
  widths[0] = L->d.b1;
  widths[1] = L->d.b2 - L->d.b1;
  widths[2] = L->d.hidden_dim - L->d.b2;
  return SP_OK;
}

int sp_forward_batch(const sp_call* calls, int n_calls, const void* x, int xdtype, int64_t T,
                     void* y, int ydtype, unsigned flags, void* stream) {
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  if (C->host_only)
    return fail(SP_ERR_STATE, "host-only context: the GG/CG blocks need a CUDA device (no CPU fallback)");
  // x / y may be NULL for an empty batch (an empty torch tensor has no storage)
  if (!calls || ((!x || !y) && T > 0)) return fail(SP_ERR_VALUE, "NULL argument");
  SP_TRY(bind_device(C));
  std::lock_guard<std::mutex> g(C->mu);
  return forward_batch(C, calls, n_calls, x, xdtype, T, y, ydtype, flags,
                       static_cast<cudaStream_t>(stream));
}

int sp_moe_route(const float* router, int64_t model_dim, int n_experts, int top_k, const void* x,
                 int xdtype, int64_t T, int32_t* ids, float* gates) {
  if (!router || !x || !ids || !gates) return fail(SP_ERR_VALUE, "NULL argument");
  if (model_dim < 1 || T < 0) return fail(SP_ERR_SHAPE, "bad router shape");
  return moe_route(router, model_dim, n_experts, top_k, x, xdtype, T, ids, gates);
}

int sp_moe_forward(const sp_layer_t* layers, int n_experts, const float* router, int top_k, const void* x,
                   int xdtype, int64_t T, void* y, int ydtype, unsigned flags, void* stream) {
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  if (C->host_only)
    return fail(SP_ERR_STATE, "host-only context: the GG/CG blocks need a CUDA device (no CPU fallback)");
  SP_TRY(bind_device(C));
  std::lock_guard<std::mutex> g(C->mu);
  return moe_forward(C, layers, n_experts, router, top_k, x, xdtype, T, y, ydtype, flags,
                     static_cast<cudaStream_t>(stream));
}

int sp_cc_forward_host(sp_layer_t L, const void* x, int xdtype, int64_t T, float* y_cc,
                       int threads) {
  if (!L || !x || !y_cc) return fail(SP_ERR_VALUE, "NULL argument");
  if (T < 0) return fail(SP_ERR_SHAPE, "negative token count");
  if (xdtype != SP_F32 && xdtype != SP_BF16) return fail(SP_ERR_VALUE, "x dtype must be SP_F32 or SP_BF16");
  const int64_t M = L->d.model_dim, N = L->d.out_dim;
  const int64_t ldx = round_up(M, kPadElems);
  std::vector<float> xh(size_t(T * ldx), 0.f);
  gather_host_x(xh.data(), ldx, x, xdtype, M, nullptr, T);
  std::vector<HostChunk> hc = host_cc_chunks(L);
  CCProblem pr{L->d.wdtype, L->d.gated, L->d.act, M, N, L->ldm, L->ldn, hc.data(), L->n_cc_chunks,
               L->d.b1, xh.data(), ldx, T, y_cc};
  Context* C = ctx_or_null();
  // the layer's prepacked W2 for the AMX down phase, as a forward's CC block uses
  // it (only under C->mu, like every other use of it)
  auto prepack = [&](ThreadPool& pool, int nthr) {
    if (!g_cc_prepack || !cc_uses_amx(pr)) return;
    if (!L->w2_vnni) {
      const size_t elems = amx_w2_prepack_elems(pr);
      L->w2_vnni = static_cast<uint16_t*>(aligned_alloc(64, (elems * 2 + 63) / 64 * 64));
      if (L->w2_vnni) amx_prepack_w2(pr, L->w2_vnni, pool, nthr);
    }
    pr.w2p = L->w2_vnni;
  };
  if (C && threads != 1) {
    // the pool is shared with forwards' CC blocks and ThreadPool::run is not
    // re-entrant: hold the context lock (a forward holds it until its CC join)
    std::lock_guard<std::mutex> g(C->mu);
    const int nthr = threads > 0 ? threads : C->host_threads;
    prepack(*C->pool, nthr);
    cc_forward(pr, *C->pool, nthr);
  } else {
    // unlocked: the layer's prepacked W2 (built and read under C->mu) is not touched
    ThreadPool local(std::max(1, threads));
    cc_forward(pr, local, std::max(1, threads));
  }
  return SP_OK;
}

int sp_round_bf16(const float* src, uint16_t* dst, int64_t n) {
  if (n < 0 || (n > 0 && (!src || !dst))) return fail(SP_ERR_VALUE, "NULL argument");
  round_bf16_host(src, dst, n);
  return SP_OK;
}

int sp_set_cc_executor(sp_cc_fn fn, void* user) {
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  std::lock_guard<std::mutex> g(C->mu);  // never while a forward is in flight
  C->cc_fn = fn;
  C->cc_user = fn ? user : nullptr;
  return SP_OK;
}

int sp_trace_enable(int on) {
  Context* C = ctx_or_null();
  if (!C || C->host_only) return fail(SP_ERR_STATE, "sp_init(device) has not been called");
  SP_TRY(bind_device(C));
  std::lock_guard<std::mutex> g(C->mu);
  Trace& tr = C->trace;
  SP_CUDA(cudaDeviceSynchronize());
  for (Span& sp : tr.spans) {
    if (sp.a) tr.pool.push_back(sp.a);
    if (sp.b) tr.pool.push_back(sp.b);
  }
  tr.spans.clear();
  tr.call = 0;
  tr.on = on != 0;
  tr.gg_only = on == 2;
  tr.kspan_next = 0;
  tr.kslot_cur = -1;
  if (tr.on) {
    // events for the spans of the traced region, created up front: cudaEventCreate
    // inside a forward costs microseconds per span on the launching thread
    while (tr.pool.size() < size_t(kTracePoolEvents)) {
      cudaEvent_t e = nullptr;
      SP_CUDA(cudaEventCreate(&e));
      tr.pool.push_back(e);
    }
    if (!tr.kspan) SP_CUDA(cudaMalloc(&tr.kspan, size_t(2) * kKSlots * sizeof(unsigned long long)));
    SP_CUDA(cudaMemset(tr.kspan, 0xff, size_t(kKSlots) * sizeof(unsigned long long)));
    SP_CUDA(cudaMemset(tr.kspan + kKSlots, 0, size_t(kKSlots) * sizeof(unsigned long long)));
    if (!tr.t0) SP_CUDA(cudaEventCreate(&tr.t0));
    SP_CUDA(cudaEventRecord(tr.t0, C->s_comp));
    SP_CUDA(cudaEventSynchronize(tr.t0));
    tr.host_t0 = now_s();
  }
  return SP_OK;
}

int sp_trace_fetch(sp_trace_record* out, int* n) {
  Context* C = ctx_or_null();
  if (!C || C->host_only) return fail(SP_ERR_STATE, "sp_init(device) has not been called");
  if (!n) return fail(SP_ERR_VALUE, "n is NULL");
  SP_TRY(bind_device(C));
  std::lock_guard<std::mutex> g(C->mu);
  Trace& tr = C->trace;
  const int have = int(tr.spans.size());
  if (!out) {
    *n = have;
    return SP_OK;
  }
  SP_CUDA(cudaDeviceSynchronize());
  const int k = std::min(*n, have);
  int counters[4] = {0, 0, 0, 0};
  std::vector<unsigned long long> ks;
  if (tr.kspan && tr.kspan_next > 0) {
    ks.resize(size_t(2) * kKSlots);
    SP_CUDA(cudaMemcpy(ks.data(), tr.kspan, ks.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  }
  for (int i = 0; i < k; ++i) {
    const Span& sp = tr.spans[i];
    sp_trace_record r{};
    r.index = ++counters[sp.stream & 3];
    r.stream = sp.stream;
    r.kind = sp.kind;
    r.call = sp.call;
    r.bytes = sp.bytes;
    if (sp.kslot >= 0 && !ks.empty()) {
      const unsigned long long k0 = ks[size_t(sp.kslot)], k1 = ks[size_t(kKSlots + sp.kslot)];
      r.dev_s = k1 > k0 ? double(k1 - k0) * 1e-9 : 0.0;
    }
    if (sp.a) {
      float ma = 0, mb = 0;
      SP_CUDA(cudaEventElapsedTime(&ma, tr.t0, sp.a));
      SP_CUDA(cudaEventElapsedTime(&mb, tr.t0, sp.b));
      r.start_s = ma * 1e-3;
      r.end_s = mb * 1e-3;
    } else {
      r.start_s = sp.ha;
      r.end_s = sp.hb;
    }
    out[i] = r;
  }
  *n = k;
  return SP_OK;
}

int sp_stats(uint64_t* kernel_launches, uint64_t* h2d_bytes) {
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  if (kernel_launches) *kernel_launches = C->launches;
  if (h2d_bytes) *h2d_bytes = C->h2d_bytes;
  return SP_OK;
}

// Internal (not in sliced.h): copy the last ffn_block launch's per-CTA stamps.
int sp_debug_stamps(unsigned long long* out, int n) {
  Context* C = ctx_or_null();
  if (!C || !C->stamps) return fail(SP_ERR_STATE, "stamps disabled (set SP_KSTAMPS=1)");
  SP_CUDA(cudaDeviceSynchronize());
  SP_CUDA(cudaMemcpy(out, C->stamps, size_t(std::min(n, 4096 * 8)) * 8, cudaMemcpyDeviceToHost));
  return SP_OK;
}

int sp_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return fail(SP_ERR_VALUE, "ptr is NULL");
  if (cudaHostAlloc(ptr, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return fail(SP_ERR_NOMEM, "cudaHostAlloc(%zu) failed", bytes);
  }
  return SP_OK;
}

int sp_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
  return SP_OK;
}

}  // extern "C"
