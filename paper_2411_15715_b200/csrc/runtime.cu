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
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sliced.h"
#include "host_cc.h"
#include "kernels.cuh"

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

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  int ensure(size_t bytes) {
    if (bytes <= n) return SP_OK;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    const size_t want = std::max(bytes, size_t(1) << 20);
    if (cudaMalloc(&p, want) != cudaSuccess) return fail(SP_ERR_NOMEM, "cudaMalloc(%zu) failed", want);
    n = want;
    return SP_OK;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t n = 0;
  int ensure(size_t bytes) {
    if (bytes <= n) return SP_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    const size_t want = std::max(bytes, size_t(1) << 16);
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess)
      return fail(SP_ERR_NOMEM, "cudaHostAlloc(%zu) failed", want);
    n = want;
    return SP_OK;
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

constexpr int kRingSlots = 3;

// Measured timeline: CUDA events on the library's streams (GPU spans) and the
// host clock (launch / CC spans), both relative to one synchronised origin.
struct Span {
  cudaEvent_t a = nullptr, b = nullptr;  // GPU span
  double ha = 0, hb = 0;                 // host span (seconds since host_t0)
  int stream, kind, call;
  double bytes;
};
struct Trace {
  bool on = false;
  cudaEvent_t t0 = nullptr;
  double host_t0 = 0;
  int call = 0;
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
};

struct Context {
  int device = -1;
  bool host_only = false;  // sp_init(-1): CC kernels only, for GPU-less hosts
  int num_sms = 0;
  cudaStream_t s_comp = nullptr, s_copy = nullptr, s_aux = nullptr;
  cudaEvent_t ev_user, ev_x, ev_ycc, ev_done;
  cudaEvent_t ev_copied[kRingSlots], ev_free[kRingSlots];
  DevBuf ring[kRingSlots];
  size_t ring_bytes = 0;
  int ring_next = 0;
  DevBuf ws;         // device workspace
  PinnedBuf hpin;    // pinned host staging (ids/gates, x, y_cc, y)
  std::vector<float> hscratch;
  std::unique_ptr<ThreadPool> pool;
  int host_threads = 1;
  std::mutex mu;
  Trace trace;
  std::map<std::pair<const void*, size_t>, int> occ_cache;
  uint64_t launches = 0, h2d_bytes = 0;
};

static std::mutex g_ctx_mu;
static std::unique_ptr<Context> g_ctx;

static Context* ctx_or_null() { return g_ctx.get(); }

// ---------------------------------------------------------------------------
// layer placement

struct Chunk {
  int64_t r0, rc, ldc;
  size_t off, bytes;       // within the pinned host region
  size_t w3_off, w2_off;   // offsets inside the chunk
  bool cc;
};

}  // namespace sp

struct sp_layer {
  sp_layer_desc d;
  int device;
  size_t esz;
  int64_t ldm;             // padded M
  // GG (HBM)
  int64_t h_gg, ld_gg;
  void* gg = nullptr;
  size_t gg_bytes = 0, gg_w3_off = 0, gg_w2_off = 0;
  // host region (pinned): CC chunks then CG chunks
  void* host = nullptr;
  size_t host_bytes = 0, cc_bytes = 0, cg_bytes = 0;
  std::vector<sp::Chunk> chunks;
  bool host_only = false;
  int n_cc_chunks = 0;
  size_t max_chunk_bytes = 0;
};

namespace sp {

static int pack_layer(sp_layer* L, const void* w1t, const void* w3t, const void* w2t) {
  const sp_layer_desc& d = L->d;
  const int64_t M = d.model_dim, H = d.hidden_dim, N = d.out_dim;
  const size_t esz = L->esz;
  const char* s1 = static_cast<const char*>(w1t);
  const char* s3 = static_cast<const char*>(w3t);
  const char* s2 = static_cast<const char*>(w2t);
  const int G = d.gated ? 2 : 1;

  // ---- GG block -> HBM: [W1t rows b2..H | W3t rows | W2t[:, b2:H]] ----
  L->h_gg = H - d.b2;
  L->ld_gg = round_up(std::max<int64_t>(L->h_gg, 1), kPadElems);
  if (L->h_gg > 0 && L->host_only)
    return fail(SP_ERR_STATE, "host-only context: a GG block (b2 < H) needs a CUDA device");
  if (L->h_gg > 0) {
    const size_t up = size_t(L->h_gg) * L->ldm * esz;
    L->gg_w3_off = up;
    L->gg_w2_off = up * G;
    L->gg_bytes = up * G + size_t(N) * L->ld_gg * esz;
    SP_CUDA(cudaMalloc(&L->gg, L->gg_bytes));
    SP_CUDA(cudaMemset(L->gg, 0, L->gg_bytes));
    char* g = static_cast<char*>(L->gg);
    SP_CUDA(cudaMemcpy2D(g, L->ldm * esz, s1 + size_t(d.b2) * M * esz, M * esz, M * esz, L->h_gg,
                         cudaMemcpyHostToDevice));
    if (G == 2)
      SP_CUDA(cudaMemcpy2D(g + L->gg_w3_off, L->ldm * esz, s3 + size_t(d.b2) * M * esz, M * esz,
                           M * esz, L->h_gg, cudaMemcpyHostToDevice));
    SP_CUDA(cudaMemcpy2D(g + L->gg_w2_off, L->ld_gg * esz, s2 + size_t(d.b2) * esz, H * esz,
                         L->h_gg * esz, N, cudaMemcpyHostToDevice));
  }

  // ---- CC and CG blocks -> pinned host, chunk-interleaved ----
  int64_t cr = d.chunk_rows;
  if (cr <= 0) {
    const int64_t row_bytes = (G * L->ldm + N) * int64_t(esz);
    cr = std::max<int64_t>(kPadElems, ((int64_t(8) << 20) / row_bytes) / kPadElems * kPadElems);
  }
  cr = round_up(cr, kPadElems);
  L->d.chunk_rows = int32_t(cr);
  size_t off = 0;
  auto add_segment = [&](int64_t lo, int64_t hi, bool cc) {
    for (int64_t r0 = lo; r0 < hi; r0 += cr) {
      Chunk c;
      c.r0 = r0;
      c.rc = std::min(cr, hi - r0);
      c.ldc = round_up(c.rc, kPadElems);
      c.cc = cc;
      const size_t up = size_t(c.rc) * L->ldm * esz;
      c.w3_off = up;
      c.w2_off = up * G;
      c.bytes = up * G + size_t(N) * c.ldc * esz;
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
    } else if (cudaHostAlloc(&L->host, off, cudaHostAllocDefault) != cudaSuccess) {
      return fail(SP_ERR_NOMEM, "cudaHostAlloc(%zu) for the CC/CG blocks failed", off);
    }
    memset(L->host, 0, off);
    char* h = static_cast<char*>(L->host);
    for (const Chunk& c : L->chunks) {
      char* base = h + c.off;
      for (int64_t r = 0; r < c.rc; ++r) {
        memcpy(base + size_t(r) * L->ldm * esz, s1 + size_t(c.r0 + r) * M * esz, M * esz);
        if (G == 2)
          memcpy(base + c.w3_off + size_t(r) * L->ldm * esz, s3 + size_t(c.r0 + r) * M * esz,
                 M * esz);
      }
      for (int64_t n = 0; n < N; ++n)
        memcpy(base + c.w2_off + size_t(n) * c.ldc * esz, s2 + (size_t(n) * H + c.r0) * esz,
               c.rc * esz);
    }
  }
  return SP_OK;
}

// ---------------------------------------------------------------------------
// kernel dispatch

template <typename WT, int TT, int MODE, int WPR>
static int launch_rowdot_t(Context* C, const RowDotArgs& a, cudaStream_t s) {
  auto kern = rowdot_kernel<WT, TT, MODE, WPR>;
  constexpr int G = MODE == kUpGated ? 2 : 1;
  static bool attr_set = false;
  if (!attr_set) {
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set = true;
  }
  // first guess of the grid: occupancy at the per-CTA accumulator size for 1 wave
  const size_t fixed = size_t(TT) * a.kt + 2 * kWarps * kRowGroup * G * TT;
  auto key = std::make_pair(reinterpret_cast<const void*>(kern), fixed);
  int occ;
  auto it = C->occ_cache.find(key);
  if (it == C->occ_cache.end()) {
    SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads,
                                                          (fixed + 64 * G * TT) * sizeof(float)));
    occ = std::max(1, std::min(occ, 4));
    C->occ_cache[key] = occ;
  } else {
    occ = it->second;
  }
  const int grid = std::max(1, std::min(a.rows, C->num_sms * occ));
  const int per_cta = (a.rows + grid - 1) / grid;
  const size_t smem = (fixed + size_t(per_cta) * G * TT) * sizeof(float);
  kern<<<grid, kThreads, smem, s>>>(a);
  SP_CUDA(cudaGetLastError());
  ++C->launches;
  return SP_OK;
}

template <typename WT, int TT, int MODE>
static int launch_wpr(Context* C, int wpr, const RowDotArgs& a, cudaStream_t s) {
  switch (wpr) {
    case 1: return launch_rowdot_t<WT, TT, MODE, 1>(C, a, s);
    case 4: return launch_rowdot_t<WT, TT, MODE, 4>(C, a, s);
    default: return launch_rowdot_t<WT, TT, MODE, 8>(C, a, s);
  }
}

template <typename WT, int MODE>
static int launch_tt(Context* C, int tt, int wpr, const RowDotArgs& a, cudaStream_t s) {
  switch (tt) {
    case 1: return launch_wpr<WT, 1, MODE>(C, wpr, a, s);
    case 2: return launch_wpr<WT, 2, MODE>(C, wpr, a, s);
    case 4: return launch_wpr<WT, 4, MODE>(C, wpr, a, s);
    default: return launch_wpr<WT, 8, MODE>(C, wpr, a, s);
  }
}

// Launches enough token blocks of <= 8 rows to cover tokens [t0, t0 + T).
static int rowdot(Context* C, int wdtype, int mode, RowDotArgs a, int t0, int T, cudaStream_t s) {
  if (a.rows <= 0 || T <= 0) return SP_OK;
  const int wpr = a.K > 4096 ? 8 : (a.K > 1024 ? 4 : 1);
  for (int tb = 0; tb < T; tb += 8) {
    const int n = std::min(8, T - tb);
    const int tt = n <= 1 ? 1 : n <= 2 ? 2 : n <= 4 ? 4 : 8;
    a.t0 = t0 + tb;
    a.T = n;
    a.kt = int(std::min<int64_t>(round_up(a.K, 256), (kMaxTileFloats / tt) / 256 * 256));
    int st;
    if (wdtype == SP_BF16) {
      st = mode == kUp ? launch_tt<__nv_bfloat16, kUp>(C, tt, wpr, a, s)
         : mode == kUpGated ? launch_tt<__nv_bfloat16, kUpGated>(C, tt, wpr, a, s)
                            : launch_tt<__nv_bfloat16, kDown>(C, tt, wpr, a, s);
    } else {
      st = mode == kUp ? launch_tt<float, kUp>(C, tt, wpr, a, s)
         : mode == kUpGated ? launch_tt<float, kUpGated>(C, tt, wpr, a, s)
                            : launch_tt<float, kDown>(C, tt, wpr, a, s);
    }
    SP_TRY(st);
  }
  return SP_OK;
}

// One weight block (GG or a streamed chunk) applied to tokens [t0, t0 + T) of a call:
//   a[:, col0 : col0 + rows] = act(W1t x) [* W3t x];   y += W2t a[:, col0 : ...]
struct BlockView {
  const char* base;    // W1t at base, W3t at base + w3_off, W2t at base + w2_off
  size_t w3_off, w2_off;
  int64_t rows, ldm, ldc, col0;
};

struct CallWs {
  float* a;      // [T_e, ldh]
  float* y;      // [T_e, N]
  float* ycc;    // [T_e, N]
  int32_t* ids;  // device
  float* gates;  // device
  int64_t ldh;
};

static int run_block(Context* C, const sp_layer* L, const BlockView& b, const void* x, int xdtype,
                     int64_t ldx, const CallWs& w, int t0, int T, bool accumulate, cudaStream_t s) {
  RowDotArgs up{};
  up.w0 = b.base;
  up.w1 = L->d.gated ? b.base + b.w3_off : nullptr;
  up.ldw = b.ldm;
  up.rows = int(b.rows);
  up.K = int(L->d.model_dim);
  up.x = x;
  up.xdtype = xdtype;
  up.ldx = ldx;
  up.xcol0 = 0;
  up.ids = w.ids;
  up.out = w.a;
  up.ldo = w.ldh;
  up.ocol0 = b.col0;
  up.act = L->d.act;
  SP_TRY(rowdot(C, L->d.wdtype, L->d.gated ? kUpGated : kUp, up, t0, T, s));

  RowDotArgs dn{};
  dn.w0 = b.base + b.w2_off;
  dn.ldw = b.ldc;
  dn.rows = int(L->d.out_dim);
  dn.K = int(b.rows);
  dn.x = w.a;
  dn.xdtype = 0;
  dn.ldx = w.ldh;
  dn.xcol0 = b.col0;
  dn.ids = nullptr;
  dn.out = w.y;
  dn.ldo = L->d.out_dim;
  dn.ocol0 = 0;
  dn.accumulate = accumulate ? 1 : 0;
  return rowdot(C, L->d.wdtype, kDown, dn, t0, T, s);
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

// GPU span bracketing the work enqueued on `s` between begin and end.
struct GpuSpan {
  Context* C;
  cudaStream_t s;
  Span sp;
  bool on;
  GpuSpan(Context* c, cudaStream_t st, int stream, int kind, double bytes)
      : C(c), s(st), on(c->trace.on) {
    if (!on) return;
    sp.stream = stream;
    sp.kind = kind;
    sp.call = c->trace.call;
    sp.bytes = bytes;
    sp.a = trace_event(C);
    sp.b = trace_event(C);
    cudaEventRecord(sp.a, s);
  }
  void end() {
    if (!on) return;
    cudaEventRecord(sp.b, s);
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
  C->trace.spans.push_back(sp);
}

// ---------------------------------------------------------------------------
// forward

static int forward_batch(Context* C, const sp_call* calls, int n_calls, const void* x, int xdtype,
                         int64_t T, void* y, int ydtype, unsigned flags, cudaStream_t user) {
  // ---- validate everything before enqueuing anything ----
  if (n_calls < 0 || n_calls > kMaxMergeCalls)
    return fail(SP_ERR_VALUE, "n_calls must lie in [0, %d], got %d", kMaxMergeCalls, n_calls);
  if (T < 1) return fail(SP_ERR_SHAPE, "input must have at least one row, got T=%lld", (long long)T);
  if ((xdtype != SP_F32 && xdtype != SP_BF16) || (ydtype != SP_F32 && ydtype != SP_BF16))
    return fail(SP_ERR_VALUE, "x/y dtype must be SP_F32 or SP_BF16");
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
  if (n_calls == 0) return fail(SP_ERR_VALUE, "sp_forward_batch needs at least one call");
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
  std::vector<size_t> o_a(n_calls), o_y(n_calls), o_ycc(n_calls), o_ids(n_calls), o_g(n_calls);
  int64_t total_rows = 0;
  for (int c = 0; c < n_calls; ++c) {
    const sp_layer* L = calls[c].layer;
    const int64_t Te = calls[c].tokens;
    ws[c].ldh = round_up(L->d.hidden_dim, kPadElems);
    o_a[c] = dalloc(size_t(Te) * ws[c].ldh * 4);
    o_y[c] = dalloc(size_t(Te) * N * 4);
    o_ycc[c] = dalloc(size_t(Te) * N * 4);
    o_ids[c] = dalloc(size_t(Te) * 4);
    o_g[c] = dalloc(size_t(Te) * 4);
    total_rows += Te;
  }
  const size_t o_acc = dalloc(size_t(T) * N * 4);
  const size_t o_xdev = dalloc(host_io ? size_t(T) * M * xel : 0);
  const size_t o_ydev = dalloc(host_io ? size_t(T) * N * yel : 0);
  SP_TRY(C->ws.ensure(dev_off));
  char* dws = static_cast<char*>(C->ws.p);
  for (int c = 0; c < n_calls; ++c) {
    ws[c].a = reinterpret_cast<float*>(dws + o_a[c]);
    ws[c].y = reinterpret_cast<float*>(dws + o_y[c]);
    ws[c].ycc = reinterpret_cast<float*>(dws + o_ycc[c]);
    ws[c].ids = reinterpret_cast<int32_t*>(dws + o_ids[c]);
    ws[c].gates = reinterpret_cast<float*>(dws + o_g[c]);
  }

  // pinned staging: [meta (ids+gates) | x | ycc per call | y]
  size_t pin_off = 0;
  auto palloc = [&](size_t bytes) {
    const size_t o = pin_off;
    pin_off += size_t(round_up(int64_t(bytes), 256));
    return o;
  };
  const size_t p_meta = palloc(size_t(total_rows) * 8);
  const size_t p_x = palloc(size_t(T) * M * xel);
  std::vector<size_t> p_ycc(n_calls);
  for (int c = 0; c < n_calls; ++c) p_ycc[c] = palloc(size_t(calls[c].tokens) * N * 4);
  const size_t p_y = palloc(host_io ? size_t(T) * N * yel : 0);
  SP_TRY(C->hpin.ensure(pin_off));
  char* hp = static_cast<char*>(C->hpin.p);

  // ---- stream ordering against the caller ----
  SP_CUDA(cudaEventRecord(C->ev_user, user));
  SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_user, 0));

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
      SP_CUDA(cudaMemcpyAsync(ws[c].ids, ids, Te * 4, cudaMemcpyHostToDevice, C->s_comp));
      SP_CUDA(cudaMemcpyAsync(ws[c].gates, g, Te * 4, cudaMemcpyHostToDevice, C->s_comp));
      mo += Te * 8;
    }
  }

  // ---- x: device copy for the GPU, host copy for the CC threads ----
  bool need_cc = false;
  for (int c = 0; c < n_calls; ++c)
    need_cc |= calls[c].layer->d.b1 > 0 && calls[c].tokens - calls[c].n_g > 0;
  const void* x_dev = x;
  const void* x_host = nullptr;
  if (host_io) {
    memcpy(hp + p_x, x, size_t(T) * M * xel);
    SP_CUDA(cudaMemcpyAsync(dws + o_xdev, hp + p_x, size_t(T) * M * xel, cudaMemcpyHostToDevice,
                            C->s_comp));
    x_dev = dws + o_xdev;
    x_host = x;
  } else if (need_cc) {
    SP_CUDA(cudaMemcpyAsync(hp + p_x, x, size_t(T) * M * xel, cudaMemcpyDeviceToHost, C->s_comp));
    SP_CUDA(cudaEventRecord(C->ev_x, C->s_comp));
    x_host = hp + p_x;
  }

  // ---- GG blocks (HBM resident) ----
  for (int c = 0; c < n_calls; ++c) {
    const sp_layer* L = calls[c].layer;
    const int Te = int(calls[c].tokens);
    if (Te == 0) continue;
    if (L->h_gg > 0) {
      BlockView b{static_cast<const char*>(L->gg), L->gg_w3_off, L->gg_w2_off, L->h_gg, L->ldm,
                  L->ld_gg, L->d.b2};
      GpuSpan span(C, C->s_comp, 2, SP_TRACE_GG, double(L->gg_bytes));
      SP_TRY(run_block(C, L, b, x_dev, xdtype, M, ws[c], 0, Te, false, C->s_comp));
      span.end();
    } else {
      SP_CUDA(cudaMemsetAsync(ws[c].y, 0, size_t(Te) * N * 4, C->s_comp));
    }
  }

  // ---- CG chunks (and CC chunks for the n_g diverted rows) through the ring ----
  int chunk_seq = 0;
  for (int c = 0; c < n_calls; ++c) {
    const sp_layer* L = calls[c].layer;
    const int Te = int(calls[c].tokens);
    const int ng = int(calls[c].n_g);
    if (Te == 0) continue;
    for (size_t ci = 0; ci < L->chunks.size(); ++ci) {
      const Chunk& ch = L->chunks[ci];
      const bool is_cc = int(ci) < L->n_cc_chunks;
      if (is_cc && ng == 0) continue;
      const int slot = C->ring_next;
      C->ring_next = (C->ring_next + 1) % kRingSlots;
      SP_CUDA(cudaStreamWaitEvent(C->s_copy, C->ev_free[slot], 0));
      {
        GpuSpan span(C, C->s_copy, 1, SP_TRACE_COPY, double(ch.bytes));
        SP_CUDA(cudaMemcpyAsync(C->ring[slot].p, static_cast<const char*>(L->host) + ch.off,
                                ch.bytes, cudaMemcpyHostToDevice, C->s_copy));
        span.end();
      }
      C->h2d_bytes += ch.bytes;
      SP_CUDA(cudaEventRecord(C->ev_copied[slot], C->s_copy));
      SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_copied[slot], 0));
      BlockView b{static_cast<const char*>(C->ring[slot].p), ch.w3_off, ch.w2_off, ch.rc, L->ldm,
                  ch.ldc, ch.r0};
      const int t0 = is_cc ? Te - ng : 0;
      {
        GpuSpan span(C, C->s_comp, 2, is_cc ? SP_TRACE_CG_PRIME : SP_TRACE_CG, double(ch.bytes));
        SP_TRY(run_block(C, L, b, x_dev, xdtype, M, ws[c], t0, Te - t0, true, C->s_comp));
        span.end();
      }
      SP_CUDA(cudaEventRecord(C->ev_free[slot], C->s_comp));
      ++chunk_seq;
    }
  }

  // ---- CC block on host threads (overlaps everything enqueued above) ----
  host_span(C, 0, SP_TRACE_LAUNCH, t_call, now_s(), 0.0);
  if (need_cc) {
    if (!host_io) SP_CUDA(cudaEventSynchronize(C->ev_x));
    for (int c = 0; c < n_calls; ++c) {
      const double t_cc0 = now_s();
      const sp_layer* L = calls[c].layer;
      const int64_t Tcc = calls[c].tokens - calls[c].n_g;
      if (L->d.b1 <= 0 || Tcc <= 0) continue;
      const int64_t ldx = round_up(M, kPadElems), lda = round_up(L->d.b1, kPadElems);
      C->hscratch.assign(size_t(Tcc * ldx + Tcc * lda), 0.f);
      float* xh = C->hscratch.data();
      float* ah = xh + Tcc * ldx;
      for (int64_t i = 0; i < Tcc; ++i) {
        const int64_t row = calls[c].token_ids ? calls[c].token_ids[i] : i;
        if (xdtype == SP_BF16) {
          const uint16_t* src = static_cast<const uint16_t*>(x_host) + row * M;
          for (int64_t k = 0; k < M; ++k) {
            const uint32_t u = uint32_t(src[k]) << 16;
            memcpy(&xh[i * ldx + k], &u, 4);
          }
        } else {
          memcpy(&xh[i * ldx], static_cast<const float*>(x_host) + row * M, M * 4);
        }
      }
      std::vector<HostChunk> hc(L->n_cc_chunks);
      for (int k = 0; k < L->n_cc_chunks; ++k) {
        const Chunk& ch = L->chunks[k];
        const char* base = static_cast<const char*>(L->host) + ch.off;
        hc[k] = HostChunk{base, L->d.gated ? base + ch.w3_off : nullptr, base + ch.w2_off, ch.r0,
                          ch.rc, ch.ldc};
      }
      CCProblem pr{L->d.wdtype, L->d.gated, L->d.act, M, N, L->ldm, hc.data(), L->n_cc_chunks,
                   L->d.b1, xh, ldx, Tcc, ah, lda,
                   reinterpret_cast<float*>(hp + p_ycc[c])};
      cc_forward(pr, *C->pool, (flags & SP_NO_CC_THREADS) ? 1 : C->host_threads);
      host_span(C, 3, SP_TRACE_CC, t_cc0, now_s(), double(L->cc_bytes));
      SP_CUDA(cudaMemcpyAsync(ws[c].ycc, hp + p_ycc[c], size_t(Tcc) * N * 4, cudaMemcpyHostToDevice,
                              C->s_aux));
    }
    SP_CUDA(cudaEventRecord(C->ev_ycc, C->s_aux));
    SP_CUDA(cudaStreamWaitEvent(C->s_comp, C->ev_ycc, 0));
  }

  // ---- merge ----
  MergeArgs ma{};
  ma.n_calls = n_calls;
  ma.T = int(T);
  ma.N = N;
  ma.acc = reinterpret_cast<float*>(dws + o_acc);
  ma.out = host_io ? static_cast<void*>(dws + o_ydev) : y;
  ma.odtype = ydtype;
  for (int c = 0; c < n_calls; ++c) {
    const sp_layer* L = calls[c].layer;
    const int64_t Tcc = calls[c].tokens - calls[c].n_g;
    ma.c[c] = MergeCall{ws[c].y, (L->d.b1 > 0 && Tcc > 0) ? ws[c].ycc : nullptr, ws[c].ids,
                        ws[c].gates, int(calls[c].tokens), int(Tcc)};
  }
  if (ydtype == SP_F32 && !host_io) ma.acc = static_cast<float*>(y);
  {
    const int threads = 256;
    const int blocks = int(std::min<int64_t>((N + threads - 1) / threads, int64_t(C->num_sms) * 4));
    GpuSpan span(C, C->s_comp, 2, SP_TRACE_MERGE, 0.0);
    merge_kernel<<<blocks, threads, 0, C->s_comp>>>(ma);
    SP_CUDA(cudaGetLastError());
    span.end();
    ++C->launches;
  }
  if (host_io) {
    SP_CUDA(cudaMemcpyAsync(hp + p_y, dws + o_ydev, size_t(T) * N * yel, cudaMemcpyDeviceToHost,
                            C->s_comp));
    SP_CUDA(cudaStreamSynchronize(C->s_comp));
    memcpy(y, hp + p_y, size_t(T) * N * yel);
  } else {
    SP_CUDA(cudaEventRecord(C->ev_done, C->s_comp));
    SP_CUDA(cudaStreamWaitEvent(user, C->ev_done, 0));
  }
  if (C->trace.on) ++C->trace.call;
  (void)chunk_seq;
  return SP_OK;
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
  for (cudaEvent_t* e : {&C->ev_user, &C->ev_x, &C->ev_ycc, &C->ev_done})
    SP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (int i = 0; i < kRingSlots; ++i) {
    SP_CUDA(cudaEventCreateWithFlags(&C->ev_copied[i], cudaEventDisableTiming));
    SP_CUDA(cudaEventCreateWithFlags(&C->ev_free[i], cudaEventDisableTiming));
  }
  C->host_threads = host_threads > 0 ? host_threads : std::max(1, hw);
  C->pool = std::make_unique<ThreadPool>(C->host_threads);
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
  cudaDeviceSynchronize();
  for (cudaEvent_t e : {C->ev_user, C->ev_x, C->ev_ycc, C->ev_done}) cudaEventDestroy(e);
  for (int i = 0; i < kRingSlots; ++i) {
    cudaEventDestroy(C->ev_copied[i]);
    cudaEventDestroy(C->ev_free[i]);
  }
  cudaStreamDestroy(C->s_comp);
  cudaStreamDestroy(C->s_copy);
  cudaStreamDestroy(C->s_aux);
  g_ctx.reset();
  return SP_OK;
}

int sp_layer_create(const sp_layer_desc* desc, const void* w1t, const void* w3t, const void* w2t,
                    sp_layer_t* out) {
  if (!desc || !out || !w1t || !w2t) return fail(SP_ERR_VALUE, "NULL argument");
  const sp_layer_desc& d = *desc;
  if (d.model_dim < 1 || d.hidden_dim < 1 || d.out_dim < 1)
    return fail(SP_ERR_SHAPE, "layer dims must be >= 1 (M=%lld H=%lld N=%lld)", (long long)d.model_dim,
                (long long)d.hidden_dim, (long long)d.out_dim);
  if (d.model_dim > (1 << 30) || d.hidden_dim > (1 << 30) || d.out_dim > (1 << 30))
    return fail(SP_ERR_SHAPE, "layer dims too large");
  if (d.b1 < 0 || d.b2 < d.b1 || d.b2 > d.hidden_dim)
    return fail(SP_ERR_VALUE, "boundaries must satisfy 0 <= b1 <= b2 <= H (b1=%lld b2=%lld H=%lld)",
                (long long)d.b1, (long long)d.b2, (long long)d.hidden_dim);
  if (d.gated && !w3t) return fail(SP_ERR_VALUE, "gated layer needs w3t");
  if (d.act < 0 || d.act > 2) return fail(SP_ERR_VALUE, "unknown activation %d", d.act);
  if (d.wdtype != SP_F32 && d.wdtype != SP_BF16) return fail(SP_ERR_VALUE, "unknown weight dtype");
  Context* C = ctx_or_null();
  if (!C) return fail(SP_ERR_STATE, "sp_init has not been called");
  std::lock_guard<std::mutex> g(C->mu);
  auto L = std::make_unique<sp_layer>();
  L->d = d;
  L->device = C->device;
  L->esz = d.wdtype == SP_BF16 ? 2 : 4;
  L->ldm = round_up(d.model_dim, kPadElems);
  L->host_only = C->host_only;
  int st = pack_layer(L.get(), w1t, d.gated ? w3t : nullptr, w2t);
  if (st != SP_OK) {
    if (L->gg) cudaFree(L->gg);
    if (L->host) L->host_only ? free(L->host) : (void)cudaFreeHost(L->host);
    return st;
  }
  if (C->host_only) {
    *out = L.release();
    return SP_OK;
  }
  if (L->max_chunk_bytes > C->ring_bytes) {
    SP_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < kRingSlots; ++i) SP_TRY(C->ring[i].ensure(L->max_chunk_bytes));
    C->ring_bytes = C->ring[0].n;
  }
  *out = L.release();
  return SP_OK;
}

int sp_layer_destroy(sp_layer_t L) {
  if (!L) return SP_OK;
  Context* C = ctx_or_null();
  if (C && !C->host_only) {
    std::lock_guard<std::mutex> g(C->mu);
    cudaStreamSynchronize(C->s_comp);
    cudaStreamSynchronize(C->s_copy);
  }
  if (L->gg) cudaFree(L->gg);
  if (L->host) L->host_only ? free(L->host) : (void)cudaFreeHost(L->host);
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
  if (!calls || !x || !y) return fail(SP_ERR_VALUE, "NULL argument");
  std::lock_guard<std::mutex> g(C->mu);
  return forward_batch(C, calls, n_calls, x, xdtype, T, y, ydtype, flags,
                       static_cast<cudaStream_t>(stream));
}

int sp_cc_forward_host(sp_layer_t L, const void* x, int xdtype, int64_t T, float* y_cc,
                       int threads) {
  if (!L || !x || !y_cc) return fail(SP_ERR_VALUE, "NULL argument");
  if (T < 0) return fail(SP_ERR_SHAPE, "negative token count");
  const int64_t M = L->d.model_dim, N = L->d.out_dim;
  const int64_t ldx = round_up(M, kPadElems), lda = round_up(std::max<int64_t>(L->d.b1, 1), kPadElems);
  std::vector<float> xh(size_t(T * ldx), 0.f), ah(size_t(T * lda), 0.f);
  for (int64_t i = 0; i < T; ++i) {
    if (xdtype == SP_BF16) {
      const uint16_t* src = static_cast<const uint16_t*>(x) + i * M;
      for (int64_t k = 0; k < M; ++k) {
        const uint32_t u = uint32_t(src[k]) << 16;
        memcpy(&xh[i * ldx + k], &u, 4);
      }
    } else {
      memcpy(&xh[i * ldx], static_cast<const float*>(x) + i * M, M * 4);
    }
  }
  std::vector<HostChunk> hc(L->n_cc_chunks);
  for (int k = 0; k < L->n_cc_chunks; ++k) {
    const Chunk& ch = L->chunks[k];
    const char* base = static_cast<const char*>(L->host) + ch.off;
    hc[k] = HostChunk{base, L->d.gated ? base + ch.w3_off : nullptr, base + ch.w2_off, ch.r0, ch.rc,
                      ch.ldc};
  }
  CCProblem pr{L->d.wdtype, L->d.gated, L->d.act, M, N, L->ldm, hc.data(), L->n_cc_chunks, L->d.b1,
               xh.data(), ldx, T, ah.data(), lda, y_cc};
  Context* C = ctx_or_null();
  if (C && threads != 1) {
    cc_forward(pr, *C->pool, threads > 0 ? threads : C->host_threads);
  } else {
    ThreadPool local(std::max(1, threads));
    cc_forward(pr, local, std::max(1, threads));
  }
  return SP_OK;
}

int sp_trace_enable(int on) {
  Context* C = ctx_or_null();
  if (!C || C->host_only) return fail(SP_ERR_STATE, "sp_init(device) has not been called");
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
  if (tr.on) {
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
  for (int i = 0; i < k; ++i) {
    const Span& sp = tr.spans[i];
    sp_trace_record r{};
    r.index = ++counters[sp.stream & 3];
    r.stream = sp.stream;
    r.kind = sp.kind;
    r.call = sp.call;
    r.bytes = sp.bytes;
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
