/*
 * sliced.h -- C ABI of the B200-native sliced-weight FFN path (libsliced.so).
 *
 * The reference has no FFI: its boundary is the Python operator API of
 * /root/reference/pkg/src/sliceplan/slicing_kernel.py.  Each entry point below
 * replaces one piece of it (file:line cited per function); the Python host
 * (paper_2411_15715_b200/sliced.py) keeps the reference's names, argument
 * meaning and exception classes on top of this ABI.
 *
 * Conventions
 *   - Plain C: integers, sizes and raw pointers.  No torch / CUDA types in the
 *     signatures except the opaque stream handle (a cudaStream_t, passed as
 *     void*; NULL = the legacy default stream).
 *   - Every function returns an sp_status; on failure sp_last_error() returns
 *     a thread-local message.  Codes map 1:1 onto the reference exception
 *     classes (sliceplan/errors.py:24-29): SP_ERR_SHAPE -> ShapeMismatch,
 *     SP_ERR_TOKENS -> TokenCountOutOfRange, SP_ERR_VALUE -> ValueError.
 *     Argument errors are detected before any work is enqueued, as the
 *     reference raises before computing (slicing_kernel.py:64-70,111-118).
 *   - Weights are copied into library-owned placement at layer creation
 *     (GG -> HBM, CC and CG -> pinned host, chunk-interleaved); activations
 *     and outputs stay caller-owned.  This deviates from SURVEY.md 8(b)
 *     ("the caller owns all weight buffers") on purpose: the CG block must
 *     sit in pinned, chunk-interleaved host memory and the GG block in HBM
 *     with 128-byte rows, which a caller's numpy / torch views are not; the
 *     caller may free its copies after sp_layer_create (host RAM is held
 *     twice only while both exist).  Caller-side CC is still possible:
 *     sp_set_cc_executor runs the CC block through the caller's own code.
 *   - One device per process/thread context (sp_init); forwards on one device
 *     are serialised by the library.
 *
 * Limits (each violation is reported as SP_ERR_VALUE before any work):
 *   - out_dim N <= 8192 for bf16 weights, <= 4096 for f32 (the decode kernel
 *     keeps 4 W2 column vectors per thread: kMaxVec, csrc/kernels.cuh);
 *   - model_dim M <= 16384 (the decode kernel's x tile, TT * roundup(M, 256)
 *     floats <= 16384, so 4 tokens per launch up to M = 4096, 1 up to 16384);
 *   - at most 32 calls per sp_forward_batch and 32 active experts per
 *     sp_moe_forward (kMaxCalls: the finalize kernel's by-value call table).
 *   All five BASELINE configs (M <= 8192, N <= 8192, <= 16 experts) fit.
 */
#ifndef SLICED_H_
#define SLICED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 4

typedef enum sp_status {
  SP_OK = 0,
  SP_ERR_SHAPE = 1,   /* ShapeMismatch        */
  SP_ERR_TOKENS = 2,  /* TokenCountOutOfRange */
  SP_ERR_VALUE = 3,   /* ValueError           */
  SP_ERR_CUDA = 4,    /* CUDA runtime failure */
  SP_ERR_NOMEM = 5,   /* allocation failure   */
  SP_ERR_STATE = 6    /* not initialised / wrong device */
} sp_status;

typedef enum sp_dtype { SP_F32 = 0, SP_BF16 = 1 } sp_dtype;

/* sliceplan.slicing_kernel.Activation (slicing_kernel.py:27-38) */
typedef enum sp_act { SP_ACT_IDENTITY = 0, SP_ACT_SILU = 1, SP_ACT_GELU = 2 } sp_act;

/* sp_forward_batch flags */
#define SP_IO_DEVICE 0u     /* x / y are device pointers (inputs resident in HBM) */
#define SP_IO_HOST 1u       /* x / y are host pointers; H2D / D2H inside the call  */
#define SP_NO_CC_THREADS 2u /* run the CC slice on the calling thread only         */
#define SP_X_TO_BF16 4u     /* with SP_IO_HOST and f32 x: round x to bf16 while staging
                               it (the activations of a bf16 layer), no caller-side cast */

typedef struct sp_layer* sp_layer_t;

/*
 * One FFN instance (a dense MLP or one MoE expert) and its column split.
 * Replaces SlicedWeights (slicing_kernel.py:41-54) + the floor rule of
 * slice_weights (slicing_kernel.py:71-74): b1 = floor(cc*H), b2 =
 * floor((cc+cg)*H) are computed by the caller and passed here.
 *   cc block = hidden columns [0, b1)    host-resident, run on host threads
 *   cg block = hidden columns [b1, b2)   host-resident, streamed, run on GPU
 *   gg block = hidden columns [b2, H)    HBM-resident, run on GPU
 */
typedef struct sp_layer_desc {
  int64_t model_dim;  /* M: input features  (rows of W1 / W3)              */
  int64_t hidden_dim; /* H: the sliced dimension                           */
  int64_t out_dim;    /* N: output features (columns of W2)                */
  int32_t gated;      /* 0: act(x W1) W2   1: (act(x W1) * (x W3)) W2      */
  int32_t act;        /* sp_act                                            */
  int32_t wdtype;     /* sp_dtype of the stored weights                    */
  int32_t chunk_rows; /* hidden rows per streamed chunk; 0 = auto (~8 MB)  */
  int64_t b1, b2;     /* block boundaries, 0 <= b1 <= b2 <= H              */
} sp_layer_desc;

/* One expert application inside a batched forward. */
typedef struct sp_call {
  sp_layer_t layer;
  int64_t tokens;           /* T_e rows this layer processes                   */
  const int32_t* token_ids; /* host array [T_e]: rows of x; NULL = 0..T_e-1     */
  const float* gates;       /* host array [T_e]: output weights; NULL = 1.0     */
  int64_t n_g;              /* last n_g of the T_e rows run the CC block on the
                               GPU (cg_prime, slicing_kernel.py:148-151)        */
} sp_call;

/* ---- library ---------------------------------------------------------- */
int sp_abi_version(void);
const char* sp_last_error(void);
/* Select / initialise the CUDA device; creates the copy + compute streams and
 * the host thread pool.  host_threads <= 0 = all online cores. */
int sp_init(int device, int host_threads);
int sp_shutdown(void);
int sp_device_count(int* count);

/* ---- placement (slice_weights, slicing_kernel.py:57-80) ---------------- */
/* w1t, w3t: [H, M] row-major (nn.Linear(M->H).weight layout, i.e. the
 * reference's w1 transposed); w3t NULL unless gated.  w2: [H, N] row-major (the
 * reference's own w2 layout, slicing_kernel.py:77).  Hidden unit h then owns
 * row h of all three, so every block is a contiguous row range.  Host pointers
 * in desc->wdtype; they are copied, the caller may free them afterwards. */
int sp_layer_create(const sp_layer_desc* desc, const void* w1t, const void* w3t,
                    const void* w2, sp_layer_t* out);
int sp_layer_destroy(sp_layer_t layer);
/* Bytes placed in HBM (gg), pinned host streamed to the GPU (cg) and pinned
 * host computed on the CPU (cc). */
int sp_layer_bytes(sp_layer_t layer, size_t* gg, size_t* cg, size_t* cc);
/* Block widths (cc, cg, gg) == SlicedWeights.block_widths (slicing_kernel.py:50-54). */
int sp_layer_widths(sp_layer_t layer, int64_t widths[3]);

/* ---- sliced weight store ---------------- */
/* A placed layer's two images: the GG block exactly as it sits in HBM
 * (W1t | W3t | W2 rows [b2, H), rows zero padded to 64 elements) and the
 * pinned host region (CC then CG chunks of chunk_rows hidden units, each
 * W1t | W3t | W2, 4 KB aligned).  Saving the images and creating a layer from
 * them skips the repack: a straight read into pinned memory plus one HBM
 * upload.  The desc must carry the chunk_rows the images were packed with
 * (sp_layer_image_sizes reports it). */
int sp_layer_image_sizes(sp_layer_t layer, size_t* gg_bytes, size_t* host_bytes, int32_t* chunk_rows);
/* Copy the images out (either destination may be NULL). */
int sp_layer_export(sp_layer_t layer, void* gg_dst, void* host_dst);
int sp_layer_create_from_images(const sp_layer_desc* desc, const void* gg_img, size_t gg_bytes,
                                const void* host_img, size_t host_bytes, sp_layer_t* out);
/* Same, reading the images from a file at the given offsets (the host image
 * lands directly in the layer's pinned region). */
int sp_layer_load_file(const sp_layer_desc* desc, const char* path, uint64_t gg_offset, size_t gg_bytes,
                       uint64_t host_offset, size_t host_bytes, sp_layer_t* out);
/* Re-slice a placed layer to new boundaries b1 <= b2 (the rates changed,
 * PAPER.md:103): rows are gathered back (GG rows from HBM) and re-placed. */
int sp_layer_reslice(sp_layer_t layer, int64_t b1, int64_t b2, sp_layer_t* out);

/* ---- forward (mlp_forward_sliced, slicing_kernel.py:97-124) ------------ */
/* y[t, :] = sum over calls c, rows i with ids_c[i] == t of
 *           gate_c[i] * FFN_c(x[t, :])   (FFN_c summed over its cc/cg/gg blocks)
 * x: [T, M] (xdtype), y: [T, N] (ydtype), overwritten.  Rows no call touches
 * are zero.  T = 0 (and every call covering 0 rows) is a valid empty forward
 * that returns SP_OK without touching the device, as the reference returns an
 * empty output (x and y may then be NULL).  With SP_IO_DEVICE the call returns once the CC slice is done and
 * the GPU work is enqueued (ordered after prior work on `stream`, and `stream`
 * is ordered after it); with SP_IO_HOST it returns with y written. */
int sp_forward_batch(const sp_call* calls, int n_calls, const void* x, int xdtype, int64_t T,
                     void* y, int ydtype, unsigned flags, void* stream);

/* ---- MoE layer (router + dispatch) -------- */
/* Top-k routing on the host in fp64: logits[t, e] = sum_m x[t, m] * router[m, e],
 * the k largest (ties -> lower expert id), softmax over those k logits.
 * ids / gates: [T, k].  Host-only; the oracle's route_topk is the parity check. */
int sp_moe_route(const float* router, int64_t model_dim, int n_experts, int top_k, const void* x,
                 int xdtype, int64_t T, int32_t* ids, float* gates);
/* One MoE FFN layer: route x (one device->host read of x serves the router
 * and the CC blocks), then a single batched forward over the active experts.
 * layers[e] == NULL marks an expert owned by another rank (expert parallel):
 * its tokens contribute nothing here.  Same x / y / flags / stream contract as
 * sp_forward_batch. */
int sp_moe_forward(const sp_layer_t* layers, int n_experts, const float* router, int top_k,
                   const void* x, int xdtype, int64_t T, void* y, int ydtype, unsigned flags,
                   void* stream);

/* ---- caller-supplied CC executor (north star: "the CC slice runs on host
 * threads through the reference CPU code") ------------------------------- */
/* Called on the library's CC coordinator thread, concurrently with the GPU
 * work of the same forward, once per call whose CC block is non-empty:
 *   x    [rows, ldx] f32: the call's CC token rows (gathered, in call order)
 *   y_cc [rows, out_dim] f32: to be OVERWRITTEN with
 *        sum over hidden units h in [0, b1) of act(x W1[:, h]) (* x W3[:, h]) W2[h, :]
 * `layer` identifies the expert (the caller maps it to its weights).  Return
 * 0 on success; non-zero fails the forward with SP_ERR_VALUE.  It must not
 * call back into this library. */
typedef int (*sp_cc_fn)(void* user, sp_layer_t layer, const float* x, int64_t ldx, int64_t rows, float* y_cc,
                        int64_t out_dim);
/* Install (fn != NULL) or remove (NULL) the executor for every later forward
 * on this context; the native AVX-512 / AMX CC kernels run when none is set. */
int sp_set_cc_executor(sp_cc_fn fn, void* user);

/* Host-only CC block (no GPU): y_cc[T, N] (f32) = sum over cc columns.  Used by
 * the CPU test suite and the host-core micro-benchmarks of the profile refit. */
int sp_cc_forward_host(sp_layer_t layer, const void* x, int xdtype, int64_t T, float* y_cc,
                       int threads);

/* ---- profiling hooks (perf-model refit, measured timelines) ------------ */
/* Last forward's measured stage intervals in the reference Gantt schema
 * (pipeline.py:347-364): stream 0 launch, 1 transfer, 2 gpu, 3 cpu; times in
 * seconds relative to the call start.  *n in: capacity, out: records. */
typedef enum sp_trace_kind {
  SP_TRACE_LAUNCH = 0,   /* host: enqueue of one forward's GPU work        */
  SP_TRACE_GG = 1,       /* gpu: GG up + down kernels of one call          */
  SP_TRACE_CG = 2,       /* gpu: one streamed CG chunk's kernels           */
  SP_TRACE_CG_PRIME = 3, /* gpu: one streamed CC chunk for the n_g rows    */
  SP_TRACE_COPY = 4,     /* transfer: one chunk's host-to-device copy      */
  SP_TRACE_CC = 5,       /* cpu: CC block of one call on host threads      */
  SP_TRACE_MERGE = 6,    /* gpu: merge kernel                              */
  SP_TRACE_ROUTE = 7,    /* host: MoE call entry -> dispatch (x read-back,
                            routing, grouping)                             */
  SP_TRACE_RETURN = 8,   /* host: forward enqueue done -> return to caller
                            (CC join, tail)                                */
  SP_TRACE_YCC = 9       /* transfer: CC partial host -> HBM (prefill-size
                            partials; small ones are read in place)        */
} sp_trace_kind;
typedef struct sp_trace_record {
  int32_t index;  /* 1-based item index within its stream                */
  int32_t stream; /* 0 launch, 1 transfer, 2 gpu, 3 cpu (pipeline.py:264) */
  int32_t kind;   /* sp_trace_kind                                        */
  int32_t call;   /* forward sequence number since sp_trace_enable        */
  double start_s, end_s;
  double bytes;   /* weight bytes moved or touched                        */
  double dev_s;   /* ffn_block launches: device-side duration, first CTA
                   * start to last CTA end (%globaltimer); 0 otherwise.
                   * start_s/end_s (CUDA events) also hold the launch's
                   * front-end latency, which grows by ~23 us while the
                   * copy engine saturates the host link.                 */
} sp_trace_record;
/* on != 0 clears the trace and starts recording (events on the library's own
 * streams, host clock for CC); on == 2 records GPU spans only around GG
 * launches (plus every host span), which leaves the step's timing untouched;
 * sp_trace_fetch synchronises the device. */
int sp_trace_enable(int on);
int sp_trace_fetch(sp_trace_record* out, int* n);
/* Kernels launched and bytes copied host-to-device by the library so far. */
int sp_stats(uint64_t* kernel_launches, uint64_t* h2d_bytes);

/* fp32 -> bf16 bit patterns, round to nearest even (the host activation cast
 * of the bf16 path; single-threaded AVX-512, no framework threads). */
int sp_round_bf16(const float* src, uint16_t* dst, int64_t n);

/* Pinned host buffer helpers (cudaHostAlloc; avoids torch's caching host
 * allocator rounding). */
int sp_host_alloc(size_t bytes, void** ptr);
int sp_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* SLICED_H_ */
