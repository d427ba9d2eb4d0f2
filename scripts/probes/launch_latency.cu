// Launch-latency probe: CUDA-event span of an (almost) empty kernel as a
// function of its parameter size, with and without a pinned H2D copy stream
// saturating the host link.  Decides whether big __grid_constant__ argument
// structs cost launch latency while the CG streamer runs.
#include <cuda_runtime.h>
#include <stdio.h>
#include <vector>
#include <algorithm>

template <int BYTES>
struct P { unsigned char b[BYTES]; };

template <int BYTES>
__global__ void k(const __grid_constant__ P<BYTES> p, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[BYTES - 1] == 7) *out = 1;
}

template <int BYTES>
float span(cudaStream_t s, int* out, int reps) {
  P<BYTES> p{};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> v;
  for (int r = 0; r < reps; ++r) {
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    k<BYTES><<<148, 128, 0, s>>>(p, out);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    v.push_back(ms * 1000.f);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

// The same span when event A, the kernel and event B are nodes of one CUDA graph
// whose kernel parameters are updated before every launch.
template <int BYTES>
float span_graph(cudaStream_t s, int* out, int reps) {
  P<BYTES> p{};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraph_t g;
  cudaGraphCreate(&g, 0);
  cudaGraphNode_t na, nk, nb;
  cudaGraphAddEventRecordNode(&na, g, nullptr, 0, a);
  void* args[2] = {&p, &out};
  cudaKernelNodeParams kp{};
  kp.func = reinterpret_cast<void*>(k<BYTES>);
  kp.gridDim = dim3(148);
  kp.blockDim = dim3(128);
  kp.kernelParams = args;
  cudaGraphAddKernelNode(&nk, g, &na, 1, &kp);
  cudaGraphAddEventRecordNode(&nb, g, &nk, 1, b);
  cudaGraphExec_t ex;
  if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) return -1.f;
  std::vector<float> v;
  for (int r = 0; r < reps; ++r) {
    cudaStreamSynchronize(s);
    p.b[0] = (unsigned char)r;
    cudaGraphExecKernelNodeSetParams(ex, nk, &kp);
    cudaGraphLaunch(ex, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    v.push_back(ms * 1000.f);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

// Stream blocked on an event that a copy completes; A, kernel, B queued behind it.
template <int BYTES>
float span_behind_copy(cudaStream_t s, cudaStream_t c, void* d, void* h, int* out, int reps) {
  P<BYTES> p{};
  cudaEvent_t a, b, e;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  std::vector<float> v;
  for (int r = 0; r < reps; ++r) {
    cudaStreamSynchronize(s);
    cudaMemcpyAsync(d, h, size_t(8) << 20, cudaMemcpyHostToDevice, c);
    cudaEventRecord(e, c);
    cudaStreamWaitEvent(s, e, 0);
    cudaEventRecord(a, s);
    k<BYTES><<<148, 128, 0, s>>>(p, out);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    v.push_back(ms * 1000.f);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

// A ~60 us kernel: is the extra latency under a busy link at the start or the end of the span?
__global__ void spin(long long cycles, int* out) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = 2;
}

float span_spin(cudaStream_t s, int* out, long long cycles, cudaStream_t c, void* d, void* h, int mode, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> v;
  for (int r = 0; r < reps; ++r) {
    cudaDeviceSynchronize();
    if (mode == 1) cudaMemcpyAsync(d, h, size_t(64) << 20, cudaMemcpyHostToDevice, c);  // link busy first
    cudaEventRecord(a, s);
    spin<<<148, 128, 0, s>>>(cycles, out);
    cudaEventRecord(b, s);
    if (mode == 2) cudaMemcpyAsync(d, h, size_t(64) << 20, cudaMemcpyHostToDevice, c);  // link busy after launch
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    v.push_back(ms * 1000.f);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  cudaStream_t s, c;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 4);
  size_t n = size_t(256) << 20;
  void *h, *d;
  cudaHostAlloc(&h, n, 0);
  cudaMalloc(&d, n);
  for (int load = 0; load < 2; ++load) {
    if (load)
      for (int i = 0; i < 40; ++i) cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, c);  // ~190 ms of copies
    printf("%s: 16 B %.1f us | 1 KB %.1f us | 2 KB %.1f us | 4 KB %.1f us\n",
           load ? "with H2D copies" : "idle link      ", span<16>(s, out, 51), span<1024>(s, out, 51),
           span<2048>(s, out, 51), span<4000>(s, out, 51));
    printf("%s: graph 16 B %.1f us | graph 2 KB %.1f us\n", load ? "with H2D copies" : "idle link      ",
           span_graph<16>(s, out, 51), span_graph<2048>(s, out, 51));
    cudaStreamSynchronize(c);
  }
  cudaStream_t c2;
  cudaStreamCreateWithFlags(&c2, cudaStreamNonBlocking);
  for (int i = 0; i < 40; ++i) cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, c2);
  printf("queued behind a copy event, link busy: 2 KB %.1f us\n", span_behind_copy<2048>(s, c, (char*)d + (size_t(128) << 20), h, out, 21));
  cudaStreamSynchronize(c2);
  const long long cyc = 60LL * 1965;  // ~60 us at 1965 MHz
  printf("60us spin kernel: idle link %.1f us | copy started before %.1f us | copy started after launch %.1f us\n",
         span_spin(s, out, cyc, c, d, h, 0, 21), span_spin(s, out, cyc, c, d, h, 1, 21),
         span_spin(s, out, cyc, c, d, h, 2, 21));
  return 0;
}
