// Event-span probe: where does a CUDA-event span of a ~60 us kernel gain its
// extra ~20 us while the host link is saturated?  (The GG ffn_block launch of
// a decode step reads 84 us by events, 58 us by in-kernel %globaltimer.)
//
// For each background load (idle, copy-engine H2D, copy-engine D2H, an SM copy
// kernel reading mapped pinned memory) it records, on one stream:
//   A  spin(60us)  B  spin(60us)  C
// and prints the medians of A->B, B->C and the in-kernel span of the first spin.
// B->C isolates the per-kernel cost once the stream is already running.
#include <cuda_runtime.h>
#include <stdio.h>
#include <algorithm>
#include <vector>

__device__ unsigned long long g_t0, g_t1;
__device__ unsigned int g_done;

__global__ void spin(long long cycles, int stamp) {
  unsigned long long t;
  if (stamp && threadIdx.x == 0 && blockIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_t0 = t;
  }
  const long long c0 = clock64();
  while (clock64() - c0 < cycles) {
  }
  __syncthreads();
  if (stamp && threadIdx.x == 0) {
    if (atomicAdd(&g_done, 1u) == gridDim.x - 1) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_t1 = t;
      g_done = 0;
    }
  }
}

// SM-driven host->device copy: each thread streams 16 B loads from mapped pinned memory
__global__ void sm_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n, volatile int* stop) {
  for (;;) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
      dst[i] = src[i];
    if (*stop) return;
  }
}

static float med(std::vector<float> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  cudaStream_t s, c;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking);
  const size_t n = size_t(256) << 20;
  void *h, *d, *d2;
  cudaHostAlloc(&h, n, cudaHostAllocMapped);
  cudaMalloc(&d, n);
  cudaMalloc(&d2, n);
  int* stop;
  cudaHostAlloc(&stop, 4, cudaHostAllocMapped);
  void* hdev;
  cudaHostGetDevicePointer(&hdev, h, 0);
  int* stop_dev;
  cudaHostGetDevicePointer((void**)&stop_dev, stop, 0);
  const long long cyc = 60LL * 1965;
  const char* names[] = {"idle", "CE H2D 8MB chunks", "CE D2H 8MB chunks", "CE H2D 64MB", "SM copy (mapped host)"};
  unsigned int eflags[] = {cudaEventDefault, cudaEventBlockingSync};
  for (int ef = 0; ef < 2; ++ef)
    for (int load = 0; load < 5; ++load) {
      cudaDeviceSynchronize();
      *stop = 0;
      if (load == 1)
        for (int i = 0; i < 400; ++i) cudaMemcpyAsync(d, (char*)h + (size_t(i % 32) << 23), size_t(8) << 20, cudaMemcpyHostToDevice, c);
      if (load == 2)
        for (int i = 0; i < 400; ++i) cudaMemcpyAsync((char*)h + (size_t(i % 32) << 23), d, size_t(8) << 20, cudaMemcpyDeviceToHost, c);
      if (load == 3)
        for (int i = 0; i < 50; ++i) cudaMemcpyAsync(d, h, size_t(64) << 20, cudaMemcpyHostToDevice, c);
      if (load == 4) sm_copy<<<16, 512, 0, c>>>((const int4*)hdev, (int4*)d2, (size_t(64) << 20) / 16, stop_dev);
      cudaEvent_t a, b, e;
      cudaEventCreateWithFlags(&a, eflags[ef]);
      cudaEventCreateWithFlags(&b, eflags[ef]);
      cudaEventCreateWithFlags(&e, eflags[ef]);
      std::vector<float> ab, bc, dev;
      for (int r = 0; r < 25; ++r) {
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        spin<<<148, 128, 0, s>>>(cyc, 1);
        cudaEventRecord(b, s);
        spin<<<148, 128, 0, s>>>(cyc, 0);
        cudaEventRecord(e, s);
        cudaEventSynchronize(e);
        float x, y;
        cudaEventElapsedTime(&x, a, b);
        cudaEventElapsedTime(&y, b, e);
        unsigned long long t0, t1;
        cudaMemcpyFromSymbol(&t0, g_t0, 8);
        cudaMemcpyFromSymbol(&t1, g_t1, 8);
        ab.push_back(x * 1000.f);
        bc.push_back(y * 1000.f);
        dev.push_back(float(t1 - t0) * 1e-3f);
      }
      *stop = 1;
      cudaDeviceSynchronize();
      // copy rate seen by the load alone over the same window is not measured here
      printf("%-24s events=%s  A->B %.1f us  B->C %.1f us  in-kernel %.1f us\n", names[load],
             ef ? "blocking" : "default ", med(ab), med(bc), med(dev));
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      cudaEventDestroy(e);
    }
  // The same A spin B spin C sequence with each spin a launch of one
  // instantiated single-kernel CUDA graph (launch descriptor uploaded once);
  // `upd` = kernel-node parameters changed before every launch.
  for (int upd = 0; upd < 2; ++upd)
    for (int load = 0; load < 5; load += (load == 1 ? 3 : 1)) {
      cudaDeviceSynchronize();
      *stop = 0;
      cudaEvent_t a, b, e;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventCreate(&e);
      cudaGraph_t g;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      spin<<<148, 128, 0, s>>>(cyc, 1);
      cudaStreamEndCapture(s, &g);
      cudaGraphExec_t ex;
      cudaGraphInstantiate(&ex, g, 0);
      cudaGraphUpload(ex, s);
      size_t nn = 0;
      cudaGraphGetNodes(g, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(g, nodes.data(), &nn);
      cudaGraphNode_t k0 = nullptr;
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t == cudaGraphNodeTypeKernel) { k0 = nd; break; }
      }
      cudaStreamSynchronize(s);
      if (load == 1)
        for (int i = 0; i < 400; ++i) cudaMemcpyAsync(d, (char*)h + (size_t(i % 32) << 23), size_t(8) << 20, cudaMemcpyHostToDevice, c);
      if (load == 4) sm_copy<<<16, 512, 0, c>>>((const int4*)hdev, (int4*)d2, (size_t(64) << 20) / 16, stop_dev);
      std::vector<float> ab, bc, dev;
      for (int r = 0; r < 25; ++r) {
        if (upd) {
          long long cy = cyc + (r & 1);
          int st = 1;
          void* args[2] = {&cy, &st};
          cudaKernelNodeParams kp{};
          kp.func = (void*)spin;
          kp.gridDim = dim3(148);
          kp.blockDim = dim3(128);
          kp.kernelParams = args;
          cudaGraphExecKernelNodeSetParams(ex, k0, &kp);
        }
        cudaEventRecord(a, s);
        cudaGraphLaunch(ex, s);
        cudaEventRecord(b, s);
        cudaGraphLaunch(ex, s);
        cudaEventRecord(e, s);
        cudaEventSynchronize(e);
        float x, y;
        cudaEventElapsedTime(&x, a, b);
        cudaEventElapsedTime(&y, b, e);
        unsigned long long t0, t1;
        cudaMemcpyFromSymbol(&t0, g_t0, 8);
        cudaMemcpyFromSymbol(&t1, g_t1, 8);
        ab.push_back(x * 1000.f);
        bc.push_back(y * 1000.f);
        dev.push_back(float(t1 - t0) * 1e-3f);
      }
      *stop = 1;
      cudaDeviceSynchronize();
      printf("graph%s %-24s A->B %.1f us  B->C %.1f us  in-kernel %.1f us\n", upd ? "+setparams" : "          ",
             names[load], med(ab), med(bc), med(dev));
    }
  // Per kernel or per event?  A spin spin spin B under the H2D load, with and
  // without an intermediate (timing-disabled) event between the kernels.
  for (int mid = 0; mid < 3; ++mid)
    for (int load = 0; load < 2; ++load) {
      cudaDeviceSynchronize();
      if (load == 1)
        for (int i = 0; i < 400; ++i) cudaMemcpyAsync(d, (char*)h + (size_t(i % 32) << 23), size_t(8) << 20, cudaMemcpyHostToDevice, c);
      cudaEvent_t a, b, m;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventCreateWithFlags(&m, mid == 2 ? cudaEventDefault : cudaEventDisableTiming);
      std::vector<float> ab;
      for (int r = 0; r < 25; ++r) {
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        for (int k = 0; k < 3; ++k) {
          spin<<<148, 128, 0, s>>>(cyc, 0);
          if (mid && k < 2) cudaEventRecord(m, s);
        }
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float x;
        cudaEventElapsedTime(&x, a, b);
        ab.push_back(x * 1000.f);
      }
      cudaDeviceSynchronize();
      printf("3 spins, %s, %-18s A->B %.1f us\n",
             mid == 0 ? "no event between   " : mid == 1 ? "no-timing events   " : "timing events      ",
             names[load], med(ab));
    }
  return 0;
}
