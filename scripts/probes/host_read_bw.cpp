// Host DRAM read bandwidth with N threads (AVX-512 streaming sum), the ceiling
// the decode CC block (csrc/host_cc.cpp) is compared against.
//   g++ -O3 -mavx512f -pthread host_read_bw.cpp -o host_read_bw && ./host_read_bw [threads] [MB]
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
  const int nt = argc > 1 ? atoi(argv[1]) : 16;
  const size_t mb = argc > 2 ? atol(argv[2]) : 2048;
  const size_t n = mb << 20;
  char* buf = static_cast<char*>(aligned_alloc(4096, n));
  memset(buf, 1, n);
  std::vector<double> sink(nt);
  for (int rep = 0; rep < 6; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        const size_t lo = n / nt * t, hi = n / nt * (t + 1);
        __m512 a0 = _mm512_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
        for (size_t i = lo; i < hi; i += 256) {
          _mm_prefetch(buf + i + 4096, _MM_HINT_T0);
          a0 = _mm512_add_ps(a0, _mm512_load_ps(reinterpret_cast<float*>(buf + i)));
          a1 = _mm512_add_ps(a1, _mm512_load_ps(reinterpret_cast<float*>(buf + i + 64)));
          a2 = _mm512_add_ps(a2, _mm512_load_ps(reinterpret_cast<float*>(buf + i + 128)));
          a3 = _mm512_add_ps(a3, _mm512_load_ps(reinterpret_cast<float*>(buf + i + 192)));
        }
        sink[t] = _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(a0, a1), _mm512_add_ps(a2, a3)));
      });
    for (auto& x : th) x.join();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %d  %zu MB  %.3f ms  %.1f GB/s\n", nt, mb, s * 1e3, n / s / 1e9);
  }
  return sink[0] == 12345.0;
}
