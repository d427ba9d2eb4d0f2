// Test driver for the AMX CC kernel built with SP_AMX_EMULATE (software tiles):
// lays bf16 weights out as the runtime's CC chunks and runs cc_forward_amx
// (with prepack: on the prepacked W2 copy, as the runtime does after a layer's first AMX call).
#include <stdint.h>
#include <string.h>

#include <vector>

#include "host_cc.h"

extern "C" int amx_emu_run(int gated, int act, int64_t M, int64_t N, int64_t b1, int64_t chunk_rows,
                           const uint16_t* w1t, const uint16_t* w3t, const uint16_t* w2,  // [b1, M] / [b1, M] / [b1, N]
                           const float* x, int64_t T, float* y, int threads, int prepack) {
  const int64_t ldm = (M + 63) / 64 * 64, ldn = (N + 63) / 64 * 64, ldx = ldm;
  std::vector<std::vector<uint16_t>> store;
  std::vector<sp::HostChunk> chunks;
  for (int64_t r0 = 0; r0 < b1; r0 += chunk_rows) {
    const int64_t rc = std::min(chunk_rows, b1 - r0);
    std::vector<uint16_t> c(size_t(rc * (2 * ldm + ldn)), 0);
    for (int64_t r = 0; r < rc; ++r) {
      memcpy(&c[size_t(r * ldm)], w1t + (r0 + r) * M, size_t(M) * 2);
      if (gated) memcpy(&c[size_t(rc * ldm + r * ldm)], w3t + (r0 + r) * M, size_t(M) * 2);
      memcpy(&c[size_t(2 * rc * ldm + r * ldn)], w2 + (r0 + r) * N, size_t(N) * 2);
    }
    store.push_back(std::move(c));
    const uint16_t* base = store.back().data();
    chunks.push_back(sp::HostChunk{base, gated ? base + rc * ldm : nullptr, base + 2 * rc * ldm, r0, rc});
  }
  std::vector<float> xs(size_t(T * ldx), 0.f);
  for (int64_t t = 0; t < T; ++t) memcpy(&xs[size_t(t * ldx)], x + t * M, size_t(M) * 4);
  sp::CCProblem p{1, gated, act, M, N, ldm, ldn, chunks.data(), int(chunks.size()), b1, xs.data(), ldx, T, y};
  sp::ThreadPool pool(threads);
  std::vector<uint16_t> w2p;
  if (prepack) {  // the layer-level VNNI copy of W2 the runtime builds once (amx_prepack_w2)
    w2p.assign(sp::amx_w2_prepack_elems(p), 0xffff);
    sp::amx_prepack_w2(p, w2p.data(), pool, threads);
    p.w2p = w2p.data();
  }
  sp::cc_forward_amx(p, pool, threads);
  return 0;
}
