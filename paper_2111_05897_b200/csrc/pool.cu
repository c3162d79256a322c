// fp64 pooling -- EmbeddingWorker::serve_pull (embedding_worker.hpp:541-557).
//
// One row group (L lanes x V floats) per (sample, group) segment: acc_d = sum over the
// segment's listings, in listing order, of (double)row[d] (duplicates counted);
// out = float(acc * scale) with scale = 1.0/n (mean) or 1.0 (sum); empty segments
// write zeros. Also emits the per-listing read version (PullResult::read_versions).
//
// Latency, not bandwidth, is what a naive version loses to: offsets -> slot -> row is
// a chain of three dependent loads. The slot of a segment's first listing is loaded
// speculatively at index sg together with the offsets, which is exactly right for
// one-hot batches (offsets[sg] == sg), so a one-hot segment costs two round trips.
// The grid covers every segment (no grid-stride loop) so the SMs stay full of
// independent chains.
//
// HBM per segment (one-hot, D=64): 256 B row read + 256 B pooled write + 8 B version
// word + 4 B slot.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "table.cuh"
#include "vec.cuh"

namespace hps {

template <int V, int L, bool kGuard>
__global__ void __launch_bounds__(256)
    pool_kernel(DevTable t, const uint32_t* __restrict__ offsets,
                const uint32_t* __restrict__ slots, uint32_t BF, uint64_t N, int mean,
                float* __restrict__ out, uint64_t* __restrict__ out_rv64,
                uint32_t* __restrict__ out_rv32) {
  using G = Geo<V, L, kGuard>;
  const int ln = G::lane();
  const uint32_t D = t.D;
  const int chunks = kGuard ? (D + G::kSpan - 1) / G::kSpan : 1;
  for (uint64_t sg = G::group(); sg < BF; sg += G::groups()) {
    const uint32_t a = offsets[sg], e = offsets[sg + 1];
    const uint32_t spec = sg < N ? slots[sg] : 0u;  // speculative: right when a == sg
    // Empty groups pool to zeros (embedding_worker.hpp:543): keep scale finite there.
    const double scale = (mean && e > a) ? __drcp_rn(static_cast<double>(e - a)) : 1.0;
    if (e == a + 1) {
      // single listing (every segment of a one-hot batch)
      const uint32_t s = a == sg ? spec : slots[a];
      const bool ok = slot_ok(t, s);
      const float* row = t.rows + static_cast<uint64_t>(ok ? s : 0) * t.stride;
      if (ln == 0) {
        const uint32_t v = ok ? t.vt[s].x : 0u;
        if (out_rv64) out_rv64[a] = v;
        if (out_rv32) out_rv32[a] = v;
      }
      for (int c = 0; c < chunks; ++c) {
        const uint32_t d0 = c * G::kSpan + ln * V;
        if (kGuard && d0 >= D) break;
        float r[V], o[V];
        if (ok) load_vec<V>(row + d0, r);
        else for (int k = 0; k < V; ++k) r[k] = 0.0f;
#pragma unroll
        for (int k = 0; k < V; ++k)
          o[k] = __double2float_rn(__dmul_rn(__dadd_rn(0.0, static_cast<double>(r[k])), scale));
        float* dst = out + sg * D + d0;
        if (kGuard) {
          for (int k = 0; k < V; ++k)
            if (d0 + k < D) dst[k] = o[k];
        } else {
          store_vec_cs<V>(dst, o);
        }
      }
      continue;
    }
    for (int c = 0; c < chunks; ++c) {
      const uint32_t d0 = c * G::kSpan + ln * V;
      if (kGuard && d0 >= D) break;
      double acc[V];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = 0.0;
      uint32_t i = a;
      // Two listings in flight per iteration for memory-level parallelism.
      for (; i + 1 < e; i += 2) {
        uint32_t s0 = slots[i], s1 = slots[i + 1];
        float r0[V], r1[V];
        if (slot_ok(t, s0)) load_vec<V>(t.rows + (uint64_t)s0 * t.stride + d0, r0);
        else for (int k = 0; k < V; ++k) r0[k] = 0.0f;
        if (slot_ok(t, s1)) load_vec<V>(t.rows + (uint64_t)s1 * t.stride + d0, r1);
        else for (int k = 0; k < V; ++k) r1[k] = 0.0f;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          acc[k] = __dadd_rn(acc[k], static_cast<double>(r0[k]));
          acc[k] = __dadd_rn(acc[k], static_cast<double>(r1[k]));
        }
        if (c == 0 && ln == 0) {
          uint32_t v0 = slot_ok(t, s0) ? t.vt[s0].x : 0, v1 = slot_ok(t, s1) ? t.vt[s1].x : 0;
          if (out_rv64) out_rv64[i] = v0, out_rv64[i + 1] = v1;
          if (out_rv32) out_rv32[i] = v0, out_rv32[i + 1] = v1;
        }
      }
      if (i < e) {
        uint32_t s0 = slots[i];
        float r0[V];
        if (slot_ok(t, s0)) load_vec<V>(t.rows + (uint64_t)s0 * t.stride + d0, r0);
        else for (int k = 0; k < V; ++k) r0[k] = 0.0f;
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = __dadd_rn(acc[k], static_cast<double>(r0[k]));
        if (c == 0 && ln == 0) {
          uint32_t v0 = slot_ok(t, s0) ? t.vt[s0].x : 0;
          if (out_rv64) out_rv64[i] = v0;
          if (out_rv32) out_rv32[i] = v0;
        }
      }
      float o[V];
#pragma unroll
      for (int k = 0; k < V; ++k) o[k] = __double2float_rn(__dmul_rn(acc[k], scale));
      float* dst = out + sg * D + d0;
      if (kGuard) {
        for (int k = 0; k < V; ++k)
          if (d0 + k < D) dst[k] = o[k];
      } else {
        store_vec_cs<V>(dst, o);
      }
    }
  }
}

void launch_pool(const DevTable& t, const uint32_t* offsets, const uint32_t* slots, uint32_t BF,
                 uint64_t N, int mean, float* out, uint64_t* out_rv64, uint32_t* out_rv32,
                 cudaStream_t st) {
  if (!BF) return;
  HPS_DISPATCH_DIM(t.D, {
    uint64_t groups_per_block = 256 / L;
    uint32_t blocks = std::min<uint64_t>(ceil_div(BF, groups_per_block), 1u << 30);
    pool_kernel<V, L, G><<<blocks, 256, 0, st>>>(t, offsets, slots, BF, N, mean, out, out_rv64,
                                                 out_rv32);
  });
  HPS_LAUNCH_CHECK();
}

}  // namespace hps
