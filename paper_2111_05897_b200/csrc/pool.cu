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
// one-hot batches (offsets[sg] == sg), so a one-hot segment costs two round trips, and
// every group keeps kPoolILP such segments in flight.
//
// HBM per segment (one-hot, D=64): 256 B row read + 256 B pooled write + 8 B version
// word + 4 B slot.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "table.cuh"
#include "vec.cuh"

namespace hps {

namespace {

constexpr int kPoolILP = 2;

template <int V, bool kGuard>
__device__ __forceinline__ void write_out(float* dst, const float (&o)[V], uint32_t d0,
                                          uint32_t D) {
  if (kGuard) {
    for (int k = 0; k < V; ++k)
      if (d0 + k < D) dst[k] = o[k];
  } else {
    store_vec_cs<V>(dst, o);
  }
}

// Any segment shape (empty, one listing, many listings with duplicates).
template <int V, int L, bool kGuard>
__device__ void pool_general(const DevTable& t, const uint32_t* __restrict__ slots, uint64_t sg,
                             uint32_t a, uint32_t e, double scale, int ln, float* out,
                             uint64_t* out_rv64, uint32_t* out_rv32) {
  using G = Geo<V, L, kGuard>;
  const uint32_t D = t.D;
  const bool want_rv = out_rv64 || out_rv32;  // row headers are only read when asked for
  const int chunks = kGuard ? (D + G::kSpan - 1) / G::kSpan : 1;
  for (int c = 0; c < chunks; ++c) {
    const uint32_t d0 = c * G::kSpan + ln * V;
    if (kGuard && d0 >= D) break;
    double acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = 0.0;
    // Four listings in flight per iteration for memory-level parallelism; the fp64 sum
    // still runs in listing order.
    for (uint32_t i0 = a; i0 < e; i0 += 4) {
      uint32_t sl[4];
      float r[4][V];
#pragma unroll
      for (int u = 0; u < 4; ++u) sl[u] = i0 + u < e ? slots[i0 + u] : kInvalidSlot;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (slot_ok(t, sl[u])) load_vec<V>(t.rows + (uint64_t)sl[u] * t.stride + d0, r[u]);
        else for (int k = 0; k < V; ++k) r[u][k] = 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u >= e) break;
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = __dadd_rn(acc[k], static_cast<double>(r[u][k]));
        if (want_rv && c == 0 && ln == 0) {
          const uint32_t v0 = slot_ok(t, sl[u]) ? vt_read(t, sl[u]).x : 0;
          if (out_rv64) out_rv64[i0 + u] = v0;
          if (out_rv32) out_rv32[i0 + u] = v0;
        }
      }
    }
    float o[V];
#pragma unroll
    for (int k = 0; k < V; ++k) o[k] = __double2float_rn(__dmul_rn(acc[k], scale));
    write_out<V, kGuard>(out + sg * D + d0, o, d0, D);
  }
}

}  // namespace

// Warp-cooperative pooling (D a multiple of 4 up to 128, or 1 / 2): a warp takes 32
// consecutive segments; lane l loads segment l's bounds and -- when it is a one-listing
// segment, every segment of a one-hot batch -- its slot (and read version), coalesced.
// Then the warp's row groups (L lanes x V floats, G per warp) gather those rows, kB rows
// in flight per lane with their owners' slots by shuffle, and write out[sg] = row + 0.0f:
// the fp64 sum of one listing, (float)((0.0 + (double)x) * 1.0), is x with -0.0 -> +0.0.
// The other segments (empty, several listings) go to pool_general group by group.
// kList: pool only the groups listed in glist[0 .. *glist_n) (the exchange's groups that
// their rows' owners did not already write).
template <int V, int L, bool kList>
__global__ void __launch_bounds__(256)
    pool_warp_kernel(DevTable t, const uint32_t* __restrict__ offsets,
                     const uint32_t* __restrict__ slots, uint32_t BF, uint64_t N, int mean,
                     float* __restrict__ out, uint64_t* __restrict__ out_rv64,
                     uint32_t* __restrict__ out_rv32, const uint32_t* __restrict__ glist,
                     const uint32_t* __restrict__ glist_n) {
  pdl_entry();
  constexpr int G = 32 / L;      // row groups per warp
  constexpr int kPer = 32 / G;   // one-listing segments per group per chunk
  constexpr int kB = kPer < 8 ? kPer : 8;
  const uint32_t lane = threadIdx.x & 31, grp = lane / L, ln = lane % L;
  const uint32_t D = t.D;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t count = kList ? *glist_n : BF;
  const bool want_rv = out_rv64 || out_rv32;
  for (uint64_t c0 = warp * 32; c0 < count; c0 += warps * 32) {
    const uint64_t k = c0 + lane;
    const bool live = k < count;
    const uint32_t sg = kList ? (live ? glist[k] : 0u) : static_cast<uint32_t>(k);
    const uint32_t a = live ? offsets[sg] : 0u, e = live ? offsets[sg + 1] : 0u;
    const bool one = live && e == a + 1;
    const uint32_t slot = one ? slots[a] : kInvalidSlot;
    if (want_rv && one) {
      const uint32_t v = slot_ok(t, slot) ? vt_read(t, slot).x : 0u;
      if (out_rv64) out_rv64[a] = v;
      if (out_rv32) out_rv32[a] = v;
    }
#pragma unroll
    for (int i0 = 0; i0 < kPer; i0 += kB) {
      float r[kB][V];
      uint32_t so[kB];
      bool on[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int j = (i0 + u) * G + grp;
        const uint32_t s = __shfl_sync(0xffffffffu, slot, j);
        so[u] = __shfl_sync(0xffffffffu, sg, j);
        on[u] = __shfl_sync(0xffffffffu, one ? 1 : 0, j) != 0;
        if (on[u] && slot_ok(t, s)) load_vec<V>(t.rows + static_cast<uint64_t>(s) * t.stride + ln * V, r[u]);
        else for (int q = 0; q < V; ++q) r[u][q] = 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (!on[u]) continue;
        float o[V];
#pragma unroll
        for (int q = 0; q < V; ++q) o[q] = __fadd_rn(r[u][q], 0.0f);
        store_vec_cs<V>(out + static_cast<uint64_t>(so[u]) * D + ln * V, o);
      }
    }
    // empty and several-listing segments: the g-th pending one goes to group g
    uint32_t rest = __ballot_sync(0xffffffffu, live && !one);
    while (rest) {
      uint32_t pick = rest;
      int mine = -1;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int j = pick ? __ffs(pick) - 1 : -1;
        if (g == static_cast<int>(grp)) mine = j;
        if (pick) pick &= pick - 1;
      }
      rest = pick;
      const int src = mine < 0 ? 0 : mine;
      const uint32_t msg = __shfl_sync(0xffffffffu, sg, src);
      const uint32_t ma = __shfl_sync(0xffffffffu, a, src);
      const uint32_t me = __shfl_sync(0xffffffffu, e, src);
      if (mine >= 0) {
        // Empty groups pool to zeros (embedding_worker.hpp:543): keep scale finite there.
        const double scale = (mean && me > ma) ? __drcp_rn(static_cast<double>(me - ma)) : 1.0;
        pool_general<V, L, false>(t, slots, msg, ma, me, scale, ln, out, out_rv64, out_rv32);
      }
    }
  }
}

// kList: pool only the groups listed in glist[0 .. *glist_n) (the exchange's groups that
// their rows' owners did not already write).
template <int V, int L, bool kGuard, bool kList>
__global__ void __launch_bounds__(256)
    pool_kernel(DevTable t, const uint32_t* __restrict__ offsets,
                const uint32_t* __restrict__ slots, uint32_t BF, uint64_t N, int mean,
                float* __restrict__ out, uint64_t* __restrict__ out_rv64,
                uint32_t* __restrict__ out_rv32, const uint32_t* __restrict__ glist,
                const uint32_t* __restrict__ glist_n) {
  pdl_entry();
  using G = Geo<V, L, kGuard>;
  const int ln = G::lane();
  const uint32_t D = t.D;
  const uint64_t groups = G::groups();
  const uint64_t count = kList ? *glist_n : BF;
  for (uint64_t k0 = G::group(); k0 < count; k0 += groups * kPoolILP) {
    uint64_t sg[kPoolILP];
    uint32_t a[kPoolILP], e[kPoolILP], spec[kPoolILP];
    bool live[kPoolILP];
#pragma unroll
    for (int u = 0; u < kPoolILP; ++u) {
      const uint64_t k = k0 + u * groups;
      live[u] = k < count;
      sg[u] = kList ? (live[u] ? glist[k] : 0u) : k;
      a[u] = live[u] ? offsets[sg[u]] : 0u;
      e[u] = live[u] ? offsets[sg[u] + 1] : 0u;
      spec[u] = (live[u] && sg[u] < N) ? slots[sg[u]] : 0u;  // right when a == sg
    }
    uint32_t s[kPoolILP];
    bool one[kPoolILP];
#pragma unroll
    for (int u = 0; u < kPoolILP; ++u) {
      one[u] = live[u] && e[u] == a[u] + 1;
      s[u] = one[u] ? (a[u] == sg[u] ? spec[u] : slots[a[u]]) : 0u;
    }
    // single-listing segments (every segment of a one-hot batch): rows in flight together
    if (!kGuard) {
      float r[kPoolILP][V];
      uint32_t ver[kPoolILP];
      const bool want_rv = out_rv64 || out_rv32;
#pragma unroll
      for (int u = 0; u < kPoolILP; ++u) {
        if (!one[u]) continue;
        const bool ok = slot_ok(t, s[u]);
        if (ok) {
          load_vec<V>(t.rows + static_cast<uint64_t>(s[u]) * t.stride + ln * V, r[u]);
        } else {
          for (int k = 0; k < V; ++k) r[u][k] = 0.0f;
        }
        ver[u] = (want_rv && ok && ln == 0) ? vt_read(t, s[u]).x : 0u;
      }
#pragma unroll
      for (int u = 0; u < kPoolILP; ++u) {
        if (!one[u]) continue;
        // acc = 0.0 + row (turns -0.0 into +0.0 exactly as the reference does), times the
        // scale of a one-listing group: 1.0/1 (mean) == 1.0 (sum).
        float o[V];
#pragma unroll
        for (int k = 0; k < V; ++k)
          o[k] = __double2float_rn(__dmul_rn(__dadd_rn(0.0, static_cast<double>(r[u][k])), 1.0));
        store_vec_cs<V>(out + sg[u] * D + ln * V, o);
        if (want_rv && ln == 0) {
          if (out_rv64) out_rv64[a[u]] = ver[u];
          if (out_rv32) out_rv32[a[u]] = ver[u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kPoolILP; ++u) {
      if (!live[u] || (one[u] && !kGuard)) continue;
      // Empty groups pool to zeros (embedding_worker.hpp:543): keep scale finite there.
      const double scale =
          (mean && e[u] > a[u]) ? __drcp_rn(static_cast<double>(e[u] - a[u])) : 1.0;
      pool_general<V, L, kGuard>(t, slots, sg[u], a[u], e[u], scale, ln, out, out_rv64,
                                 out_rv32);
    }
  }
}

// Read versions of a pulled batch, snapshotted when another push is about to mutate
// the table before this batch's own push (copy-on-write, table.cu protect_reads).
__global__ void snapshot_rv_kernel(DevTable t, const uint32_t* __restrict__ slots, uint64_t n,
                                   uint32_t* __restrict__ rv) {
  pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = slots[i];
    rv[i] = slot_ok(t, s) ? vt_read(t, s).x : 0u;
  }
}

void launch_snapshot_rv(const DevTable& t, const uint32_t* slots, uint64_t n, uint32_t* rv,
                        cudaStream_t st) {
  if (!n) return;
  launch(snapshot_rv_kernel, std::min<uint64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st, t, slots,
                                                                                     n, rv);
  HPS_LAUNCH_CHECK();
}

void launch_pool(const DevTable& t, const uint32_t* offsets, const uint32_t* slots, uint32_t BF,
                 uint64_t N, int mean, float* out, uint64_t* out_rv64, uint32_t* out_rv32,
                 cudaStream_t st, const uint32_t* glist, const uint32_t* glist_n) {
  if (!BF) return;
  HPS_DISPATCH_DIM(t.D, {
    if constexpr (!G) {
      // warp-cooperative: one resident wave of blocks strides over 32-segment chunks
      static int per_sm = 0;
      auto k = glist ? pool_warp_kernel<V, L, true> : pool_warp_kernel<V, L, false>;
      if (!per_sm) HPS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0));
      int dev = 0, sms = 148;
      HPS_CUDA(cudaGetDevice(&dev));
      HPS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const uint32_t blocks = static_cast<uint32_t>(std::max<uint64_t>(
          1, std::min<uint64_t>(ceil_div(BF, 256), static_cast<uint64_t>(sms) * per_sm)));
      launch(k, blocks, 256, 0, st, t, offsets, slots, BF, N, mean, out, out_rv64, out_rv32,
             glist, glist_n);
    } else {
      uint64_t groups_per_block = 256 / L;
      const uint32_t blocks = std::min<uint64_t>(ceil_div(BF, groups_per_block * kPoolILP),
                                                 148ull * 8);
      if (glist)
        launch(pool_kernel<V, L, G, true>, blocks, 256, 0, st, t, offsets, slots, BF, N, mean,
               out, out_rv64, out_rv32, glist, glist_n);
      else
        launch(pool_kernel<V, L, G, false>, blocks, 256, 0, st, t, offsets, slots, BF, N, mean,
               out, out_rv64, out_rv32, nullptr, nullptr);
    }
  });
  HPS_LAUNCH_CHECK();
}

}  // namespace hps
