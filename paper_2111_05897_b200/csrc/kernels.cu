// Hot-path kernels for the embedding lookup+update path (sm_100a).
//
// Every kernel is HBM-bound integer/byte or fp32/fp64 streaming work; nothing is a
// dense contraction, so there are no tensor cores here. Rows are
// moved with 128-bit vector loads by "row groups" of L lanes x V floats (L*V = D),
// grids are sized in multiples of the SM count and loop grid-stride.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "radix_sort.cuh"
#include "table.cuh"

namespace cg = cooperative_groups;

namespace hps {

namespace {

template <typename T>
__device__ __forceinline__ T ld_volatile(const T* p) {
  return *const_cast<const volatile T*>(p);
}

// Warp-aggregated atomicAdd on a u32 counter (one atomic per coalesced group).
__device__ __forceinline__ uint32_t agg_inc(uint32_t* ctr) {
  cg::coalesced_group g = cg::coalesced_threads();
  uint32_t base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(ctr, static_cast<uint32_t>(g.size()));
  return g.shfl(base, 0) + g.thread_rank();
}

// Claim a fresh row for id (lru_store.hpp:95-101: next slot below the high-water
// mark). No eviction on device: past capacity the insert fails and the sticky
// overflow counter is raised (exact LRU eviction is SURVEY.md §8f #3).
__device__ uint32_t alloc_slot(const DevTable& t, uint64_t id, uint32_t* new_slots,
                               uint32_t* new_count) {
  uint32_t slot = agg_inc(t.hwm);
  if (slot >= t.capacity) {
    atomicExch(&t.ctr[kCtrOverflow], 1ull);
    return kInvalidSlot;
  }
  t.slot_id[slot] = id;
  uint32_t q = agg_inc(new_count);
  new_slots[q] = slot;
  return slot;
}

// id -> slot with lazy insert (PsShard::find_or_init embedding_ps.hpp:417-434; the
// LruStore index lru_store.hpp:62-113). Linear probing on an open-addressing table
// of u64 keys; the inserting thread publishes the slot, racing readers of the same
// id spin on the (at most one in flight) publication.
__device__ uint32_t find_or_insert(const DevTable& t, uint64_t id, uint32_t* new_slots,
                                   uint32_t* new_count, bool insert) {
  if (id == kEmptyKey) {
    uint32_t s = ld_volatile(t.special);
    if (s == kSpecialAbsent) {
      if (!insert) return kPending;
      if (atomicCAS(t.special, kSpecialAbsent, kSpecialInserting) == kSpecialAbsent) {
        uint32_t slot = alloc_slot(t, id, new_slots, new_count);
        __threadfence();
        atomicExch(t.special, slot);
        return slot;
      }
    }
    while ((s = ld_volatile(t.special)) == kSpecialInserting) {
    }
    return s;
  }
  uint64_t h = mix64(id ^ kTableHashSalt) >> t.ht_shift;
  for (uint64_t probes = 0; probes <= t.ht_mask; ++probes) {
    uint64_t k = ld_volatile(&t.keys[h]);
    if (k == kEmptyKey) {
      if (!insert) return kPending;
      unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(&t.keys[h]),
                                         static_cast<unsigned long long>(kEmptyKey),
                                         static_cast<unsigned long long>(id));
      if (old == kEmptyKey) {
        uint32_t slot = alloc_slot(t, id, new_slots, new_count);
        __threadfence();
        atomicExch(&t.vals[h], slot);
        return slot;
      }
      k = old;
    }
    if (k == id) {
      uint32_t v;
      while ((v = ld_volatile(&t.vals[h])) == kPending) {
      }
      return v;
    }
    h = (h + 1) & t.ht_mask;
  }
  atomicExch(&t.ctr[kCtrOverflow], 1ull);
  return kInvalidSlot;
}

__device__ __forceinline__ bool slot_ok(const DevTable& t, uint32_t s) { return s < t.capacity; }

// ---- vector helpers for row groups -----------------------------------------------------

template <int V>
struct VecT;
template <>
struct VecT<1> {
  using T = float;
};
template <>
struct VecT<2> {
  using T = float2;
};
template <>
struct VecT<4> {
  using T = float4;
};

template <int V>
__device__ __forceinline__ void load_vec(const float* p, float (&v)[V]) {
  if constexpr (V == 4) {
    float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
  } else if constexpr (V == 2) {
    float2 x = *reinterpret_cast<const float2*>(p);
    v[0] = x.x, v[1] = x.y;
  } else {
    v[0] = *p;
  }
}

template <int V>
__device__ __forceinline__ void load_vec_stream(const float* p, float (&v)[V]) {
  if constexpr (V == 4) {
    float4 x = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
  } else if constexpr (V == 2) {
    float2 x = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = x.x, v[1] = x.y;
  } else {
    v[0] = __ldcs(p);
  }
}

template <int V>
__device__ __forceinline__ void store_vec(float* p, const float (&v)[V]) {
  if constexpr (V == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

template <int V>
__device__ __forceinline__ void store_vec_stream(float* p, const float (&v)[V]) {
  if constexpr (V == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  } else if constexpr (V == 2) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
  } else {
    __stcs(p, v[0]);
  }
}

// Row-group geometry: L lanes x V floats cover kSpan = L*V dims per chunk; a row of D
// dims takes ceil(D / kSpan) chunks (1 on the specialised paths). kGuard enables the
// d < D bounds check of the generic path.
template <int V, int L, bool kGuard>
struct Geo {
  static constexpr int kSpan = V * L;
  __device__ static int lane() { return threadIdx.x % L; }
  __device__ static uint64_t group() {
    return (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  }
  __device__ static uint64_t groups() { return static_cast<uint64_t>(gridDim.x) * blockDim.x / L; }
};

}  // namespace

// ---- routing --------------------------------------------------------------------------

__global__ void route_kernel(const uint64_t* __restrict__ ids, uint64_t n, uint32_t S,
                             uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = route_shard(ids[i], S);
}

void launch_route(const uint64_t* ids, uint64_t n, uint32_t S, uint32_t* out, cudaStream_t st) {
  if (!n) return;
  route_kernel<<<std::min<uint64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st>>>(ids, n, S, out);
  HPS_LAUNCH_CHECK();
}

// ---- CSR expansion: listing -> (sample*F + group) ---------------------------------------

__global__ void expand_groups_kernel(const uint32_t* __restrict__ offsets, uint32_t BF,
                                     uint32_t* __restrict__ lgrp) {
  for (uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x; sg < BF;
       sg += gridDim.x * blockDim.x) {
    uint32_t a = offsets[sg], e = offsets[sg + 1];
    for (uint32_t i = a; i < e; ++i) lgrp[i] = sg;
  }
}

void launch_expand_groups(const uint32_t* offsets, uint32_t BF, uint32_t* lgrp, cudaStream_t st) {
  if (!BF) return;
  expand_groups_kernel<<<std::min<uint64_t>(ceil_div(BF, 256), 148 * 16), 256, 0, st>>>(offsets, BF,
                                                                                    lgrp);
  HPS_LAUNCH_CHECK();
}

// ---- probe / lazy insert ------------------------------------------------------------------

__global__ void probe_kernel(DevTable t, const uint64_t* __restrict__ ids, uint64_t n,
                             uint32_t* __restrict__ slots, uint32_t* __restrict__ new_slots,
                             uint32_t* __restrict__ new_count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    slots[i] = find_or_insert(t, ids[i], new_slots, new_count, true);
  }
}

void launch_probe(const DevTable& t, const uint64_t* ids, uint64_t n, uint32_t* slots,
                  uint32_t* new_slots, uint32_t* new_count, cudaStream_t st) {
  if (!n) return;
  probe_kernel<<<ceil_div(n, 256), 256, 0, st>>>(t, ids, n, slots, new_slots, new_count);
  HPS_LAUNCH_CHECK();
}

// Lazy init of freshly inserted rows (embedding_ps.hpp:423-432): one warp per row,
// w[d] from the id's random stream, acc = 0, version 0, no step tag. The miss counter
// (embedding_ps.hpp:420) advances by the number of rows initialised.
__global__ void lazy_init_kernel(DevTable t, const uint32_t* __restrict__ new_slots,
                                 const uint32_t* __restrict__ new_count) {
  const uint32_t cnt = *new_count;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (warp == 0 && lane == 0 && cnt) atomicAdd(&t.ctr[kCtrMisses], (unsigned long long)cnt);
  const double limit = 1.0 / sqrt(static_cast<double>(t.D));
  const double lo = -limit, span = __dsub_rn(limit, lo);
  for (uint64_t q = warp; q < cnt; q += warps) {
    uint32_t slot = new_slots[q];
    uint64_t id = t.slot_id[slot];
    uint64_t seed = mix64(id ^ mix64(t.salts[route_shard(id, t.S)]));
    float* row = t.rows + static_cast<uint64_t>(slot) * t.stride;
    for (uint32_t d = lane; d < t.D; d += 32) {
      row[d] = init_value(seed, d, lo, span);
      row[t.D + d] = 0.0f;
    }
    if (lane == 0) {
      t.ver[slot] = 0;
      t.tag[slot] = kNoStep;
    }
  }
}

void launch_lazy_init(const DevTable& t, const uint32_t* new_slots, const uint32_t* new_count,
                      uint64_t max_new, int sms, cudaStream_t st) {
  if (!max_new) return;
  uint32_t blocks = std::min<uint64_t>(ceil_div(max_new, 8), (uint64_t)sms * 8);
  lazy_init_kernel<<<blocks, 256, 0, st>>>(t, new_slots, new_count);
  HPS_LAUNCH_CHECK();
}

// ---- gather (PsShard::lookup) / peek ---------------------------------------------------

__global__ void gather_kernel(DevTable t, const uint32_t* __restrict__ slots, uint64_t n,
                              float* __restrict__ out, uint64_t* __restrict__ out_ver) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    uint32_t s = slots[i];
    bool ok = slot_ok(t, s);
    const float* row = t.rows + static_cast<uint64_t>(ok ? s : 0) * t.stride;
    for (uint32_t d = lane; d < t.D; d += 32) out[i * t.D + d] = ok ? row[d] : 0.0f;
    if (out_ver && lane == 0) out_ver[i] = ok ? t.ver[s] : 0;
  }
}

void launch_gather(const DevTable& t, const uint32_t* slots, uint64_t n, float* out,
                   uint64_t* out_ver, cudaStream_t st) {
  if (!n) return;
  gather_kernel<<<std::min<uint64_t>(ceil_div(n, 8), 148 * 32), 256, 0, st>>>(t, slots, n, out,
                                                                          out_ver);
  HPS_LAUNCH_CHECK();
}

__global__ void peek_kernel(DevTable t, const uint64_t* __restrict__ ids, uint64_t n,
                            float* __restrict__ out_w, float* __restrict__ out_acc,
                            uint64_t* __restrict__ out_ver, uint8_t* __restrict__ out_present) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    uint32_t s = 0;
    if (lane == 0) s = find_or_insert(t, ids[i], nullptr, nullptr, false);
    s = __shfl_sync(0xffffffffu, s, 0);
    bool ok = slot_ok(t, s);
    const float* row = t.rows + static_cast<uint64_t>(ok ? s : 0) * t.stride;
    for (uint32_t d = lane; d < t.D; d += 32) {
      if (out_w) out_w[i * t.D + d] = ok ? row[d] : 0.0f;
      if (out_acc) out_acc[i * t.D + d] = ok ? row[t.D + d] : 0.0f;
    }
    if (lane == 0) {
      if (out_ver) out_ver[i] = ok ? t.ver[s] : 0;
      if (out_present) out_present[i] = ok ? 1 : 0;
    }
  }
}

void launch_peek(const DevTable& t, const uint64_t* ids, uint64_t n, float* out_w, float* out_acc,
                 uint64_t* out_ver, uint8_t* out_present, cudaStream_t st) {
  if (!n) return;
  peek_kernel<<<std::min<uint64_t>(ceil_div(n, 8), 148 * 32), 256, 0, st>>>(t, ids, n, out_w, out_acc,
                                                                        out_ver, out_present);
  HPS_LAUNCH_CHECK();
}

// ---- pooling (EmbeddingWorker::serve_pull, embedding_worker.hpp:541-557) ----------------
// One row group per (sample, group) segment: acc_d = sum over listings, in listing
// order, of (double)row[d] (duplicates counted); out = float(acc * scale) with
// scale = 1.0/n (mean) or 1.0 (sum); empty segments write zeros. Also emits the
// per-listing read version (PullResult::read_versions).

template <int V, int L, bool kGuard>
__global__ void __launch_bounds__(256)
    pool_kernel(DevTable t, const uint32_t* __restrict__ offsets,
                const uint32_t* __restrict__ slots, uint32_t BF, int mean,
                float* __restrict__ out, uint64_t* __restrict__ out_rv64,
                uint32_t* __restrict__ out_rv32) {
  using G = Geo<V, L, kGuard>;
  const int ln = G::lane();
  const uint32_t D = t.D;
  const int chunks = kGuard ? (D + G::kSpan - 1) / G::kSpan : 1;
  for (uint64_t sg = G::group(); sg < BF; sg += G::groups()) {
    const uint32_t a = offsets[sg], e = offsets[sg + 1];
    const double scale = mean ? __drcp_rn(static_cast<double>(e - a)) : 1.0;
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
          uint32_t v0 = slot_ok(t, s0) ? t.ver[s0] : 0, v1 = slot_ok(t, s1) ? t.ver[s1] : 0;
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
          uint32_t v0 = slot_ok(t, s0) ? t.ver[s0] : 0;
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
        store_vec_stream<V>(dst, o);
      }
    }
  }
}

// Dispatch on embedding dim: 128-bit row groups where D allows, else the generic
// one-float-per-lane path.
#define HPS_DISPATCH_DIM(D, ...)                      \
  do {                                                        \
    switch (D) {                                              \
      case 1: { constexpr int V = 1, L = 1; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 2: { constexpr int V = 2, L = 1; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 4: { constexpr int V = 4, L = 1; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 8: { constexpr int V = 4, L = 2; constexpr bool G = false; __VA_ARGS__; } break;   \
      case 16: { constexpr int V = 4, L = 4; constexpr bool G = false; __VA_ARGS__; } break;  \
      case 32: { constexpr int V = 4, L = 8; constexpr bool G = false; __VA_ARGS__; } break;  \
      case 64: { constexpr int V = 4, L = 16; constexpr bool G = false; __VA_ARGS__; } break; \
      case 128: { constexpr int V = 4, L = 32; constexpr bool G = false; __VA_ARGS__; } break; \
      default: { constexpr int V = 1, L = 32; constexpr bool G = true; __VA_ARGS__; } break;  \
    }                                                         \
  } while (0)

void launch_pool(const DevTable& t, const uint32_t* offsets, const uint32_t* slots, uint32_t BF,
                 int mean, float* out, uint64_t* out_rv64, uint32_t* out_rv32, cudaStream_t st) {
  if (!BF) return;
  HPS_DISPATCH_DIM(t.D, {
    uint64_t groups_per_block = 256 / L;
    uint32_t blocks = std::min<uint64_t>(ceil_div(BF, groups_per_block), 148ull * 16);
    pool_kernel<V, L, G><<<blocks, 256, 0, st>>>(t, offsets, slots, BF, mean, out, out_rv64,
                                                 out_rv32);
  });
  HPS_LAUNCH_CHECK();
}

// ---- segment heads over the slot-sorted listings -----------------------------------------
// head: first element of a slot's run (one unique row); pair head: first element of
// a (slot, sample) run -- one optimizer application per (sample, unique id).

__global__ void heads_kernel(const uint32_t* __restrict__ ss, const uint32_t* __restrict__ sl,
                             const uint32_t* __restrict__ lgrp, uint32_t F, uint64_t n,
                             bool direct, uint32_t* __restrict__ heads,
                             uint32_t* __restrict__ small) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = ss[p];
    bool head = p == 0 || ss[p - 1] != s;
    bool pair = head || direct;
    if (!pair) pair = lgrp[sl[p]] / F != lgrp[sl[p - 1]] / F;
    if (head) heads[agg_inc(&small[0])] = static_cast<uint32_t>(p);
    if (pair) agg_inc(&small[1]);
  }
}

void launch_heads(const uint32_t* ss, const uint32_t* sl, const uint32_t* lgrp, uint32_t F,
                  uint64_t n, bool direct, uint32_t* heads, uint32_t* small, cudaStream_t st) {
  if (!n) return;
  heads_kernel<<<std::min<uint64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st>>>(ss, sl, lgrp, F, n,
                                                                          direct, heads, small);
  HPS_LAUNCH_CHECK();
}

// ---- validation before mutation (embedding_ps.hpp:146-153) --------------------------------

__global__ void check_direct_kernel(const float* __restrict__ g, uint64_t n,
                                    unsigned long long* ctr) {
  bool bad = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&ctr[kCtrDivergence], 1ull);
}

void launch_check_direct(const float* grads, uint64_t n, unsigned long long* ctr,
                         cudaStream_t st) {
  if (!n) return;
  check_direct_kernel<<<std::min<uint64_t>(ceil_div(n, 256), 148 * 8), 256, 0, st>>>(grads, n, ctr);
  HPS_LAUNCH_CHECK();
}

// Batch validation: every gradient of a non-empty group feeds some contribution, so
// a non-finite one is a certain rejection. Finite gradients can still overflow a
// contribution in the float narrowing; per sample, |c| <= sum_g |grad_g|_inf * (n_g
// for sum, 1 for mean), and only when that bound reaches 2^127 is the exact dry run
// of the update kernel requested.
__global__ void check_batch_kernel(const float* __restrict__ grads,
                                   const uint32_t* __restrict__ offsets, uint32_t B, uint32_t F,
                                   uint32_t D, int mean, unsigned long long* ctr) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  bool bad = false, exact = false;
  for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; b < B; b += warps) {
    double bound = 0.0;
    for (uint32_t g = 0; g < F; ++g) {
      uint32_t n = offsets[b * F + g + 1] - offsets[b * F + g];
      if (!n) continue;
      const float* gr = grads + (b * F + g) * (uint64_t)D;
      float m = 0.0f;
      for (uint32_t d = lane; d < D; d += 32) {
        float x = __ldcs(gr + d);
        bad |= !isfinite(x);
        m = fmaxf(m, fabsf(x));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      bound += static_cast<double>(m) * (mean ? 1.0 : static_cast<double>(n));
    }
    exact |= bound >= 0x1.0p127;
  }
  bad = __syncthreads_or(bad);
  exact = __syncthreads_or(exact);
  if (threadIdx.x == 0) {
    if (bad) atomicExch(&ctr[kCtrDivergence], 1ull);
    if (exact) atomicExch(&ctr[kCtrNeedExact], 1ull);
  }
}

void launch_check_batch(const float* grads, const uint32_t* offsets, uint32_t B, uint32_t F,
                        uint32_t D, int mean, unsigned long long* ctr, cudaStream_t st) {
  if (!B) return;
  check_batch_kernel<<<std::min<uint64_t>(ceil_div(B, 8), 148 * 8), 256, 0, st>>>(grads, offsets, B,
                                                                             F, D, mean, ctr);
  HPS_LAUNCH_CHECK();
}

// ---- ordered fused optimizer update ------------------------------------------------------
// One row group per unique row (a slot run of the slot-sorted listings). The group
// walks the run in apply order; consecutive listings of one sample form one pair
// whose contribution is the fp64 chain-rule sum (push_to_shards :728-743, product
// rounded then added), narrowed to float and applied once (apply_one
// embedding_ps.hpp:436-449, each op individually rounded). The row [w | acc] stays in
// registers across the whole run and is written back once. Versions / delays follow
// count_delay + bump_version (embedding_ps.hpp:454-488) with the latest bump tag
// standing in for the 16-deep ring (exact when steps apply in order, which the
// stream-ordered pipeline guarantees).
template <int V, int L, bool kGuard, bool kDirect>
__global__ void __launch_bounds__(256)
    update_kernel(DevTable t, UpdateArgs a) {
  using G = Geo<V, L, kGuard>;
  __shared__ unsigned long long s_hist[17];
  __shared__ unsigned int s_resets, s_max;
  if (threadIdx.x < 17) s_hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_resets = 0, s_max = 0;
  __syncthreads();
  const bool gated = ld_volatile(&t.ctr[kCtrDivergence]) | ld_volatile(&t.ctr[kCtrOverflow]) |
                     (a.dry_run ? !ld_volatile(&t.ctr[kCtrNeedExact]) : 0ull);
  const int ln = G::lane();
  const uint32_t D = t.D;
  const int chunks = kGuard ? (D + G::kSpan - 1) / G::kSpan : 1;
  const uint32_t U = gated ? 0u : a.small[0];
  const bool adagrad = t.opt == HPS_ADAGRAD;
  bool bad = false;
  for (uint64_t u = G::group(); u < U; u += G::groups()) {
    const uint32_t p0 = a.heads[u];
    const uint32_t slot = a.sorted_slot[p0];
    if (!slot_ok(t, slot)) continue;
    float* row = t.rows + static_cast<uint64_t>(slot) * t.stride;
    for (int c = 0; c < chunks; ++c) {
      const uint32_t d0 = c * G::kSpan + ln * V;
      const bool dims_ok = !kGuard || d0 < D;
      float w[V], acc[V];
      if (dims_ok && !a.dry_run) {
        load_vec<V>(row + d0, w);
        if (adagrad) load_vec<V>(row + D + d0, acc);
      }
      uint32_t ver = t.ver[slot], tag = t.tag[slot];
      uint64_t p = p0;
      while (p < a.n && a.sorted_slot[p] == slot) {
        float cval[V];
        uint64_t rv = 0;
        uint32_t entry = a.sorted_listing[p];
        if constexpr (kDirect) {
          if (dims_ok) {
            if (kGuard) cval[0] = a.grads[(uint64_t)entry * D + d0];
            else load_vec<V>(a.grads + (uint64_t)entry * D + d0, cval);
          }
          if (a.tracked) rv = a.rv64 ? a.rv64[entry] : a.rv32[entry];
          ++p;
        } else {
          if (a.tracked) rv = a.rv32 ? a.rv32[entry] : a.rv64[entry];
          uint32_t lg = a.lgrp[entry];
          const uint32_t b = lg / a.F;
          double sum[V];
#pragma unroll
          for (int k = 0; k < V; ++k) sum[k] = 0.0;
          while (true) {
            const double scale =
                a.mean ? __drcp_rn(static_cast<double>(a.offsets[lg + 1] - a.offsets[lg])) : 1.0;
            if (dims_ok) {
              float gv[V];
              if (kGuard) gv[0] = a.grads[(uint64_t)lg * D + d0];
              else load_vec<V>(a.grads + (uint64_t)lg * D + d0, gv);
#pragma unroll
              for (int k = 0; k < V; ++k)
                sum[k] = __dadd_rn(sum[k], __dmul_rn(static_cast<double>(gv[k]), scale));
            }
            ++p;
            if (p >= a.n || a.sorted_slot[p] != slot) break;
            uint32_t lg2 = a.lgrp[a.sorted_listing[p]];
            if (lg2 / a.F != b) break;
            lg = lg2;
          }
#pragma unroll
          for (int k = 0; k < V; ++k) cval[k] = __double2float_rn(sum[k]);
        }
        if (a.dry_run) {
          if (dims_ok)
#pragma unroll
            for (int k = 0; k < V; ++k) bad |= !isfinite(cval[k]);
          continue;
        }
        if (c == 0) {
          uint32_t delay = 0;
          if (a.tracked) {
            if (rv > ver) {
              if (ln == 0) atomicAdd(&s_resets, 1u);
            } else {
              uint64_t gap = ver - rv;
              delay = static_cast<uint32_t>(gap < kTagRing ? gap : kTagRing);
              if (gap > 0 && tag != kNoStep && tag >= a.step_tag) delay -= 1;
            }
            if (!(ver > 0 && tag == a.step_tag)) {
              ++ver;
              tag = a.step_tag;
            }
            if (ln == 0) {
              atomicAdd(&s_hist[delay < 16 ? delay : 16], 1ull);
              atomicMax(&s_max, delay);
              if (kDirect && a.out_delays) a.out_delays[entry] = delay;
            }
          } else {
            ++ver;
          }
        }
        if (dims_ok) {
          if (adagrad) {
#pragma unroll
            for (int k = 0; k < V; ++k) {
              acc[k] = __fadd_rn(acc[k], __fmul_rn(cval[k], cval[k]));
              float den = __fadd_rn(__fsqrt_rn(acc[k]), kAdagradEps);
              w[k] = __fsub_rn(w[k], __fdiv_rn(__fmul_rn(a.lr, cval[k]), den));
            }
          } else {
#pragma unroll
            for (int k = 0; k < V; ++k) w[k] = __fsub_rn(w[k], __fmul_rn(a.lr, cval[k]));
          }
        }
      }
      if (a.dry_run) continue;
      if (dims_ok) {
        if (kGuard) {
          row[d0] = w[0];
          if (adagrad) row[D + d0] = acc[0];
        } else {
          store_vec<V>(row + d0, w);
          if (adagrad) store_vec<V>(row + D + d0, acc);
        }
      }
      if (c == 0 && ln == 0) {
        t.ver[slot] = ver;
        t.tag[slot] = tag;
      }
    }
  }
  if (a.dry_run) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&t.ctr[kCtrDivergence], 1ull);
    return;
  }
  __syncthreads();
  if (a.tracked) {
    if (threadIdx.x < 17 && s_hist[threadIdx.x])
      atomicAdd(&t.ctr[kCtrDelayHist + threadIdx.x], s_hist[threadIdx.x]);
    if (threadIdx.x == 0) {
      if (s_resets) atomicAdd(&t.ctr[kCtrClockResets], (unsigned long long)s_resets);
      if (s_max) atomicMax(&t.ctr[kCtrMaxDelay], (unsigned long long)s_max);
    }
  }
}

void launch_update(const DevTable& t, const UpdateArgs& a, bool direct, int sms, cudaStream_t st) {
  if (!a.n) return;
  HPS_DISPATCH_DIM(t.D, {
    uint64_t groups_per_block = 256 / L;
    uint32_t blocks = std::min<uint64_t>(ceil_div(a.n, groups_per_block), (uint64_t)sms * 8);
    if (direct) update_kernel<V, L, G, true><<<blocks, 256, 0, st>>>(t, a);
    else update_kernel<V, L, G, false><<<blocks, 256, 0, st>>>(t, a);
  });
  HPS_LAUNCH_CHECK();
}

// ---- small helpers --------------------------------------------------------------------

__global__ void iota_kernel(uint32_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<uint32_t>(i);
}

void launch_iota(uint32_t* out, uint64_t n, cudaStream_t st) {
  if (!n) return;
  iota_kernel<<<std::min<uint64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st>>>(out, n);
  HPS_LAUNCH_CHECK();
}

__global__ void copy_u32_kernel(const uint32_t* __restrict__ s, uint32_t* __restrict__ d,
                                uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

void launch_copy_u32(const uint32_t* src, uint32_t* dst, uint64_t n, cudaStream_t st) {
  if (!n) return;
  copy_u32_kernel<<<std::min<uint64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st>>>(src, dst, n);
  HPS_LAUNCH_CHECK();
}

__global__ void sample_order_kernel(const uint64_t* __restrict__ sk, uint32_t B,
                                    uint64_t* __restrict__ keys, uint32_t* __restrict__ perm) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    keys[b] = sk[b];
    perm[b] = b;
  }
}

void launch_sample_order(const uint64_t* sk, uint32_t B, uint64_t* keys, uint32_t* perm,
                         cudaStream_t st) {
  if (!B) return;
  sample_order_kernel<<<ceil_div(B, 256), 256, 0, st>>>(sk, B, keys, perm);
  HPS_LAUNCH_CHECK();
}

__global__ void sample_lengths_kernel(const uint32_t* __restrict__ perm,
                                      const uint32_t* __restrict__ off, uint32_t B, uint32_t F,
                                      uint32_t* __restrict__ lens) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < B; r += gridDim.x * blockDim.x) {
    uint64_t b = perm[r];
    lens[r] = off[(b + 1) * F] - off[b * F];
  }
}

void launch_sample_lengths(const uint32_t* perm, const uint32_t* off, uint32_t B, uint32_t F,
                           uint32_t* lens, cudaStream_t st) {
  if (!B) return;
  sample_lengths_kernel<<<ceil_div(B, 256), 256, 0, st>>>(perm, off, B, F, lens);
  HPS_LAUNCH_CHECK();
}

void launch_scan_inplace(uint32_t* data, uint32_t n, uint32_t* total, cudaStream_t st) {
  radix::scan_digits<<<1, 1024, 0, st>>>(data, n, total);
  HPS_LAUNCH_CHECK();
}

__global__ void permuted_listing_kernel(const uint32_t* __restrict__ perm,
                                        const uint32_t* __restrict__ starts,
                                        const uint32_t* __restrict__ off,
                                        const uint32_t* __restrict__ slots, uint32_t B,
                                        uint32_t F, uint32_t* __restrict__ keys,
                                        uint32_t* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < B; r += warps) {
    uint64_t b = perm[r];
    uint32_t a = off[b * F], e = off[(b + 1) * F], dst = starts[r];
    for (uint32_t k = lane; a + k < e; k += 32) {
      keys[dst + k] = slots[a + k];
      vals[dst + k] = a + k;
    }
  }
}

void launch_permuted_listing(const uint32_t* perm, const uint32_t* starts, const uint32_t* off,
                             const uint32_t* slots, uint32_t B, uint32_t F, uint32_t* keys,
                             uint32_t* vals, cudaStream_t st) {
  if (!B) return;
  permuted_listing_kernel<<<std::min<uint64_t>(ceil_div(B, 8), 148 * 16), 256, 0, st>>>(
      perm, starts, off, slots, B, F, keys, vals);
  HPS_LAUNCH_CHECK();
}

__global__ void add_counter_kernel(unsigned long long* ctr, int idx, const uint32_t* src) {
  atomicAdd(&ctr[idx], (unsigned long long)*src);
}

void launch_add_counter_from(unsigned long long* ctr, int idx, const uint32_t* src,
                             cudaStream_t st) {
  add_counter_kernel<<<1, 1, 0, st>>>(ctr, idx, src);
  HPS_LAUNCH_CHECK();
}

}  // namespace hps
