// Hot-path kernels except the ordered update (update.cu) and the radix sort
// (radix_sort.cuh): routing, CSR expansion, id-index probe with lazy insert, lazy
// init, gather / peek, fp64 pooling and the pre-mutation validation.
//
// Everything here is HBM-bound integer/byte or fp32/fp64 streaming work; nothing is a
// dense contraction, so there are no tensor cores. Rows move as
// 128-bit vectors by "row groups" of L lanes x V floats (vec.cuh).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "radix_sort.cuh"
#include "table.cuh"
#include "vec.cuh"

namespace cg = cooperative_groups;

namespace hps {

namespace {

// Warp-aggregated atomicAdd on a u32 counter (one atomic per coalesced group).
__device__ __forceinline__ uint32_t agg_inc(uint32_t* ctr) {
  cg::coalesced_group g = cg::coalesced_threads();
  uint32_t base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(ctr, static_cast<uint32_t>(g.size()));
  return g.shfl(base, 0) + g.thread_rank();
}

// find_or_init's initialisation (embedding_ps.hpp:424-432) of one row by one thread:
// weights from the id's random stream, accumulators 0, version 0, no step tag.
__device__ void init_row(const DevTable& t, uint64_t id, uint32_t slot) {
  const uint64_t seed = mix64(id ^ mix64(t.salts[route_shard(id, t.S)]));
  const double limit = 1.0 / sqrt(static_cast<double>(t.D));
  const double lo = -limit, span = __dsub_rn(limit, lo);
  float* row = t.rows + static_cast<uint64_t>(slot) * t.stride;
  for (uint32_t d = 0; d < t.D; ++d) {
    row[d] = init_value(seed, d, lo, span);
    row[t.D + d] = (t.svt && d < 64 && (d & 3) >= 2) ? -0.0f : 0.0f;
  }
  if (t.ring)
    for (uint32_t k = 0; k < kTagRing; ++k) t.ring[static_cast<uint64_t>(slot) * kTagRing + k] = kNoStep;
  if (!t.svt) t.vt[slot] = make_uint2(0u, kNoStep);
}

// Claim a fresh row for id (lru_store.hpp:95-101: next slot below the high-water
// mark). No eviction on device: past capacity the insert fails and the sticky
// overflow counter is raised (exact LRU eviction is SURVEY.md §8f #3).
__device__ uint32_t alloc_slot(const DevTable& t, uint64_t id, uint32_t* new_slots,
                               uint32_t* new_count) {
  uint32_t slot;
  if (t.lru) {
    // the shard's own slot range (the host checked the call fits before taking this
    // parallel path; otherwise lru.cu's sequential path evicts)
    const uint32_t s = route_shard(id, t.S);
    const uint32_t k = atomicAdd(&t.shard_hwm[s], 1u);
    if (k >= t.shard_cap) {
      atomicExch(&t.ctr[kCtrOverflow], 1ull);
      return kInvalidSlot;
    }
    slot = s * t.shard_cap + k;
  } else {
    slot = agg_inc(t.hwm);
    if (slot >= t.capacity) {
      atomicExch(&t.ctr[kCtrOverflow], 1ull);
      return kInvalidSlot;
    }
  }
  t.slot_id[slot] = id;
  if (!new_slots) {  // initialise the row here instead of queueing it for lazy_init_kernel
    init_row(t, id, slot);
    cg::coalesced_group g = cg::coalesced_threads();
    if (g.thread_rank() == 0) atomicAdd(&t.ctr[kCtrMisses], static_cast<unsigned long long>(g.size()));
    return slot;
  }
  uint32_t q = agg_inc(new_count);
  new_slots[q] = slot;
  return slot;
}

// id -> slot with lazy insert (PsShard::find_or_init embedding_ps.hpp:417-434; the
// LruStore index lru_store.hpp:62-113). Linear probing over 16-byte {key, slot}
// entries; the inserting thread publishes the slot, racing readers of the same id
// spin on that (single, in-flight) publication.
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
    HashEntry* e = &t.ht[h];
    // one 16-byte load brings key and slot together
    unsigned long long k, sv;
    asm volatile("ld.volatile.v2.u64 {%0, %1}, [%2];" : "=l"(k), "=l"(sv) : "l"(e));
    if (k == kEmptyKey) {
      if (!insert) return kPending;
      unsigned long long old = atomicCAS(&e->key, static_cast<unsigned long long>(kEmptyKey),
                                         static_cast<unsigned long long>(id));
      if (old == kEmptyKey) {
        uint32_t slot = alloc_slot(t, id, new_slots, new_count);
        __threadfence();
        atomicExch(&e->slot, slot);
        return slot;
      }
      k = old;
      sv = kPending;
    }
    if (k == id) {
      uint32_t v = static_cast<uint32_t>(sv);
      while (v == kPending) v = ld_volatile(&e->slot);
      return v;
    }
    h = (h + 1) & t.ht_mask;
  }
  atomicExch(&t.ctr[kCtrOverflow], 1ull);
  return kInvalidSlot;
}

}  // namespace

// ---- routing --------------------------------------------------------------------------

__global__ void route_kernel(const uint64_t* __restrict__ ids, uint64_t n, uint32_t S,
                             uint32_t* __restrict__ out) {
  pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = route_shard(ids[i], S);
}

void launch_route(const uint64_t* ids, uint64_t n, uint32_t S, uint32_t* out, cudaStream_t st) {
  if (!n) return;
  launch(route_kernel, std::min<uint64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st, ids, n, S, out);
  HPS_LAUNCH_CHECK();
}

// ---- CSR expansion: listing -> (sample*F + group) ---------------------------------------

// kind (optional): bit 2 marks a listing that is alone in its group (its contribution
// scale is 1 under mean pooling too), for the plan (plan.cu) and update_single.
// copy (optional): also keep a copy of the offsets; zero[0 .. nzero): scalars to clear
// (the batch's counters and flags) -- one launch instead of a copy and a memset node.
__global__ void expand_groups_kernel(const uint32_t* __restrict__ offsets, uint32_t BF,
                                     uint32_t* __restrict__ lgrp, uint8_t* __restrict__ kind,
                                     uint32_t* __restrict__ copy, uint32_t* __restrict__ zero,
                                     uint32_t nzero) {
  pdl_entry();
  if (blockIdx.x == 0)
    for (uint32_t k = threadIdx.x; k < nzero; k += blockDim.x) zero[k] = 0;
  for (uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x; sg < BF;
       sg += gridDim.x * blockDim.x) {
    uint32_t a = offsets[sg], e = offsets[sg + 1];
    if (copy) {
      copy[sg] = a;
      if (sg == BF - 1) copy[BF] = e;
    }
    for (uint32_t i = a; i < e; ++i) {
      lgrp[i] = sg;
      if (kind) kind[i] = e - a == 1 ? kKindAlone : 0;
    }
  }
}

void launch_expand_groups(const uint32_t* offsets, uint32_t BF, uint32_t* lgrp, cudaStream_t st,
                          uint8_t* kind, uint32_t* copy, uint32_t* zero, uint32_t nzero) {
  if (!BF && !nzero) return;
  launch(expand_groups_kernel, std::max<uint32_t>(1, std::min<uint64_t>(ceil_div(BF, 256), 148 * 16)),
         256, 0, st, offsets, BF, lgrp, kind, copy, zero, nzero);
  HPS_LAUNCH_CHECK();
}

// ---- probe / lazy insert ------------------------------------------------------------------

__global__ void __launch_bounds__(256)
    probe_kernel(DevTable t, const uint64_t* __restrict__ ids, uint64_t n,
                 uint32_t* __restrict__ slots, uint32_t* __restrict__ sort_keys,
                 uint32_t* __restrict__ sort_vals, uint32_t* __restrict__ new_slots,
                 uint32_t* __restrict__ new_count, bool plan, const uint32_t* n_dev) {
  pdl_entry();
  // n_dev: the live listing count is device-side (<= n); listings past it get no row.
  const uint64_t n_live = n_dev ? min(n, static_cast<uint64_t>(*n_dev)) : n;
  // One listing per thread (two back to back measured slower beside the pooling: the
  // register runs on the side, and fewer, longer-lived warps cost the critical path
  // more, profiles/r2_check_probe_ab.txt).
  constexpr int kProbeILP = 1;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x * kProbeILP + threadIdx.x;
  uint64_t id[kProbeILP];
  ulonglong2 kv[kProbeILP];
#pragma unroll
  for (int k = 0; k < kProbeILP; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * blockDim.x;
    id[k] = i < n_live ? ids[i] : kEmptyKey;
  }
#pragma unroll
  for (int k = 0; k < kProbeILP; ++k) {
    const uint64_t h = mix64(id[k] ^ kTableHashSalt) >> t.ht_shift;
    kv[k] = id[k] != kEmptyKey ? __ldcg(reinterpret_cast<const ulonglong2*>(t.ht + h))
                               : make_ulonglong2(0, 0);
  }
#pragma unroll
  for (int k = 0; k < kProbeILP; ++k) {
    const uint64_t i = base + static_cast<uint64_t>(k) * blockDim.x;
    if (i >= n) break;
    uint32_t s;
    if (i >= n_live)
      s = kInvalidSlot;
    else if (id[k] != kEmptyKey && kv[k].x == id[k] && static_cast<uint32_t>(kv[k].y) != kPending)
      s = static_cast<uint32_t>(kv[k].y);  // hit in the home entry
    else
      s = find_or_insert(t, id[k], new_slots, new_count, true);
    slots[i] = s;
    // Batch plan (plan.cu): a row seen before in this batch is "multi". Both bitmaps
    // are L2-resident, so this is one L2 atomic round trip.
    if (plan && slot_ok(t, s)) {
      const uint32_t bit = 1u << (s & 31);
      if (atomicOr(&t.seen[s >> 5], bit) & bit) atomicOr(&t.multi[s >> 5], bit);
    }
    if (sort_keys) {
      sort_keys[i] = s;
      sort_vals[i] = static_cast<uint32_t>(i);
    }
  }
}

void launch_probe(const DevTable& t, const uint64_t* ids, uint64_t n, uint32_t* slots,
                  uint32_t* sort_keys, uint32_t* sort_vals, uint32_t* new_slots,
                  uint32_t* new_count, bool plan, cudaStream_t st, const uint32_t* n_dev) {
  if (!n) return;
  launch(probe_kernel, ceil_div(n, 256), 256, 0, st, t, ids, n, slots, sort_keys, sort_vals,
         new_slots, new_count, plan, n_dev);
  HPS_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256)
    probe_regions_kernel(DevTable t, const uint64_t* __restrict__ ids, uint64_t stride,
                         const XHdr* __restrict__ hdr, uint32_t* __restrict__ slots,
                         uint64_t* __restrict__ ids_copy, uint32_t* __restrict__ cnt_copy,
                         uint32_t* __restrict__ new_slots, uint32_t* __restrict__ new_count) {
  pdl_entry();
  const uint32_t r = blockIdx.y;
  const uint64_t n = ld_volatile(&hdr->fwd_cnt[r]);
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt_copy[r] = static_cast<uint32_t>(n);
  const uint64_t* rid = ids + r * stride;
  uint32_t* rs = slots + r * stride;
  uint64_t* rc = ids_copy + r * stride;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = rid[j];
    rc[j] = id;
    rs[j] = find_or_insert(t, id, new_slots, new_count, true);
  }
}

void launch_probe_regions(const DevTable& t, const uint64_t* ids, uint64_t stride, uint32_t W,
                          const XHdr* hdr, uint32_t* slots, uint64_t* ids_copy,
                          uint32_t* cnt_copy, uint32_t* new_slots, uint32_t* new_count, int sms,
                          cudaStream_t st) {
  if (!stride || !W) return;
  const uint32_t bx = static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(stride, 256), (uint64_t)sms * 8 / W + 1)));
  launch(probe_regions_kernel, dim3(bx, W), 256, 0, st, t, ids, stride, hdr, slots, ids_copy,
                                                    cnt_copy, new_slots, new_count);
  HPS_LAUNCH_CHECK();
}

// Empty index: every key kEmptyKey, every slot kPending (both all-ones).
void launch_ht_clear(const DevTable& t, cudaStream_t st) {
  HPS_CUDA(cudaMemsetAsync(t.ht, 0xff, (t.ht_mask + 1) * sizeof(HashEntry), st));
}

// Lazy init of freshly inserted rows (embedding_ps.hpp:423-432): one warp per row,
// w[d] from the id's random stream, acc = 0, version 0, no step tag. The miss counter
// (embedding_ps.hpp:420) advances by the number of rows initialised.
__global__ void lazy_init_kernel(DevTable t, const uint32_t* __restrict__ new_slots,
                                 const uint32_t* __restrict__ new_count) {
  pdl_entry();
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
      // svt: version 0, tag kNoStep (all ones) -> sign bits of elements 4l+2, 4l+3
      row[t.D + d] = (t.svt && d < 64 && (d & 3) >= 2) ? -0.0f : 0.0f;
    }
    if (t.ring && lane < kTagRing) t.ring[static_cast<uint64_t>(slot) * kTagRing + lane] = kNoStep;
    if (lane == 0 && !t.svt) t.vt[slot] = make_uint2(0u, kNoStep);
  }
}

void launch_lazy_init(const DevTable& t, const uint32_t* new_slots, const uint32_t* new_count,
                      uint64_t max_new, int sms, cudaStream_t st) {
  if (!max_new) return;
  uint32_t blocks = std::min<uint64_t>(ceil_div(max_new, 8), (uint64_t)sms * 8);
  launch(lazy_init_kernel, blocks, 256, 0, st, t, new_slots, new_count);
  HPS_LAUNCH_CHECK();
}

// ---- gather (PsShard::lookup) / peek ---------------------------------------------------

// One row group (L lanes x V floats, 128-bit accesses) per id, kGatherILP ids in flight
// per group: slot -> row + header are two dependent round trips per id.
constexpr int kGatherILP = 2;

template <int V, int L, bool kGuard>
__global__ void __launch_bounds__(256)
    gather_kernel(DevTable t, const uint32_t* __restrict__ slots, uint64_t n,
                  float* __restrict__ out, uint64_t* __restrict__ out_ver) {
  pdl_entry();
  using G = Geo<V, L, kGuard>;
  const int ln = G::lane();
  const uint32_t D = t.D;
  const uint64_t groups = G::groups();
  for (uint64_t i0 = G::group(); i0 < n; i0 += groups * kGatherILP) {
    uint32_t s[kGatherILP];
#pragma unroll
    for (int u = 0; u < kGatherILP; ++u) {
      const uint64_t i = i0 + u * groups;
      s[u] = i < n ? slots[i] : kInvalidSlot;
    }
    if constexpr (!kGuard) {
      float r[kGatherILP][V];
      uint32_t ver[kGatherILP];
#pragma unroll
      for (int u = 0; u < kGatherILP; ++u) {
        const bool ok = slot_ok(t, s[u]);
        if (ok) load_vec<V>(t.rows + static_cast<uint64_t>(s[u]) * t.stride + ln * V, r[u]);
        else for (int k = 0; k < V; ++k) r[u][k] = 0.0f;
        ver[u] = (out_ver && ok && ln == 0) ? vt_read(t, s[u]).x : 0u;
      }
#pragma unroll
      for (int u = 0; u < kGatherILP; ++u) {
        const uint64_t i = i0 + u * groups;
        if (i >= n) continue;
        store_vec_cs<V>(out + i * D + ln * V, r[u]);
        if (out_ver && ln == 0) out_ver[i] = ver[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < kGatherILP; ++u) {
        const uint64_t i = i0 + u * groups;
        if (i >= n) continue;
        const bool ok = slot_ok(t, s[u]);
        const float* row = t.rows + static_cast<uint64_t>(ok ? s[u] : 0) * t.stride;
        for (uint32_t d = ln; d < D; d += L) out[i * D + d] = ok ? row[d] : 0.0f;
        if (out_ver && ln == 0) out_ver[i] = ok ? vt_read(t, s[u]).x : 0;
      }
    }
  }
}

void launch_gather(const DevTable& t, const uint32_t* slots, uint64_t n, float* out,
                   uint64_t* out_ver, cudaStream_t st) {
  if (!n) return;
  HPS_DISPATCH_DIM(t.D, {
    const uint64_t per_block = (256 / L) * kGatherILP;
    const uint32_t blocks = static_cast<uint32_t>(
        std::min<uint64_t>(ceil_div(n, per_block), 148ull * 48));
    launch(gather_kernel<V, L, G>, blocks, 256, 0, st, t, slots, n, out, out_ver);
  });
  HPS_LAUNCH_CHECK();
}

__global__ void peek_kernel(DevTable t, const uint64_t* __restrict__ ids, uint64_t n,
                            float* __restrict__ out_w, float* __restrict__ out_acc,
                            uint64_t* __restrict__ out_ver, uint8_t* __restrict__ out_present) {
  pdl_entry();
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
      if (out_acc) out_acc[i * t.D + d] = ok ? (t.svt ? fabsf(row[t.D + d]) : row[t.D + d]) : 0.0f;
    }
    if (lane == 0) {
      if (out_ver) out_ver[i] = ok ? vt_read(t, s).x : 0;
      if (out_present) out_present[i] = ok ? 1 : 0;
    }
  }
}

void launch_peek(const DevTable& t, const uint64_t* ids, uint64_t n, float* out_w, float* out_acc,
                 uint64_t* out_ver, uint8_t* out_present, cudaStream_t st) {
  if (!n) return;
  launch(peek_kernel, std::min<uint64_t>(ceil_div(n, 8), 148 * 32), 256, 0, st, 
      t, ids, n, out_w, out_acc, out_ver, out_present);
  HPS_LAUNCH_CHECK();
}

// ---- checkpoint images (PsShard::save_checkpoint / adopt, embedding_ps.hpp:222-260,390-402)

// Rows of `slots` as the HPS1 body stores them: [w D | acc D] (accumulators without the
// svt sign bits) and the version. One warp per row.
__global__ void ckpt_gather_kernel(DevTable t, const uint32_t* __restrict__ slots, uint64_t n,
                                   float* __restrict__ rows2d, uint64_t* __restrict__ vers) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const uint32_t s = slots[i];
    const float* row = t.rows + static_cast<uint64_t>(s) * t.stride;
    float* o = rows2d + i * 2 * t.D;
    for (uint32_t d = lane; d < t.D; d += 32) {
      o[d] = row[d];
      o[t.D + d] = t.svt ? fabsf(row[t.D + d]) : row[t.D + d];
    }
    if (lane == 0) vers[i] = vt_read(t, s).x;
  }
}

// Adopt rows: find-or-insert each id, then write its weights, accumulators and version;
// the latest-bump tag is reset (adopt_locked refills the tag ring with kNoStep, :400).
// at (LRU mode, optional): the slot each row takes (the image's own slot in its shard's
// range) and its stamp; the index entry is inserted for that slot.
__device__ void insert_at(const DevTable& t, uint64_t id, uint32_t slot) {
  if (id == kEmptyKey) {
    *t.special = slot;
    return;
  }
  for (uint64_t h = mix64(id ^ kTableHashSalt) >> t.ht_shift, k = 0; k <= t.ht_mask;
       ++k, h = (h + 1) & t.ht_mask) {
    if (atomicCAS(&t.ht[h].key, static_cast<unsigned long long>(kEmptyKey),
                  static_cast<unsigned long long>(id)) == kEmptyKey) {
      t.ht[h].slot = slot;
      return;
    }
  }
  atomicExch(&t.ctr[kCtrOverflow], 1ull);
}

__global__ void ckpt_restore_kernel(DevTable t, const uint64_t* __restrict__ ids,
                                    const float* __restrict__ rows2d,
                                    const uint64_t* __restrict__ vers, uint64_t n,
                                    uint32_t* new_slots, uint32_t* new_count,
                                    const uint32_t* __restrict__ at,
                                    const unsigned long long* __restrict__ stamps) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    uint32_t s = 0;
    if (lane == 0) {
      if (at) {
        s = at[i];
        insert_at(t, ids[i], s);
        t.slot_id[s] = ids[i];
        t.stamp[s] = stamps[i];
      } else {
        s = find_or_insert(t, ids[i], new_slots, new_count, true);
      }
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    if (!slot_ok(t, s)) continue;  // capacity: kCtrOverflow is set
    const uint32_t ver = static_cast<uint32_t>(vers[i]);
    float* row = t.rows + static_cast<uint64_t>(s) * t.stride;
    const float* src = rows2d + i * 2 * t.D;
    for (uint32_t d = lane; d < t.D; d += 32) {
      row[d] = src[d];
      float a = src[t.D + d];
      if (t.svt && d < 64) {
        const uint32_t l = d >> 2, k = d & 3;
        const uint32_t word = k == 0 ? (ver & 0xffffu) : k == 1 ? (ver >> 16)
                            : k == 2 ? (kNoStep & 0xffffu) : (kNoStep >> 16);
        a = with_sign(a, (word >> l) & 1u);
      }
      row[t.D + d] = a;
    }
    if (t.ring && lane < kTagRing) t.ring[static_cast<uint64_t>(s) * kTagRing + lane] = kNoStep;
    if (lane == 0 && !t.svt) t.vt[s] = make_uint2(ver, kNoStep);
  }
}

void launch_ckpt_gather(const DevTable& t, const uint32_t* slots, uint64_t n, float* rows2d,
                        uint64_t* vers, cudaStream_t st) {
  if (!n) return;
  launch(ckpt_gather_kernel, std::min<uint64_t>(ceil_div(n, 8), 148 * 32), 256, 0, st, t, slots,
         n, rows2d, vers);
  HPS_LAUNCH_CHECK();
}

void launch_ckpt_restore(const DevTable& t, const uint64_t* ids, const float* rows2d,
                         const uint64_t* vers, uint64_t n, uint32_t* new_slots,
                         uint32_t* new_count, cudaStream_t st, const uint32_t* at,
                         const unsigned long long* stamps) {
  if (!n) return;
  launch(ckpt_restore_kernel, std::min<uint64_t>(ceil_div(n, 8), 148 * 32), 256, 0, st, t, ids,
         rows2d, vers, n, new_slots, new_count, at, stamps);
  HPS_LAUNCH_CHECK();
}

// ---- validation before mutation (embedding_ps.hpp:146-153) --------------------------------

__global__ void check_direct_kernel(const float* __restrict__ g, uint64_t n, uint32_t* flag) {
  pdl_entry();
  bool bad = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1u);
}

void launch_check_direct(const float* grads, uint64_t n, uint32_t* flag, cudaStream_t st) {
  if (!n) return;
  launch(check_direct_kernel, std::min<uint64_t>(ceil_div(n, 256), 148 * 8), 256, 0, st, grads, n,
         flag);
  HPS_LAUNCH_CHECK();
}

// ---- small helpers --------------------------------------------------------------------

__global__ void iota_kernel(uint32_t* out, uint64_t n) {
  pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<uint32_t>(i);
}

void launch_iota(uint32_t* out, uint64_t n, cudaStream_t st) {
  if (!n) return;
  launch(iota_kernel, std::min<uint64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st, out, n);
  HPS_LAUNCH_CHECK();
}

__global__ void sample_order_kernel(const uint64_t* __restrict__ sk, uint32_t B,
                                    uint64_t* __restrict__ keys, uint32_t* __restrict__ perm) {
  pdl_entry();
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    keys[b] = sk[b];
    perm[b] = b;
  }
}

void launch_sample_order(const uint64_t* sk, uint32_t B, uint64_t* keys, uint32_t* perm,
                         cudaStream_t st) {
  if (!B) return;
  launch(sample_order_kernel, ceil_div(B, 256), 256, 0, st, sk, B, keys, perm);
  HPS_LAUNCH_CHECK();
}

__global__ void sample_lengths_kernel(const uint32_t* __restrict__ perm,
                                      const uint32_t* __restrict__ off, uint32_t B, uint32_t F,
                                      uint32_t* __restrict__ lens) {
  pdl_entry();
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < B; r += gridDim.x * blockDim.x) {
    uint64_t b = perm[r];
    lens[r] = off[(b + 1) * F] - off[b * F];
  }
}

void launch_sample_lengths(const uint32_t* perm, const uint32_t* off, uint32_t B, uint32_t F,
                           uint32_t* lens, cudaStream_t st) {
  if (!B) return;
  launch(sample_lengths_kernel, ceil_div(B, 256), 256, 0, st, perm, off, B, F, lens);
  HPS_LAUNCH_CHECK();
}

void launch_scan_inplace(uint32_t* data, uint32_t n, uint32_t* total, cudaStream_t st) {
  launch(radix::scan_digits, 1, 1024, 0, st, data, n, total);
  HPS_LAUNCH_CHECK();
}

__global__ void permuted_listing_kernel(const uint32_t* __restrict__ perm,
                                        const uint32_t* __restrict__ starts,
                                        const uint32_t* __restrict__ off,
                                        const uint32_t* __restrict__ slots, uint32_t B,
                                        uint32_t F, uint32_t* __restrict__ keys,
                                        uint32_t* __restrict__ vals) {
  pdl_entry();
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
  launch(permuted_listing_kernel, std::min<uint64_t>(ceil_div(B, 8), 148 * 16), 256, 0, st, 
      perm, starts, off, slots, B, F, keys, vals);
  HPS_LAUNCH_CHECK();
}

__global__ void add_counter_kernel(unsigned long long* ctr, int idx, const uint32_t* src) {
  pdl_entry();
  atomicAdd(&ctr[idx], (unsigned long long)*src);
}

void launch_add_counter_from(unsigned long long* ctr, int idx, const uint32_t* src,
                             cudaStream_t st) {
  launch(add_counter_kernel, 1, 1, 0, st, ctr, idx, src);
  HPS_LAUNCH_CHECK();
}

__global__ void add_counter_const_kernel(unsigned long long* ctr, int idx, unsigned long long v) {
  pdl_entry();
  atomicAdd(&ctr[idx], v);
}

void launch_add_counter_const(unsigned long long* ctr, int idx, unsigned long long v,
                              cudaStream_t st) {
  launch(add_counter_const_kernel, 1, 1, 0, st, ctr, idx, v);
  HPS_LAUNCH_CHECK();
}

}  // namespace hps
