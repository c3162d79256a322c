// Exact LRU capacity / eviction (HPS_TABLE_LRU).
//
// The reference keeps each shard's rows in an LruStore (lru_store.hpp:62-113): a touch
// (find) moves the row to the front; a miss (PsShard::find_or_init embedding_ps.hpp:
// 417-434) takes a recycled slot, else the next slot below capacity, else evicts the
// least-recently-used row and re-initialises its slot for the new id. The device keeps the
// same order as a per-slot stamp = the time of the row's last touch (Table::clock counts
// accesses, array order within a call), so a shard's LRU row is its live row with the
// smallest stamp.
//
// A PS-surface call (lookup / apply, entries in array order) first counts, per shard, the
// listings that miss. If every shard has room for all of them, no eviction can happen and
// the parallel kernels run (their inserts take slots from the shard's own range); the
// call's touches then set stamp[slot] = max over the row's listings of (clock + index).
// Otherwise the whole call runs in order on one warp -- the reference's loop, on the
// device: per entry find, or insert into a free slot, or evict the shard's LRU row (the
// next untouched row of the shard's stamp-sorted candidate list; rows touched earlier in
// this call are the newest), then the lookup's copy or apply_gradients' count_delay /
// bump_version / apply_one. Evicted rows leave the open-addressing index by backward-shift
// deletion (no tombstones), so probe chains stay as short as without eviction.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "radix_sort.cuh"
#include "table.cuh"
#include "table_impl.h"
#include "vec.cuh"

namespace hps {

namespace {

__device__ __forceinline__ uint64_t home_of(const DevTable& t, uint64_t id) {
  return mix64(id ^ kTableHashSalt) >> t.ht_shift;
}

// Index lookup without insertion (single writer: the sequential path owns the table).
__device__ uint32_t seq_find(const DevTable& t, uint64_t id) {
  if (id == kEmptyKey) {
    const uint32_t s = *t.special;
    return s == kSpecialAbsent ? kInvalidSlot : s;
  }
  for (uint64_t h = home_of(t, id), k = 0; k <= t.ht_mask; ++k, h = (h + 1) & t.ht_mask) {
    const HashEntry e = t.ht[h];
    if (e.key == kEmptyKey) return kInvalidSlot;
    if (e.key == id) return e.slot;
  }
  return kInvalidSlot;
}

__device__ void seq_insert(const DevTable& t, uint64_t id, uint32_t slot) {
  if (id == kEmptyKey) {
    *t.special = slot;
    return;
  }
  for (uint64_t h = home_of(t, id), k = 0; k <= t.ht_mask; ++k, h = (h + 1) & t.ht_mask) {
    if (t.ht[h].key == kEmptyKey) {
      t.ht[h].key = id;
      t.ht[h].slot = slot;
      return;
    }
  }
  atomicExch(&t.ctr[kCtrOverflow], 1ull);
}

// Linear-probing deletion by backward shift: later entries of the cluster that may live
// at the freed position move back, so no tombstone is left behind.
__device__ void seq_erase(const DevTable& t, uint64_t id) {
  if (id == kEmptyKey) {
    *t.special = kSpecialAbsent;
    return;
  }
  uint64_t i = home_of(t, id);
  for (uint64_t k = 0; k <= t.ht_mask && t.ht[i].key != id; ++k) {
    if (t.ht[i].key == kEmptyKey) return;
    i = (i + 1) & t.ht_mask;
  }
  if (t.ht[i].key != id) return;
  for (uint64_t j = (i + 1) & t.ht_mask;; j = (j + 1) & t.ht_mask) {
    const HashEntry e = t.ht[j];
    if (e.key == kEmptyKey) break;
    const uint64_t h = home_of(t, e.key);
    // e may move to i iff i lies cyclically in [h, j)
    const bool movable = (j > i) ? (h <= i || h > j) : (h <= i && h > j);
    if (movable) {
      t.ht[i].key = e.key;
      t.ht[i].slot = e.slot;
      i = j;
    }
  }
  t.ht[i].key = kEmptyKey;
  t.ht[i].slot = kPending;
}

}  // namespace

// Per shard, the listings of a call whose id is absent (an upper bound on its inserts).
__global__ void lru_misses_kernel(DevTable t, const uint64_t* __restrict__ ids, uint64_t n,
                                  uint32_t* __restrict__ per_shard) {
  pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = ids[i];
    if (seq_find(t, id) == kInvalidSlot) atomicAdd(&per_shard[route_shard(id, t.S)], 1u);
  }
}

__global__ void lru_stamp_kernel(DevTable t, const uint32_t* __restrict__ slots, uint64_t n,
                                 unsigned long long t0) {
  pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = slots[i];
    if (slot_ok(t, s)) atomicMax(&t.stamp[s], t0 + i);
  }
}

// Sort keys of the live rows: (shard << 56 | stamp), others last.
__global__ void lru_keys_kernel(DevTable t, unsigned long long* __restrict__ keys,
                                uint32_t* __restrict__ vals) {
  pdl_entry();
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < t.capacity;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t sh = static_cast<uint32_t>(s / t.shard_cap);
    const bool live = s - static_cast<uint64_t>(sh) * t.shard_cap < t.shard_hwm[sh];
    keys[s] = live ? (static_cast<unsigned long long>(sh) << 56) | t.stamp[s] : ~0ull;
    vals[s] = static_cast<uint32_t>(s);
  }
}

struct LruSeqArgs {
  const uint64_t* ids;
  uint64_t n;
  int mode;  // 0 lookup, 1 apply (tracked: rv), 2 apply untracked (apply_gradients_map)
  const float* grads;
  const uint64_t* rv;
  float lr;
  uint32_t step_tag;
  int exact;
  float* out_values;
  uint64_t* out_versions;
  uint32_t* out_delays;
  unsigned long long t0;
  const uint32_t* cand;      // live slots sorted by (shard, stamp)
  uint32_t* cand_pos;        // [S] next candidate per shard
  const uint32_t* cand_end;  // [S]
};

// The reference's per-entry loop on one warp (lane 0: index / LRU / clocks; lanes: the
// row's dimensions). count_delay / bump_version follow update.cu's version_step rules.
__global__ void __launch_bounds__(32) lru_seq_kernel(DevTable t, LruSeqArgs a) {
  pdl_entry();
  const uint32_t lane = threadIdx.x;
  const uint32_t D = t.D;
  const bool adagrad = t.opt == HPS_ADAGRAD;
  const double limit = 1.0 / sqrt(static_cast<double>(D));
  const double lo = -limit, span = __dsub_rn(limit, lo);
  unsigned long long misses = 0, evictions = 0, resets = 0;
  uint32_t hist0 = 0, max_delay = 0;
  __shared__ uint32_t s_hist[17];
  if (lane < 17) s_hist[lane] = 0;
  __syncwarp();
  for (uint64_t i = 0; i < a.n; ++i) {
    const uint64_t id = a.ids[i];
    uint32_t slot = 0, fresh = 0;
    if (lane == 0) {
      slot = seq_find(t, id);
      if (slot == kInvalidSlot) {
        fresh = 1;
        const uint32_t sh = route_shard(id, t.S);
        const uint32_t base = sh * t.shard_cap;
        if (t.shard_hwm[sh] < t.shard_cap) {
          slot = base + t.shard_hwm[sh]++;
        } else {
          // LruStore::put: evict the tail -- the shard's oldest row not touched by
          // this call (touched rows are newer than every untouched one)
          slot = kInvalidSlot;
          while (a.cand_pos[sh] < a.cand_end[sh]) {
            const uint32_t v = a.cand[a.cand_pos[sh]++];
            if (t.stamp[v] < a.t0) {
              slot = v;
              break;
            }
          }
          if (slot == kInvalidSlot) {  // every row was touched by this call: oldest touch
            unsigned long long best = ~0ull;
            for (uint32_t k = 0; k < t.shard_cap; ++k)
              if (t.stamp[base + k] < best) best = t.stamp[base + k], slot = base + k;
          }
          seq_erase(t, t.slot_id[slot]);
          ++evictions;
          ++t.shard_evict[sh];
        }
        seq_insert(t, id, slot);
        t.slot_id[slot] = id;
        ++misses;
      }
      t.stamp[slot] = a.t0 + i;
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    fresh = __shfl_sync(0xffffffffu, fresh, 0);
    float* row = t.rows + static_cast<uint64_t>(slot) * t.stride;
    if (fresh) {  // find_or_init's initialisation (embedding_ps.hpp:424-432)
      const uint64_t seed = mix64(id ^ mix64(t.salts[route_shard(id, t.S)]));
      for (uint32_t d = lane; d < D; d += 32) {
        row[d] = init_value(seed, d, lo, span);
        row[D + d] = (t.svt && d < 64 && (d & 3) >= 2) ? -0.0f : 0.0f;
      }
      if (t.ring && lane < kTagRing) t.ring[static_cast<uint64_t>(slot) * kTagRing + lane] = kNoStep;
      if (lane == 0 && !t.svt) t.vt[slot] = make_uint2(0u, kNoStep);
    }
    __syncwarp();
    uint2 vt = make_uint2(0, 0);
    if (lane == 0) vt = vt_read(t, slot);
    vt.x = __shfl_sync(0xffffffffu, vt.x, 0);
    vt.y = __shfl_sync(0xffffffffu, vt.y, 0);
    if (a.mode == 0) {  // PsShard::lookup: copy the row and its version
      for (uint32_t d = lane; d < D; d += 32) a.out_values[i * D + d] = row[d];
      if (lane == 0 && a.out_versions) a.out_versions[i] = vt.x;
      continue;
    }
    // apply_gradients: count_delay, bump_version, apply_one
    uint32_t ver = vt.x, tag = vt.y;
    if (lane == 0) {
      uint32_t* ring = t.ring ? t.ring + static_cast<uint64_t>(slot) * kTagRing : nullptr;
      if (a.mode == 2) {
        ++ver;
        if (ring) tag = ring[(ver - 1) % kTagRing];
      } else {
        const uint64_t rv = a.rv[i];
        uint32_t delay = 0;
        if (rv > ver) {
          ++resets;
        } else if (!a.exact || !ring) {
          const uint64_t gap = ver - rv;
          delay = static_cast<uint32_t>(gap < kTagRing ? gap : kTagRing);
          if (gap > 0 && tag != kNoStep && tag >= a.step_tag) delay -= 1;
        } else {
          uint64_t lo_v = rv + 1;
          if (ver >= kTagRing && lo_v < ver - kTagRing + 1) lo_v = ver - kTagRing + 1;
          uint32_t distinct[kTagRing], nd = 0;
          for (uint64_t k = lo_v; k <= ver; ++k) {
            const uint32_t tg = ring[(k - 1) % kTagRing];
            if (tg == kNoStep || tg >= a.step_tag) continue;
            bool dup = false;
            for (uint32_t j = 0; j < nd; ++j) dup |= distinct[j] == tg;
            if (!dup) distinct[nd++] = tg;
          }
          delay = nd;
        }
        if (!(ver > 0 && tag == a.step_tag)) {
          if (ring) ring[ver % kTagRing] = a.step_tag;
          ++ver;
          tag = a.step_tag;
        }
        s_hist[delay < 16 ? delay : 16]++;
        max_delay = max(max_delay, delay);
        if (a.out_delays) a.out_delays[i] = delay;
      }
    }
    ver = __shfl_sync(0xffffffffu, ver, 0);
    tag = __shfl_sync(0xffffffffu, tag, 0);
    const float* g = a.grads + i * D;
    for (uint32_t d = lane; d < D; d += 32) {
      float w = row[d];
      float acc = row[D + d];
      if (t.svt) acc = fabsf(acc);
      const float c = g[d];
      if (adagrad) {
        acc = __fadd_rn(acc, __fmul_rn(c, c));
        w = __fsub_rn(w, __fdiv_rn(__fmul_rn(a.lr, c), __fadd_rn(__fsqrt_rn(acc), kAdagradEps)));
      } else {
        w = __fsub_rn(w, __fmul_rn(a.lr, c));
      }
      if (t.svt && d < 64) {
        const uint32_t l = d >> 2, k = d & 3;
        const uint32_t word = k == 0 ? ver & 0xffffu : k == 1 ? ver >> 16
                            : k == 2 ? tag & 0xffffu : tag >> 16;
        acc = with_sign(acc, (word >> l) & 1u);
      }
      row[d] = w;
      if (adagrad) row[D + d] = acc;
    }
    if (lane == 0 && !t.svt) t.vt[slot] = make_uint2(ver, tag);
    __syncwarp();
  }
  __syncwarp();
  if (lane == 0) {
    if (misses) atomicAdd(&t.ctr[kCtrMisses], misses);
    if (evictions) atomicAdd(&t.ctr[kCtrEvictions], evictions);
    if (resets) atomicAdd(&t.ctr[kCtrClockResets], resets);
    if (max_delay) atomicMax(&t.ctr[kCtrMaxDelay], (unsigned long long)max_delay);
  }
  if (a.mode == 1 && lane < 17 && s_hist[lane])
    atomicAdd(&t.ctr[kCtrDelayHist + lane], (unsigned long long)s_hist[lane]);
  (void)hist0;
}

// ---- host ------------------------------------------------------------------------------

// Returns true when the call must take the sequential (evicting) path.
bool lru_needs_eviction(Table* t, const uint64_t* d_ids, uint64_t n, cudaStream_t st) {
  DevTable& d = t->d;
  const uint32_t S = d.S;
  if (!t->lru_scratch) HPS_CUDA(cudaMalloc(&t->lru_scratch, 3 * S * sizeof(uint32_t) + 64));
  HPS_CUDA(cudaMemsetAsync(t->lru_scratch, 0, S * sizeof(uint32_t), st));
  if (n) {
    launch(lru_misses_kernel, std::min<uint64_t>(ceil_div(n, 256), t->sm_count * 4ull), 256, 0,
           st, d, d_ids, n, t->lru_scratch);
    HPS_LAUNCH_CHECK();
  }
  std::vector<uint32_t> h(2 * S);
  HPS_CUDA(cudaMemcpyAsync(h.data(), t->lru_scratch, S * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           st));
  HPS_CUDA(cudaMemcpyAsync(h.data() + S, d.shard_hwm, S * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
  for (uint32_t s = 0; s < S; ++s)
    if (static_cast<uint64_t>(h[S + s]) + h[s] > d.shard_cap) return true;
  return false;
}

void lru_stamp(Table* t, const uint32_t* slots, uint64_t n, cudaStream_t st) {
  if (!n) return;
  launch(lru_stamp_kernel, std::min<uint64_t>(ceil_div(n, 256), t->sm_count * 8ull), 256, 0, st,
         t->d, slots, n, static_cast<unsigned long long>(t->clock));
  HPS_LAUNCH_CHECK();
  t->clock += n;
}

// The sequential path of one call (mode: 0 lookup, 1 tracked apply, 2 untracked apply).
void lru_sequential(Table* t, int mode, const uint64_t* ids, uint64_t n, const float* grads,
                    const uint64_t* rv, float lr, uint32_t step_tag, int exact, float* out_values,
                    uint64_t* out_versions, uint32_t* out_delays, cudaStream_t st) {
  DevTable& d = t->d;
  const uint32_t S = d.S;
  const uint64_t C = d.capacity;
  // candidate lists: live slots sorted by (shard, stamp)
  Batch& b = t->scratch;
  batch_reserve(b, C, 0, 0);
  if (C > t->lru_cap) {
    if (t->lru_keys) cudaFree(t->lru_keys);
    if (t->lru_keys2) cudaFree(t->lru_keys2);
    HPS_CUDA(cudaMalloc(&t->lru_keys, C * sizeof(unsigned long long)));
    HPS_CUDA(cudaMalloc(&t->lru_keys2, C * sizeof(unsigned long long)));
    t->lru_cap = C;
  }
  launch(lru_keys_kernel, std::min<uint64_t>(ceil_div(C, 256), t->sm_count * 8ull), 256, 0, st,
         d, reinterpret_cast<unsigned long long*>(t->lru_keys), b.vals_a);
  HPS_LAUNCH_CHECK();
  const bool in_b = radix::sort_pairs<uint64_t>(
      reinterpret_cast<uint64_t*>(t->lru_keys), b.vals_a,
      reinterpret_cast<uint64_t*>(t->lru_keys2), b.vals_b, C, 64, b.hist, st, t->sm_count);
  const uint32_t* cand = in_b ? b.vals_b : b.vals_a;
  // per-shard candidate ranges from the shards' row counts
  std::vector<uint32_t> hwm(S), pos(2 * S);
  HPS_CUDA(cudaMemcpyAsync(hwm.data(), d.shard_hwm, S * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           st));
  HPS_CUDA(cudaStreamSynchronize(st));
  uint32_t run = 0;
  for (uint32_t s = 0; s < S; ++s) {
    pos[s] = run;
    run += hwm[s];
    pos[S + s] = run;
  }
  HPS_CUDA(cudaMemcpyAsync(t->lru_scratch, pos.data(), 2 * S * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, st));
  LruSeqArgs a{};
  a.ids = ids;
  a.n = n;
  a.mode = mode;
  a.grads = grads;
  a.rv = rv;
  a.lr = lr;
  a.step_tag = step_tag;
  a.exact = exact;
  a.out_values = out_values;
  a.out_versions = out_versions;
  a.out_delays = out_delays;
  a.t0 = t->clock;
  a.cand = cand;
  a.cand_pos = t->lru_scratch;
  a.cand_end = t->lru_scratch + S;
  launch(lru_seq_kernel, 1, 32, 0, st, d, a);
  HPS_LAUNCH_CHECK();
  t->clock += n;
}

}  // namespace hps
