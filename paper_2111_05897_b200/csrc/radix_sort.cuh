// Stable LSD radix sort of (key, u32 value) pairs, hand-written for sm_100a.
//
// Two shapes:
//  * small (n <= kSmallN): one CTA sorts in shared memory, every pass in one launch --
//    the common case of a one-hot batch's multi-listing list;
//  * large ("onesweep"): one histogram kernel for all digit passes, then ONE kernel
//    per 8-bit pass whose tiles find their global offsets by decoupled look-back.
//    Per pass every key/value is read and written once (2*(sizeof(K)+4) B/element).
// The large path can be gated on a device-side count (run only if *gate > kSmallN)
// so the host never waits for the device to choose between the two.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"

namespace hps {
namespace radix {

constexpr int kBits = 8;
constexpr int kBins = 1 << kBits;
constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kMaxPasses = 8;

constexpr int kSmallBlock = 1024;
constexpr int kSmallItems = 4;
constexpr uint32_t kSmallN = kSmallBlock * kSmallItems;

template <typename K>
struct Tile {
  static constexpr int kItems = 8;
  static constexpr int kTile = kBlock * kItems;
  static constexpr size_t kSmem =
      kTile * (sizeof(K) + sizeof(uint32_t)) + (kWarps * kBins + 3 * kBins) * sizeof(uint32_t);
};

// status word: [63:32] epoch of the pass, [31] inclusive-prefix flag, [30:0] count
constexpr unsigned long long kPrefixFlag = 1ull << 31;

inline std::atomic<uint32_t> g_epoch{1};

// Decoupled look-back by one full warp (all 32 lanes call it): returns the exclusive
// prefix of `tile` over status[0..tile) (one word per tile, published with `epoch`),
// reading 32 predecessors per round trip instead of one.
__device__ __forceinline__ uint32_t warp_lookback(const unsigned long long* status, uint32_t tile,
                                                  uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  uint32_t excl = 0;
  int64_t end = tile;
  while (end > 0) {
    const int64_t idx = end - 32 + lane;  // lane 31 = nearest predecessor
    unsigned long long v = kPrefixFlag;   // below tile 0: an empty prefix
    if (idx >= 0) {
      const volatile unsigned long long* s = status + idx;
      do {
        v = *s;
      } while ((v >> 32) != epoch);
    }
    const uint32_t pmask = __ballot_sync(0xffffffffu, (v & kPrefixFlag) != 0);
    const int hi = pmask ? 31 - __clz(pmask) : 0;
    const uint32_t val = lane >= hi ? static_cast<uint32_t>(v & (kPrefixFlag - 1)) : 0u;
    excl += __reduce_add_sync(0xffffffffu, val);
    if (pmask) break;
    end -= 32;
  }
  return excl;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return static_cast<uint32_t>(key >> shift) & (kBins - 1);
}

__device__ __forceinline__ bool gate_open(const uint32_t* gate) {
  return gate == nullptr || *gate > kSmallN;
}

// Block-wide exclusive scan over kBins values held by threads 0..kBins-1 (every thread
// of the block calls it; threads >= kBins pass 0 and get garbage).
__device__ __forceinline__ uint32_t block_excl_scan_bins(uint32_t v, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31 && warp < kBins / 32) scratch[warp] = x;
  __syncthreads();
  uint32_t off = 0;
  for (int w = 0; w < warp && w < kBins / 32; ++w) off += scratch[w];
  __syncthreads();
  return off + x - v;
}

// ---- small path: all passes in one CTA --------------------------------------------------

// LSD passes over sk/sv (double-buffered in shared memory, n <= kSmallN); returns the
// buffer index holding the result.
template <typename K>
__device__ int smem_lsd(K* sk, uint32_t* sv, uint32_t* wc, uint32_t* dstart, uint32_t* scr,
                        uint32_t n, int first_shift, int passes) {
  constexpr int kW = kSmallBlock / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    const int shift = first_shift + p * kBits;
    for (int i = threadIdx.x; i < kW * kBins; i += kSmallBlock) wc[i] = 0;
    __syncthreads();
    K k[kSmallItems];
    uint32_t v[kSmallItems], r[kSmallItems];
#pragma unroll
    for (int j = 0; j < kSmallItems; ++j) {
      const uint32_t idx = warp * 32 * kSmallItems + j * 32 + lane;
      const bool ok = idx < n;
      k[j] = ok ? sk[cur * kSmallN + idx] : K(0);
      v[j] = ok ? sv[cur * kSmallN + idx] : 0u;
      const uint32_t d = ok ? digit_of(k[j], shift) : static_cast<uint32_t>(kBins);
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t before = wc[warp * kBins + (d & (kBins - 1))];
      r[j] = before + __popc(peers & lt_mask);
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) wc[warp * kBins + d] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    uint32_t tot = 0;
    if (threadIdx.x < kBins) {
      for (int w = 0; w < kW; ++w) {
        const uint32_t c = wc[w * kBins + threadIdx.x];
        wc[w * kBins + threadIdx.x] = tot;
        tot += c;
      }
    }
    const uint32_t start = block_excl_scan_bins(threadIdx.x < kBins ? tot : 0u, scr);
    if (threadIdx.x < kBins) dstart[threadIdx.x] = start;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSmallItems; ++j) {
      const uint32_t idx = warp * 32 * kSmallItems + j * 32 + lane;
      if (idx < n) {
        const uint32_t d = digit_of(k[j], shift);
        const uint32_t pos = dstart[d] + wc[warp * kBins + d] + r[j];
        sk[(cur ^ 1) * kSmallN + pos] = k[j];
        sv[(cur ^ 1) * kSmallN + pos] = v[j];
      }
    }
    cur ^= 1;
    __syncthreads();
  }
  return cur;
}

template <typename K>
constexpr size_t small_smem() {
  return 2 * kSmallN * (sizeof(K) + sizeof(uint32_t)) + (kSmallBlock / 32 + 2) * kBins * 4;
}

// Host-sized small sort; vals_in == nullptr means values 0..n-1.
template <typename K>
__global__ void __launch_bounds__(kSmallBlock)
    small_sort_kernel(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                      K* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n,
                      int passes) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + 2 * kSmallN);
  uint32_t* wc = sv + 2 * kSmallN;
  uint32_t* dstart = wc + (kSmallBlock / 32) * kBins;
  uint32_t* scr = dstart + kBins;
  for (uint32_t i = threadIdx.x; i < n; i += kSmallBlock) {
    sk[i] = keys_in[i];
    sv[i] = vals_in ? vals_in[i] : i;
  }
  __syncthreads();
  const int cur = smem_lsd<K>(sk, sv, wc, dstart, scr, n, 0, passes);
  for (uint32_t i = threadIdx.x; i < n; i += kSmallBlock) {
    keys_out[i] = sk[cur * kSmallN + i];
    vals_out[i] = sv[cur * kSmallN + i];
  }
}

// Device-sized small sort of composite keys (slot << lbits | listing): runs only when
// *n_dev <= kSmallN and writes the sorted slots and listings separately. The keys are
// unique (the listing is part of them), so each key's final position is its rank --
// the number of smaller keys. One warp ranks one key by scanning the (L1-resident)
// list: O(n^2) comparisons, but spread over the whole GPU with no barrier at all,
// where a one-CTA sort is bound by a single SM's issue rate.
constexpr int kRankBlock = 256;

static __global__ void __launch_bounds__(kRankBlock)
    small_composite_kernel(const unsigned long long* __restrict__ keys, const uint32_t* n_dev,
                           int lbits, uint32_t* __restrict__ out_slot,
                           uint32_t* __restrict__ out_listing) {
  pdl_entry();
  const uint32_t n = *n_dev;
  if (n > kSmallN) return;  // the large path (gated on the same count) takes it
  const int lane = threadIdx.x & 31;
  const uint32_t e = (blockIdx.x * kRankBlock + threadIdx.x) >> 5;
  if (e >= n) return;
  const unsigned long long me = keys[e];
  uint32_t less = 0;
  for (uint32_t i = lane; i < n; i += 32) less += __ldg(keys + i) < me;
  less = __reduce_add_sync(0xffffffffu, less);
  if (lane == 0) {
    out_slot[less] = static_cast<uint32_t>(me >> lbits);
    out_listing[less] = static_cast<uint32_t>(me & ((1ull << lbits) - 1));
  }
}

// ---- large path ("onesweep") -------------------------------------------------------------

// Digit histograms of every pass in one read of the keys: hist[p * kBins + d].
template <typename K>
__global__ void __launch_bounds__(kBlock)
    hist_kernel(const K* __restrict__ keys, uint32_t n, int passes, uint32_t* __restrict__ hist,
                const uint32_t* gate) {
  pdl_entry();
  if (!gate_open(gate)) return;
  __shared__ uint32_t cnt[kMaxPasses * kBins];
  for (int i = threadIdx.x; i < passes * kBins; i += kBlock) cnt[i] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
    K k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&cnt[p * kBins + digit_of(k, p * kBits)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kBins; i += kBlock)
    if (cnt[i]) atomicAdd(&hist[i], cnt[i]);
}

// Optional output of the final pass (hps batch plan): meta.out[g] = lgrp[v] | (size of
// group lgrp[v]) << 32 for the value v sorted to position g -- what the ordered update
// reads per position, computed where the random lookups overlap the scatter.
struct SortMeta {
  const uint32_t* lgrp = nullptr;
  const uint32_t* offsets = nullptr;
  uint64_t* out = nullptr;
};

// vals_in == nullptr: values are the input positions (pass 0 of an index sort).
template <typename K>
__global__ void __launch_bounds__(kBlock)
    pass_kernel(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                K* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
                const uint32_t* __restrict__ hist, unsigned long long* status, uint32_t* tile_ctr,
                uint32_t epoch, const uint32_t* gate, const SortMeta meta) {
  pdl_entry();
  constexpr int kItems = Tile<K>::kItems;
  constexpr int kTileN = Tile<K>::kTile;
  if (!gate_open(gate)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  K* skeys = reinterpret_cast<K*>(smem);
  uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + kTileN);
  uint32_t* wcnt = svals + kTileN;              // [kWarps][kBins]
  uint32_t* block_off = wcnt + kWarps * kBins;  // [kBins]
  uint32_t* gbase = block_off + kBins;          // [kBins]
  uint32_t* scratch = gbase + kBins;            // [kBins] (uses 32 + 1)

  const uint32_t tiles = (n + kTileN - 1) / kTileN;
  // Dynamic tile order: a tile only ever waits on tiles that were scheduled before it.
  if (threadIdx.x == 0) scratch[32] = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < kWarps * kBins; i += kBlock) wcnt[i] = 0;
  __syncthreads();
  const uint32_t tile = scratch[32];
  if (tile >= tiles) return;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile_base = static_cast<uint64_t>(tile) * kTileN;
  const uint64_t warp_base = tile_base + static_cast<uint64_t>(warp) * 32 * kItems;
  K k[kItems];
  uint32_t v[kItems];
  uint32_t r[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    uint64_t idx = warp_base + static_cast<uint64_t>(j) * 32 + lane;
    bool ok = idx < n;
    k[j] = ok ? keys_in[idx] : K(0);
    v[j] = ok ? (vals_in ? vals_in[idx] : static_cast<uint32_t>(idx)) : 0u;
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    uint64_t idx = warp_base + static_cast<uint64_t>(j) * 32 + lane;
    bool ok = idx < n;
    uint32_t d = ok ? digit_of(k[j], shift) : static_cast<uint32_t>(kBins);
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = wcnt[warp * kBins + (d & (kBins - 1))];
    r[j] = before + __popc(peers & lt_mask);
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) wcnt[warp * kBins + d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const uint32_t d = threadIdx.x;  // kBlock == kBins: thread d owns digit d below
  uint32_t tile_cnt = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    uint32_t c = wcnt[w * kBins + d];
    wcnt[w * kBins + d] = tile_cnt;
    tile_cnt += c;
  }
  // Publish this tile's aggregate, then look back for the exclusive prefix.
  unsigned long long* my = status + static_cast<uint64_t>(tile) * kBins + d;
  const unsigned long long ep = static_cast<unsigned long long>(epoch) << 32;
  *reinterpret_cast<volatile unsigned long long*>(my) =
      ep | (tile == 0 ? kPrefixFlag : 0ull) | tile_cnt;
  uint32_t excl = 0;
  if (tile > 0) {
    for (int64_t t = static_cast<int64_t>(tile) - 1; t >= 0; --t) {
      const volatile unsigned long long* s = status + static_cast<uint64_t>(t) * kBins + d;
      unsigned long long x;
      do {
        x = *s;
      } while ((x >> 32) != epoch);
      excl += static_cast<uint32_t>(x & (kPrefixFlag - 1));
      if (x & kPrefixFlag) break;
    }
    *reinterpret_cast<volatile unsigned long long*>(my) = ep | kPrefixFlag | (excl + tile_cnt);
  }
  // Global digit start (exclusive scan of the pass histogram) + this tile's prefix.
  const uint32_t start = block_excl_scan_bins(hist[d], scratch);
  gbase[d] = start + excl;
  block_off[d] = block_excl_scan_bins(tile_cnt, scratch);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    uint64_t idx = warp_base + static_cast<uint64_t>(j) * 32 + lane;
    if (idx < n) {
      uint32_t dd = digit_of(k[j], shift);
      uint32_t pos = block_off[dd] + wcnt[warp * kBins + dd] + r[j];
      skeys[pos] = k[j];
      svals[pos] = v[j];
    }
  }
  __syncthreads();
  const uint32_t tile_n =
      static_cast<uint32_t>(n - tile_base < (uint64_t)kTileN ? n - tile_base : (uint64_t)kTileN);
  for (uint32_t p = threadIdx.x; p < tile_n; p += kBlock) {
    K key = skeys[p];
    uint32_t dd = digit_of(key, shift);
    uint32_t g = gbase[dd] + (p - block_off[dd]);
    keys_out[g] = key;
    vals_out[g] = svals[p];
    if (meta.out) {  // final pass: per sorted position, the listing's group and its size
      const uint32_t lg = meta.lgrp[svals[p]];
      meta.out[g] = lg | (static_cast<uint64_t>(meta.offsets[lg + 1] - meta.offsets[lg]) << 32);
    }
  }
}

// Scratch words (u32 units) to sort up to n pairs on the large path.
template <typename K>
inline size_t scratch_words(uint64_t n) {
  uint64_t tiles = (n + Tile<K>::kTile - 1) / Tile<K>::kTile;
  if (tiles == 0) tiles = 1;
  return kMaxPasses * kBins + kMaxPasses * 2 + tiles * kBins * 2 + 2;
}

template <typename K>
inline void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  HPS_CUDA(cudaFuncSetAttribute(pass_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(Tile<K>::kSmem)));
  HPS_CUDA(cudaFuncSetAttribute(small_sort_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(small_smem<K>())));
  done = true;
}

// Sorts n (host count) pairs by key bits [0, key_bits). vals_a == nullptr sorts the
// positions 0..n-1. gate != nullptr: the whole sort runs only if *gate > kSmallN
// (device-side choice between this and the small composite path). Returns true when
// the result lives in the (b) buffers. scratch needs scratch_words<K>(n) words.
// keys_in0 != nullptr: the first pass reads its keys from there (left untouched) and
// keys_a is only scratch. iota_vals: the values are the positions 0..n-1 (vals_a is
// then only scratch too).
template <typename K>
inline bool sort_pairs(K* keys_a, uint32_t* vals_a, K* keys_b, uint32_t* vals_b, uint64_t n,
                       int key_bits, uint32_t* scratch, cudaStream_t stream, int sms = 148,
                       const uint32_t* gate = nullptr, const K* keys_in0 = nullptr,
                       bool iota_vals = false, bool zero_scratch = true,
                       SortMeta meta = SortMeta{}) {
  if (n == 0) return false;
  if (key_bits <= 0) key_bits = 1;
  set_smem_attrs<K>();
  const int passes = (key_bits + kBits - 1) / kBits;
  const K* first = keys_in0 ? keys_in0 : keys_a;
  const uint32_t* first_vals = iota_vals ? nullptr : vals_a;
  if (!gate && n <= kSmallN) {
    if (n == 0) return false;
    launch(small_sort_kernel<K>, 1, kSmallBlock, small_smem<K>(), stream, 
        first, first_vals, keys_b, vals_b, static_cast<uint32_t>(n), passes);
    HPS_LAUNCH_CHECK();
    return true;
  }
  const uint32_t tiles = ceil_div(n, Tile<K>::kTile);
  uint32_t* hist = scratch;                       // [kMaxPasses][kBins]
  uint32_t* tile_ctr = hist + kMaxPasses * kBins;  // [kMaxPasses * 2]
  uint64_t off = (kMaxPasses * kBins + kMaxPasses * 2 + 1) & ~1ull;
  unsigned long long* status = reinterpret_cast<unsigned long long*>(scratch + off);
  if (zero_scratch)  // (else the caller zeroed it: see sort_scratch_zero)
    HPS_CUDA(cudaMemsetAsync(scratch, 0,
                             (kMaxPasses * kBins + kMaxPasses * 2) * sizeof(uint32_t), stream));
  const uint32_t n32 = static_cast<uint32_t>(n);
  const uint32_t hblocks = std::min<uint32_t>(tiles, static_cast<uint32_t>(sms) * 4);
  launch(hist_kernel<K>, hblocks, kBlock, 0, stream, first, n32, passes, hist, gate);
  bool in_b = false;
  for (int p = 0; p < passes; ++p) {
    const K* ki = p == 0 ? first : (in_b ? keys_b : keys_a);
    const uint32_t* vi = p == 0 ? first_vals : (in_b ? vals_b : vals_a);
    K* ko = in_b ? keys_a : keys_b;
    uint32_t* vo = in_b ? vals_a : vals_b;
    const uint32_t epoch = g_epoch.fetch_add(1) + 1;
    launch(pass_kernel<K>, tiles, kBlock, Tile<K>::kSmem, stream, 
        ki, vi, ko, vo, n32, p * kBits, hist + p * kBins, status, tile_ctr + p, epoch, gate,
        p == passes - 1 ? meta : SortMeta{});
    in_b = !in_b;
  }
  HPS_LAUNCH_CHECK_N(1 + passes);
  return in_b;
}

// The large path's scratch counters, zeroed ahead of a sort_pairs(zero_scratch = false)
// (a sort captured inside a conditional graph body launches kernels only).
inline void sort_scratch_zero(uint32_t* scratch, cudaStream_t stream) {
  HPS_CUDA(cudaMemsetAsync(scratch, 0, (kMaxPasses * kBins + kMaxPasses * 2) * sizeof(uint32_t),
                           stream));
}

// The small composite path (see small_composite_kernel).
inline void sort_composite_small(const unsigned long long* keys, const uint32_t* n_dev, int lbits,
                                 uint32_t* out_slot, uint32_t* out_listing,
                                 cudaStream_t stream) {
  launch(small_composite_kernel, kSmallN * 32 / kRankBlock, kRankBlock, 0, stream, 
      keys, n_dev, lbits, out_slot, out_listing);
  HPS_LAUNCH_CHECK();
}

// Exclusive scan of one row of `tiles` u32 per block (blockIdx.x = row), in place;
// totals[row] receives the row sum. Used for small host-sized scans.
static __global__ void __launch_bounds__(1024) scan_digits(uint32_t* __restrict__ hist,
                                                           uint32_t tiles,
                                                           uint32_t* __restrict__ totals) {
  pdl_entry();
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry;
  uint32_t* row = hist + static_cast<uint64_t>(blockIdx.x) * tiles;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < tiles; base += 1024) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < tiles ? row[i] : 0;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t s = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;
    }
    __syncthreads();
    uint32_t excl = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
    if (i < tiles) row[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

}  // namespace radix
}  // namespace hps
