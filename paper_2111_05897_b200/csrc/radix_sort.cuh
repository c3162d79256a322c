// Stable LSD radix sort of (key, value) pairs, hand-written for sm_100a.
//
// Used for the two orderings the hot path needs:
//   * listings grouped by table slot, listing order preserved inside a slot (the
//     per-row apply order of the ordered optimizer update), u32 keys;
//   * ids sorted ascending with their positions (batch dedup / compress_indices),
//     u64 keys.
// Each 8-bit pass is reduce-then-scan: upsweep (per-tile digit histogram) ->
// per-digit scan over tiles -> downsweep (stable in-tile ranking with
// __match_any_sync, staging the tile in shared memory in digit order so the global
// scatter is written in contiguous runs). Keys/values are read and written once
// per pass: 2*(sizeof(K)+sizeof(V)) bytes per element per pass.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hps {
namespace radix {

constexpr int kBits = 8;
constexpr int kBins = 1 << kBits;
constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

template <typename K>
struct Tile {
  static constexpr int kItems = sizeof(K) == 8 ? 8 : 16;
  static constexpr int kTile = kBlock * kItems;
  static constexpr size_t kSmem =
      kTile * (sizeof(K) + sizeof(uint32_t)) + (kWarps * kBins + 3 * kBins) * sizeof(uint32_t);
};

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return static_cast<uint32_t>(key >> shift) & (kBins - 1);
}

// hist[d * tiles + tile] = count of digit d in tile.
template <typename K>
__global__ void __launch_bounds__(kBlock) upsweep(const K* __restrict__ keys, uint32_t n, int shift,
                                                  uint32_t* __restrict__ hist, uint32_t tiles) {
  constexpr int kTileN = Tile<K>::kTile;
  __shared__ uint32_t cnt[kWarps][kBins];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kBins; i += kBlock) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTileN;
#pragma unroll 4
  for (int j = 0; j < Tile<K>::kItems; ++j) {
    uint64_t idx = base + static_cast<uint64_t>(j) * kBlock + threadIdx.x;
    if (idx < n) atomicAdd(&cnt[warp][digit_of(keys[idx], shift)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kBins; d += kBlock) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += cnt[w][d];
    hist[static_cast<uint64_t>(d) * tiles + blockIdx.x] = s;
  }
}

// One block per digit: exclusive scan of hist[d, 0..tiles) in place; totals[d].
static __global__ void __launch_bounds__(1024) scan_digits(uint32_t* __restrict__ hist, uint32_t tiles,
                                                    uint32_t* __restrict__ totals) {
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
      warp_sums[lane] = s;  // inclusive
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

// Block-wide exclusive scan of one value per thread for the first kBins threads.
__device__ __forceinline__ uint32_t block_excl_scan_bins(uint32_t v, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  uint32_t off = 0;
  for (int w = 0; w < warp; ++w) off += scratch[w];
  __syncthreads();
  return off + x - v;
}

template <typename K>
__global__ void __launch_bounds__(kBlock)
    downsweep(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
              K* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
              const uint32_t* __restrict__ hist, const uint32_t* __restrict__ totals,
              uint32_t tiles) {
  constexpr int kItems = Tile<K>::kItems;
  constexpr int kTileN = Tile<K>::kTile;
  extern __shared__ __align__(16) unsigned char smem[];
  K* skeys = reinterpret_cast<K*>(smem);
  uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + kTileN);
  uint32_t* wcnt = svals + kTileN;            // [kWarps][kBins]
  uint32_t* block_off = wcnt + kWarps * kBins;  // [kBins]
  uint32_t* gbase = block_off + kBins;          // [kBins]
  uint32_t* scratch = gbase + kBins;            // [kBins] (uses 32)

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kBins; i += kBlock) wcnt[i] = 0;

  // Global base of every digit for this tile: digit start + this tile's offset.
  {
    uint32_t d = threadIdx.x;  // kBlock == kBins
    uint32_t tot = totals[d];
    uint32_t start = block_excl_scan_bins(tot, scratch);
    gbase[d] = start + hist[static_cast<uint64_t>(d) * tiles + blockIdx.x];
  }
  __syncthreads();

  const uint64_t tile_base = static_cast<uint64_t>(blockIdx.x) * kTileN;
  const uint64_t warp_base = tile_base + static_cast<uint64_t>(warp) * 32 * kItems;
  K k[kItems];
  uint32_t v[kItems];
  uint32_t r[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    uint64_t idx = warp_base + static_cast<uint64_t>(j) * 32 + lane;
    bool ok = idx < n;
    k[j] = ok ? keys_in[idx] : K(0);
    v[j] = ok ? vals_in[idx] : 0u;
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
  {
    uint32_t d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      uint32_t t = wcnt[w * kBins + d];
      wcnt[w * kBins + d] = run;
      run += t;
    }
    block_off[d] = block_excl_scan_bins(run, scratch);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    uint64_t idx = warp_base + static_cast<uint64_t>(j) * 32 + lane;
    if (idx < n) {
      uint32_t d = digit_of(k[j], shift);
      uint32_t pos = block_off[d] + wcnt[warp * kBins + d] + r[j];
      skeys[pos] = k[j];
      svals[pos] = v[j];
    }
  }
  __syncthreads();
  const uint32_t tile_n = static_cast<uint32_t>(n - tile_base < (uint64_t)kTileN ? n - tile_base : (uint64_t)kTileN);
  for (uint32_t p = threadIdx.x; p < tile_n; p += kBlock) {
    K key = skeys[p];
    uint32_t d = digit_of(key, shift);
    uint32_t g = gbase[d] + (p - block_off[d]);
    keys_out[g] = key;
    vals_out[g] = svals[p];
  }
}

// Scratch sizing for sorting n pairs.
template <typename K>
inline size_t hist_words(uint64_t n) {
  uint64_t tiles = (n + Tile<K>::kTile - 1) / Tile<K>::kTile;
  return static_cast<size_t>(tiles ? tiles : 1) * kBins + kBins;
}

// Sorts (keys, vals) by key bits [0, key_bits). Ping-pongs between the (a) and (b)
// buffers; returns true when the result lives in the (b) buffers. hist needs
// hist_words<K>(n) words.
template <typename K>
inline bool sort_pairs(K* keys_a, uint32_t* vals_a, K* keys_b, uint32_t* vals_b, uint32_t n,
                       int key_bits, uint32_t* hist, cudaStream_t stream) {
  if (n <= 1 || key_bits <= 0) return false;
  static bool attr_set = false;
  if (!attr_set) {
    HPS_CUDA(cudaFuncSetAttribute(downsweep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tile<K>::kSmem)));
    attr_set = true;
  }
  const uint32_t tiles = ceil_div(n, Tile<K>::kTile);
  uint32_t* totals = hist + static_cast<size_t>(tiles) * kBins;
  bool in_b = false;
  for (int shift = 0; shift < key_bits; shift += kBits) {
    const K* ki = in_b ? keys_b : keys_a;
    const uint32_t* vi = in_b ? vals_b : vals_a;
    K* ko = in_b ? keys_a : keys_b;
    uint32_t* vo = in_b ? vals_a : vals_b;
    upsweep<K><<<tiles, kBlock, 0, stream>>>(ki, n, shift, hist, tiles);
    scan_digits<<<kBins, 1024, 0, stream>>>(hist, tiles, totals);
    downsweep<K><<<tiles, kBlock, Tile<K>::kSmem, stream>>>(ki, vi, ko, vo, n, shift, hist, totals,
                                                             tiles);
    HPS_LAUNCH_CHECK_N(3);
    in_b = !in_b;
  }
  return in_b;
}

}  // namespace radix
}  // namespace hps
