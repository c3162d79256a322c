// Per-batch apply plan: which listings can be applied independently and which need
// the ordered per-row recurrence.
//
// During the probe every listing adds 1 to its row's batch counter, which lives in
// the row's hash entry (the sector the probe just read, so counting costs no extra
// DRAM traffic). A row listed once in the batch ("single") gets exactly one optimizer
// application, so its listing needs no ordering at all -- for the one-hot Criteo
// shape that is >99% of all listings. Listings of rows hit more than once ("multi")
// are compacted, in listing (= apply) order, by a single-pass chained scan, and only
// they go through the stable slot sort. Single rows' counters are cleared right here;
// multi rows' by the update that consumes them -- a batch that is never pushed leaves
// those high, which can only move later rows from the single path to the (always
// correct) multi path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "radix_sort.cuh"
#include "table.cuh"
#include "vec.cuh"

namespace hps {

namespace {
constexpr int kPlanBlock = 256;
constexpr int kPlanItems = 4;
constexpr int kPlanTile = kPlanBlock * kPlanItems;
}  // namespace

// kind[i] = 1 single / 2 multi; multi listings are written, in listing order, to
// (mkeys = slot, mvals = listing) and counted into *n_multi. One tile per block,
// dynamically numbered; tile prefixes by decoupled look-back (status words as in
// radix_sort.cuh: [63:32] epoch, [31] prefix flag, [30:0] count).
__global__ void __launch_bounds__(kPlanBlock)
    classify_kernel(DevTable t, const uint32_t* __restrict__ slots,
                    const uint32_t* __restrict__ eidx, uint64_t n, uint8_t* __restrict__ kind,
                    uint32_t* __restrict__ mkeys, uint32_t* __restrict__ mvals,
                    uint32_t* __restrict__ n_multi, unsigned long long* status,
                    uint32_t* tile_ctr, uint32_t epoch) {
  __shared__ uint32_t s_tile, s_warp[kPlanBlock / 32], s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t tiles = static_cast<uint32_t>((n + kPlanTile - 1) / kPlanTile);
  if (tile >= tiles) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Lane owns kPlanItems consecutive listings of its warp's stripe, so the flag order
  // (warp, lane, item) is listing order.
  const uint64_t base = static_cast<uint64_t>(tile) * kPlanTile +
                        static_cast<uint64_t>(warp) * 32 * kPlanItems +
                        static_cast<uint64_t>(lane) * kPlanItems;
  uint32_t s[kPlanItems], e[kPlanItems], c[kPlanItems];
#pragma unroll
  for (int j = 0; j < kPlanItems; ++j) {
    const bool valid = base + j < n;
    s[j] = valid ? slots[base + j] : kInvalidSlot;
    e[j] = valid ? eidx[base + j] : 0u;
  }
#pragma unroll
  for (int j = 0; j < kPlanItems; ++j)
    c[j] = s[j] < t.capacity ? (e[j] == kSpecialEntry ? *t.special_cnt : t.ht[e[j]].cnt) : 0u;
  uint32_t mine = 0;
  uint32_t mbits = 0;
#pragma unroll
  for (int j = 0; j < kPlanItems; ++j) {
    const bool multi = c[j] > 1;
    mbits |= multi ? (1u << j) : 0u;
    mine += multi;
    if (base + j < n) kind[base + j] = multi ? 2 : 1;
    // A single row's counter is read by exactly this listing: clear it now, while its
    // sector is resident (multi rows are cleared by the update that consumes them).
    if (c[j] == 1) {
      if (e[j] == kSpecialEntry) *t.special_cnt = 0;
      else t.ht[e[j]].cnt = 0;
    }
  }
  // warp-inclusive scan of per-lane counts
  uint32_t x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < kPlanBlock / 32; ++w) tot += s_warp[w];
    const unsigned long long ep = static_cast<unsigned long long>(epoch) << 32;
    volatile unsigned long long* my = status + tile;
    if (lane == 0) *my = ep | (tile == 0 ? radix::kPrefixFlag : 0ull) | tot;
    const uint32_t excl = tile == 0 ? 0u : radix::warp_lookback(status, tile, epoch);
    if (lane == 0) {
      if (tile > 0) *my = ep | radix::kPrefixFlag | (excl + tot);
      uint32_t run = 0;
      for (int w = 0; w < kPlanBlock / 32; ++w) {
        uint32_t cw = s_warp[w];
        s_warp[w] = run;
        run += cw;
      }
      s_excl = excl;
      if (tile == tiles - 1) *n_multi = excl + tot;
    }
  }
  __syncthreads();
  uint32_t pos = s_excl + s_warp[warp] + x - mine;
#pragma unroll
  for (int j = 0; j < kPlanItems; ++j) {
    if (mbits & (1u << j)) {
      mkeys[pos] = s[j];
      mvals[pos] = static_cast<uint32_t>(base + j);
      ++pos;
    }
  }
}

void launch_classify(const DevTable& t, const uint32_t* slots, const uint32_t* eidx, uint64_t n,
                     uint8_t* kind, uint32_t* mkeys, uint32_t* mvals, uint32_t* n_multi,
                     unsigned long long* status, uint32_t* tile_ctr, cudaStream_t st) {
  if (!n) {
    HPS_CUDA(cudaMemsetAsync(n_multi, 0, sizeof(uint32_t), st));
    return;
  }
  HPS_CUDA(cudaMemsetAsync(tile_ctr, 0, sizeof(uint32_t), st));
  const uint32_t tiles = ceil_div(n, kPlanTile);
  const uint32_t epoch = radix::g_epoch.fetch_add(1) + 1;
  classify_kernel<<<tiles, kPlanBlock, 0, st>>>(t, slots, eidx, n, kind, mkeys, mvals, n_multi,
                                                status, tile_ctr, epoch);
  HPS_LAUNCH_CHECK();
}

size_t classify_status_words(uint64_t n) { return 2 * (ceil_div(n, kPlanTile) + 1); }

}  // namespace hps
