// Per-batch apply plan: which listings can be applied independently and which need
// the ordered per-row recurrence.
//
// A row listed once in the batch ("single") gets exactly one optimizer application,
// so its listing needs no ordering at all -- for the one-hot Criteo shape that is >99%
// of all listings. The probe sets the row's bit in `seen` and, if it was already set,
// in `multi` (two bitmaps of one bit per slot: 25 MB for 100M rows, L2-resident, so
// every plan access is an L2 hit). This kernel then reads each listing's `multi` bit,
// clears `seen` for the next batch, and appends multi listings as composite keys
// (slot << lbits | listing) -- one atomic per block -- for the one-CTA sort, until
// more than kSmallN are known (then the whole batch takes the large slot sort, chosen
// on the device). `multi` bits are cleared by the update that consumes them; a batch
// that is never pushed leaves them set, which can only move later rows from the single
// path to the (always correct) multi path.
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
}  // namespace

__global__ void __launch_bounds__(kPlanBlock)
    classify_kernel(DevTable t, const uint32_t* __restrict__ slots, uint64_t n, int lbits,
                    uint8_t* __restrict__ kind, unsigned long long* __restrict__ mkeys,
                    uint32_t* __restrict__ n_multi, uint32_t* __restrict__ slist,
                    uint32_t* __restrict__ n_single, const uint32_t* n_live) {
  pdl_entry();
  if (n_live) n = min(n, static_cast<uint64_t>(*n_live));
  __shared__ uint32_t s_warp[kPlanBlock / 32];
  __shared__ uint32_t s_base;
  __shared__ bool s_open;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kPlanBlock;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kPlanBlock + threadIdx.x;
       base - threadIdx.x < n; base += stride * kPlanItems) {
    uint32_t s[kPlanItems], w[kPlanItems];
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j) {
      const uint64_t i = base + j * stride;
      s[j] = i < n ? slots[i] : kInvalidSlot;
    }
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j) w[j] = s[j] < t.capacity ? __ldcg(&t.multi[s[j] >> 5]) : 0u;
    uint32_t mine = 0, mbits = 0, sbits = 0;
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j) {
      const uint64_t i = base + j * stride;
      const bool multi = (w[j] >> (s[j] & 31)) & 1u;
      mbits |= multi ? 1u << j : 0u;
      mine += multi;
      if (i < n && s[j] < t.capacity && !multi) sbits |= 1u << j;
      if (i < n)  // (keeps expand_groups' kKindAlone bit)
        kind[i] = (kind[i] & kKindAlone) | (s[j] < t.capacity ? (multi ? 2 : 1) : 0);
      if (s[j] < t.capacity) atomicAnd(&t.seen[s[j] >> 5], ~(1u << (s[j] & 31)));
    }
    // multi-hot batches: the single-listing list (update_single walks it on a large
    // plan) -- block-aggregated appends, one atomic per block and pass, order irrelevant
    // (independent rows)
    if (slist) {  // (block-uniform)
      const uint32_t ns = __popc(sbits);
      uint32_t xs = ns;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
        if (lane >= o) xs += y;
      }
      __syncthreads();  // (s_warp / s_base free from the previous pass)
      if (lane == 31) s_warp[warp] = xs;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int q = 0; q < kPlanBlock / 32; ++q) {
          const uint32_t cw = s_warp[q];
          s_warp[q] = run;
          run += cw;
        }
        s_base = run ? atomicAdd(n_single, run) : 0u;
      }
      __syncthreads();
      uint32_t pos = s_base + s_warp[warp] + xs - ns;
#pragma unroll
      for (int j = 0; j < kPlanItems; ++j)
        if (sbits & (1u << j)) slist[pos++] = static_cast<uint32_t>(base + j * stride);
      __syncthreads();  // (s_warp / s_base reused below)
    }
    // block-aggregated append position (order is restored by the composite sort);
    // every branch below is block-uniform
    if (!__syncthreads_or(mine != 0)) continue;
    if (threadIdx.x == 0) s_open = ld_volatile(n_multi) <= radix::kSmallN;
    __syncthreads();
    if (!s_open) continue;
    uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      for (int q = 0; q < kPlanBlock / 32; ++q) {
        const uint32_t cw = s_warp[q];
        s_warp[q] = run;
        run += cw;
      }
      s_base = atomicAdd(n_multi, run);
    }
    __syncthreads();
    uint32_t pos = s_base + s_warp[warp] + x - mine;
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j) {
      if (mbits & (1u << j)) {
        if (pos < radix::kSmallN)
          mkeys[pos] = (static_cast<unsigned long long>(s[j]) << lbits) | (base + j * stride);
        ++pos;
      }
    }
  }
}

void launch_classify(const DevTable& t, const uint32_t* slots, uint64_t n, int lbits,
                     uint8_t* kind, unsigned long long* mkeys, uint32_t* n_multi,
                     uint32_t* slist, uint32_t* n_single, int sms, cudaStream_t st,
                     const uint32_t* n_live) {
  // (n_multi is zeroed by the batch's register, with its other scalars)
  if (!n) return;
  const uint32_t blocks =
      std::min<uint64_t>(ceil_div(n, kPlanBlock * kPlanItems), static_cast<uint64_t>(sms) * 8);
  launch(classify_kernel, blocks, kPlanBlock, 0, st, t, slots, n, lbits, kind, mkeys, n_multi,
         slist, n_single, n_live);
  HPS_LAUNCH_CHECK();
}

}  // namespace hps
