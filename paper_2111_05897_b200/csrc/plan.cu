// Per-batch apply plan: which listings can be applied independently and which need
// the ordered per-row recurrence.
//
// During the probe every listing adds 1 to its row's batch counter, which lives in
// the row's hash entry (the sector the probe just read, so counting costs no extra
// DRAM traffic). A row listed once in the batch ("single") gets exactly one optimizer
// application, so its listing needs no ordering at all -- for the one-hot Criteo
// shape that is >99% of all listings. Listings of rows hit more than once ("multi")
// are appended as composite keys (slot << lbits | listing) -- one atomic per block --
// and ordered by the one-CTA composite sort when there are at most kSmallN of them;
// beyond that the whole batch takes the large slot sort instead (radix_sort.cuh), the
// choice being made on the device. Single rows' counters are cleared right here;
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
}  // namespace

__global__ void __launch_bounds__(kPlanBlock)
    classify_kernel(DevTable t, const uint32_t* __restrict__ slots,
                    const uint32_t* __restrict__ eidx, uint64_t n, int lbits,
                    uint8_t* __restrict__ kind, unsigned long long* __restrict__ mkeys,
                    uint32_t* __restrict__ n_multi) {
  __shared__ uint32_t s_warp[kPlanBlock / 32];
  __shared__ uint32_t s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kPlanBlock;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kPlanBlock + threadIdx.x;
       base - threadIdx.x < n; base += stride * kPlanItems) {
    uint32_t s[kPlanItems], e[kPlanItems], c[kPlanItems];
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j) {
      const uint64_t i = base + j * stride;
      s[j] = i < n ? slots[i] : kInvalidSlot;
      e[j] = i < n ? eidx[i] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j)
      c[j] = s[j] < t.capacity ? (e[j] == kSpecialEntry ? *t.special_cnt : t.ht[e[j]].cnt) : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j) {
      const uint64_t i = base + j * stride;
      const bool multi = c[j] > 1;
      mine += multi;
      if (i < n) kind[i] = multi ? 2 : 1;
      // A single row's counter is read by exactly this listing: clear it now, while
      // its sector is resident.
      if (c[j] == 1) {
        if (e[j] == kSpecialEntry) *t.special_cnt = 0;
        else t.ht[e[j]].cnt = 0;
      }
    }
    // block-aggregated append position (order is restored by the composite sort)
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
      for (int w = 0; w < kPlanBlock / 32; ++w) {
        const uint32_t cw = s_warp[w];
        s_warp[w] = run;
        run += cw;
      }
      s_base = run ? atomicAdd(n_multi, run) : 0u;
    }
    __syncthreads();
    uint32_t pos = s_base + s_warp[warp] + x - mine;
#pragma unroll
    for (int j = 0; j < kPlanItems; ++j) {
      if (c[j] > 1) {
        const uint64_t i = base + j * stride;
        mkeys[pos++] = (static_cast<unsigned long long>(s[j]) << lbits) | i;
      }
    }
    __syncthreads();
  }
}

void launch_classify(const DevTable& t, const uint32_t* slots, const uint32_t* eidx, uint64_t n,
                     int lbits, uint8_t* kind, unsigned long long* mkeys, uint32_t* n_multi,
                     int sms, cudaStream_t st) {
  HPS_CUDA(cudaMemsetAsync(n_multi, 0, sizeof(uint32_t), st));
  if (!n) return;
  const uint32_t blocks =
      std::min<uint64_t>(ceil_div(n, kPlanBlock * kPlanItems), static_cast<uint64_t>(sms) * 8);
  classify_kernel<<<blocks, kPlanBlock, 0, st>>>(t, slots, eidx, n, lbits, kind, mkeys, n_multi);
  HPS_LAUNCH_CHECK();
}

}  // namespace hps
