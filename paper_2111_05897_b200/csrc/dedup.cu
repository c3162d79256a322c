// Batch ID de-duplication: sorted unique ids + inverse
// index, and the reference's compress_indices (codec.hpp:123-156) -- per group,
// unique ids ascending with ascending postings, within-sample duplicates collapsed.
//
// Both are a stable LSD radix sort of (key, listing) pairs followed by head flags
// and an exclusive scan. The sort uses only the key bits that vary (the OR of all
// ids bounds them), so a 27-bit id space costs 4 passes, not 8.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "radix_sort.cuh"
#include "table.cuh"
#include "table_impl.h"

namespace hps {

namespace {

constexpr int kScanTile = 4096;

__global__ void or_reduce_kernel(const uint64_t* __restrict__ k, uint64_t n,
                                 unsigned long long* out) {
  pdl_entry();
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc |= k[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicOr(out, (unsigned long long)acc);
}

__global__ void tile_sum_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                uint32_t* __restrict__ sums) {
  pdl_entry();
  __shared__ uint32_t s[32];
  uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint32_t acc = 0;
  for (int j = threadIdx.x; j < kScanTile; j += blockDim.x)
    if (base + j < n) acc += in[base + j];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    sums[blockIdx.x] = t;
  }
}

// Exclusive scan of one tile (1024 threads x 4 items) plus the tile's carried-in
// offset.
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ in,
                                                         uint64_t n,
                                                         const uint32_t* __restrict__ offs,
                                                         uint32_t* __restrict__ out) {
  pdl_entry();
  __shared__ uint32_t ws[32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + threadIdx.x * 4;
  uint32_t v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = base + k < n ? in[base + k] : 0;
  uint32_t local = v[0] + v[1] + v[2] + v[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    ws[lane] = s;
  }
  __syncthreads();
  uint32_t run = offs[blockIdx.x] + (warp ? ws[warp - 1] : 0) + x - local;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

// head[p] = 1 when sorted key p starts a run; for compress_indices also when the
// group changes (key2) and, separately, a posting head when the sample changes.
__global__ void dedup_flags_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                   uint32_t* __restrict__ head) {
  pdl_entry();
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1u : 0u;
}

__global__ void dedup_emit_kernel(const uint64_t* __restrict__ keys,
                                  const uint32_t* __restrict__ vals,
                                  const uint32_t* __restrict__ head,
                                  const uint32_t* __restrict__ excl, uint64_t n,
                                  uint64_t* __restrict__ unique, uint32_t* __restrict__ inverse,
                                  uint64_t* __restrict__ out_u) {
  pdl_entry();
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u = excl[p] + head[p] - 1;
    if (head[p]) unique[u] = keys[p];
    inverse[vals[p]] = u;
    if (p == n - 1) *out_u = u + 1;
  }
}

__global__ void ci_expand_kernel(const uint32_t* __restrict__ off, uint32_t B, uint32_t G,
                                 uint32_t* __restrict__ lgrp) {
  pdl_entry();
  for (uint32_t sg = blockIdx.x * blockDim.x + threadIdx.x; sg < B * G;
       sg += gridDim.x * blockDim.x)
    for (uint32_t i = off[sg]; i < off[sg + 1]; ++i) lgrp[i] = sg;
}

__global__ void ci_group_keys_kernel(const uint32_t* __restrict__ vals,
                                     const uint32_t* __restrict__ lgrp, uint32_t G, uint64_t n,
                                     uint32_t* __restrict__ gkeys) {
  pdl_entry();
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x)
    gkeys[p] = lgrp[vals[p]] % G;
}

// After sorting by (group, id) with listings in sample order inside each run:
// uflag = new (group, id); pflag = new posting (new run or new sample).
__global__ void ci_flags_kernel(const uint32_t* __restrict__ vals,
                                const uint64_t* __restrict__ ids,
                                const uint32_t* __restrict__ lgrp, uint32_t G, uint64_t n,
                                uint32_t* __restrict__ uflag, uint32_t* __restrict__ pflag,
                                uint32_t* __restrict__ group_cnt) {
  pdl_entry();
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t i = vals[p];
    uint32_t lg = lgrp[i];
    bool u = true, q = true;
    if (p > 0) {
      uint32_t j = vals[p - 1];
      uint32_t lg2 = lgrp[j];
      u = (lg % G) != (lg2 % G) || ids[i] != ids[j];
      q = u || (lg / G) != (lg2 / G);
    }
    uflag[p] = u;
    pflag[p] = q;
    if (u) atomicAdd(&group_cnt[lg % G], 1u);
  }
}

__global__ void ci_emit_kernel(const uint32_t* __restrict__ vals, const uint64_t* __restrict__ ids,
                               const uint32_t* __restrict__ lgrp, uint32_t G, uint64_t n,
                               const uint32_t* __restrict__ uflag,
                               const uint32_t* __restrict__ uex,
                               const uint32_t* __restrict__ pflag,
                               const uint32_t* __restrict__ pex, uint64_t* __restrict__ unique,
                               uint64_t* __restrict__ post_off, uint16_t* __restrict__ postings) {
  pdl_entry();
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t i = vals[p];
    if (uflag[p]) {
      unique[uex[p]] = ids[i];
      post_off[uex[p]] = pex[p];
    }
    if (pflag[p]) postings[pex[p]] = static_cast<uint16_t>(lgrp[i] / G);
    if (p == n - 1) post_off[uex[p] + uflag[p]] = pex[p] + pflag[p];
  }
}

__global__ void ci_group_off_kernel(const uint32_t* __restrict__ cnt, uint32_t G,
                                    uint64_t* __restrict__ out) {
  pdl_entry();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    uint64_t run = 0;
    out[0] = 0;
    for (uint32_t g = 0; g < G; ++g) {
      run += cnt[g];
      out[g + 1] = run;
    }
  }
}

struct Scratch {
  void* p[12] = {};
  ~Scratch() {
    for (void* q : p)
      if (q) cudaFree(q);
  }
  template <typename T>
  T* get(int i, uint64_t n) {
    HPS_CUDA(cudaMalloc(&p[i], std::max<uint64_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p[i]);
  }
};

uint32_t grid_for(uint64_t n) { return std::max<uint32_t>(1, std::min<uint64_t>(ceil_div(n, 256), 148 * 16)); }

}  // namespace

// out = exclusive scan of in[0..n); returns the total through *total (device).
void exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* tile_sums,
                    uint32_t* total, cudaStream_t st) {
  uint32_t tiles = ceil_div(n, kScanTile);
  launch(tile_sum_kernel, tiles, 256, 0, st, in, n, tile_sums);
  launch(radix::scan_digits, 1, 1024, 0, st, tile_sums, tiles, total);
  launch(tile_scan_kernel, tiles, 1024, 0, st, in, n, tile_sums, out);
  HPS_LAUNCH_CHECK_N(3);
}

namespace {

int key_bits_of(const uint64_t* keys, uint64_t n, unsigned long long* d_or, cudaStream_t st) {
  HPS_CUDA(cudaMemsetAsync(d_or, 0, sizeof(unsigned long long), st));
  launch(or_reduce_kernel, grid_for(n), 256, 0, st, keys, n, d_or);
  unsigned long long h = 0;
  HPS_CUDA(cudaMemcpyAsync(&h, d_or, sizeof(h), cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
  return bits_for(h);
}

}  // namespace

void dedup(const uint64_t* ids, uint64_t n, uint64_t* out_unique, uint32_t* out_inverse,
           uint64_t* out_u, cudaStream_t st) {
  if (n >= 0xffffffffull) throw Error(HPS_E_PRECONDITION, "dedup: too many ids");
  if (!out_u) throw Error(HPS_E_PRECONDITION, "dedup: out_u required");
  if (n == 0) {
    *out_u = 0;
    return;
  }
  StagePool pool;
  Stager stg(pool);
  const uint64_t* d_ids = static_cast<const uint64_t*>(stg.in(ids, n * sizeof(uint64_t), st));
  uint64_t* d_uni = static_cast<uint64_t*>(stg.out(out_unique, n * sizeof(uint64_t)));
  uint32_t* d_inv = static_cast<uint32_t*>(stg.out(out_inverse, n * sizeof(uint32_t)));
  Scratch s;
  uint64_t* ka = s.get<uint64_t>(0, n);
  uint64_t* kb = s.get<uint64_t>(1, n);
  uint32_t* va = s.get<uint32_t>(2, n);
  uint32_t* vb = s.get<uint32_t>(3, n);
  uint32_t* hist = s.get<uint32_t>(4, radix::scratch_words<uint64_t>(n));
  uint32_t* head = s.get<uint32_t>(5, n);
  uint32_t* ex = s.get<uint32_t>(6, n);
  uint32_t* tsum = s.get<uint32_t>(7, ceil_div(n, kScanTile) + 1);
  unsigned long long* d_or = s.get<unsigned long long>(8, 1);
  uint64_t* d_u = s.get<uint64_t>(9, 1);
  HPS_CUDA(cudaMemcpyAsync(ka, d_ids, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  launch_iota(va, n, st);
  int bits = key_bits_of(ka, n, d_or, st);
  bool in_b = radix::sort_pairs<uint64_t>(ka, va, kb, vb, n, bits, hist, st);
  const uint64_t* sk = in_b ? kb : ka;
  const uint32_t* sv = in_b ? vb : va;
  launch(dedup_flags_kernel, grid_for(n), 256, 0, st, sk, n, head);
  exclusive_scan(head, ex, n, tsum, tsum + ceil_div(n, kScanTile), st);
  launch(dedup_emit_kernel, grid_for(n), 256, 0, st, sk, sv, head, ex, n, d_uni, d_inv, d_u);
  HPS_LAUNCH_CHECK();
  HPS_CUDA(cudaMemcpyAsync(out_u, d_u, sizeof(uint64_t),
                           is_device_ptr(out_u) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           st));
  HPS_CUDA(cudaStreamSynchronize(st));
  stg.finish(st);
}

void compress_indices(const uint64_t* ids, uint64_t n, const uint32_t* offsets, uint32_t B,
                      uint32_t G, uint64_t* group_u_off, uint64_t* unique, uint64_t* post_off,
                      uint16_t* postings, cudaStream_t st) {
  if (B > 65535)
    throw Error(HPS_E_PRECONDITION, "compress_indices: batch size " + std::to_string(B) +
                                        " overflows uint16 sample indices");
  if (n >= 0xffffffffull) throw Error(HPS_E_PRECONDITION, "compress_indices: too many ids");
  StagePool pool;
  Stager stg(pool);
  const uint64_t BG = static_cast<uint64_t>(B) * G;
  const uint64_t* d_ids = static_cast<const uint64_t*>(stg.in(ids, n * sizeof(uint64_t), st));
  const uint32_t* d_off =
      static_cast<const uint32_t*>(stg.in(offsets, (BG + 1) * sizeof(uint32_t), st));
  uint64_t* d_guo = static_cast<uint64_t*>(stg.out(group_u_off, (G + 1) * sizeof(uint64_t)));
  uint64_t* d_uni = static_cast<uint64_t*>(stg.out(unique, std::max<uint64_t>(n, 1) * 8));
  uint64_t* d_po = static_cast<uint64_t*>(stg.out(post_off, (n + 1) * sizeof(uint64_t)));
  uint16_t* d_ps = static_cast<uint16_t*>(stg.out(postings, std::max<uint64_t>(n, 1) * 2));
  Scratch s;
  uint32_t* gcnt = s.get<uint32_t>(0, G + 1);
  HPS_CUDA(cudaMemsetAsync(gcnt, 0, (G + 1) * sizeof(uint32_t), st));
  if (n == 0) {
    launch(ci_group_off_kernel, 1, 32, 0, st, gcnt, G, d_guo);
    HPS_CUDA(cudaMemsetAsync(d_po, 0, sizeof(uint64_t), st));
    stg.finish(st);
    return;
  }
  uint64_t* ka = s.get<uint64_t>(1, n);
  uint64_t* kb = s.get<uint64_t>(2, n);
  uint32_t* va = s.get<uint32_t>(3, n);
  uint32_t* vb = s.get<uint32_t>(4, n);
  uint32_t* hist = s.get<uint32_t>(5, radix::scratch_words<uint64_t>(n));
  uint32_t* lgrp = s.get<uint32_t>(6, n);
  uint32_t* fl = s.get<uint32_t>(7, n);
  uint32_t* ex = s.get<uint32_t>(8, n);
  uint32_t* fl2 = s.get<uint32_t>(9, n);
  uint32_t* ex2 = s.get<uint32_t>(10, n);
  uint32_t* tsum = s.get<uint32_t>(11, 2 * (ceil_div(n, kScanTile) + 1));
  unsigned long long* d_or = reinterpret_cast<unsigned long long*>(kb);  // reused before sorting
  launch(ci_expand_kernel, grid_for(BG), 256, 0, st, d_off, B, G, lgrp);
  HPS_CUDA(cudaMemcpyAsync(ka, d_ids, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  launch_iota(va, n, st);
  int bits = key_bits_of(ka, n, d_or, st);
  // Pass 1: stable by id (listing order keeps samples ascending within an id).
  bool in_b = radix::sort_pairs<uint64_t>(ka, va, kb, vb, n, bits, hist, st);
  uint32_t* v1 = in_b ? vb : va;
  // Pass 2: stable by group.
  uint32_t* gk = reinterpret_cast<uint32_t*>(in_b ? ka : kb);
  uint32_t* gk2 = reinterpret_cast<uint32_t*>(in_b ? kb : ka) ;
  launch(ci_group_keys_kernel, grid_for(n), 256, 0, st, v1, lgrp, G, n, gk);
  uint32_t* v2 = in_b ? va : vb;
  bool in2 = radix::sort_pairs<uint32_t>(gk, v1, gk2, v2, n,
                                         std::max(1, bits_for(G - 1)), hist, st);
  const uint32_t* sv = in2 ? v2 : v1;
  launch(ci_flags_kernel, grid_for(n), 256, 0, st, sv, d_ids, lgrp, G, n, fl, fl2, gcnt);
  uint32_t tiles = ceil_div(n, kScanTile);
  exclusive_scan(fl, ex, n, tsum, tsum + tiles, st);
  exclusive_scan(fl2, ex2, n, tsum + tiles + 1, tsum + 2 * tiles + 1, st);
  launch(ci_emit_kernel, grid_for(n), 256, 0, st, sv, d_ids, lgrp, G, n, fl, ex, fl2, ex2, d_uni, d_po,
                                               d_ps);
  launch(ci_group_off_kernel, 1, 32, 0, st, gcnt, G, d_guo);
  HPS_LAUNCH_CHECK();
  HPS_CUDA(cudaStreamSynchronize(st));
  stg.finish(st);
}

}  // namespace hps
