// Multi-GPU exchange plan for hash-sharded tables.
//
// Rows are owned by rank route_shard(id, S) % world -- the reference's ShardSet
// partitioning (embedding_ps.hpp:521-523) with the S logical shards spread round-robin
// over the GPUs. Per step and source rank:
//
//  forward   hps_exchange_route: the batch's distinct ids grouped by owner rank
//            (send_ids[U], counts[world]) and, per listing, its position in send_ids;
//            the owner looks the ids up (hps_lookup: find_or_init + gather + version);
//            hps_exchange_pool pools the returned rows (fp64, listing order,
//            embedding_worker.hpp:541-557) exactly as serve_pull does.
//  backward  hps_exchange_pairs: one contribution per (sample, distinct id), the fp64
//            chain-rule sum of push_to_shards (embedding_worker.hpp:726-775), grouped by
//            owner and, per id, in ascending sample order; the owner applies them with
//            hps_table_apply_pairs in (source rank, sample) order = ascending SampleId
//            (sid = rank << 56 | counter, core.hpp:98-125; flush order
//            embedding_worker.hpp:788-790), through PsShard::apply_gradients semantics.
//
// The collectives themselves (NCCL all-to-all of ids, rows, pairs) are issued by the
// caller between these calls (paper_2111_05897_b200/sharded.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "radix_sort.cuh"
#include "table.cuh"
#include "table_impl.h"
#include "vec.cuh"

namespace hps {

namespace {

constexpr int kXBlock = 256;
constexpr uint32_t kInserter = 0x80000000u;
constexpr uint32_t kNoPair = 0xffffffffu;
// x.cnt layout (u32 words): [0,32) distinct ids per owner, [32] special-id claim,
// [33] listings of multi-listed ids, [64,96) single pairs per owner.
constexpr int kCntSpecial = 32, kCntMulti = 33, kCntSingle = 64, kCntWords = 128;

// Distinct ids: a transient open-addressing set (keys only). The entry index of each
// listing's id is recorded; the thread whose CAS claimed the entry is its inserter and
// every other listing of the id marks the entry "multi". Entry H is the side entry of
// id ~0 (the empty marker).
__global__ void __launch_bounds__(kXBlock)
    x_insert_kernel(const uint64_t* __restrict__ ids, uint64_t n, uint64_t* hkeys,
                    uint64_t mask, int shift, uint32_t* special, uint32_t* __restrict__ hidx,
                    uint8_t* __restrict__ hmul) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = ids[i];
    uint32_t e;
    bool ins;
    if (id == kEmptyKey) {
      e = static_cast<uint32_t>(mask + 1);
      ins = atomicCAS(special, 0u, 1u) == 0u;
    } else {
      uint64_t h = mix64(id) >> shift;
      while (true) {
        const uint64_t k = hkeys[h];
        if (k == id) {
          ins = false;
          break;
        }
        if (k == kEmptyKey) {
          const unsigned long long old = atomicCAS(
              reinterpret_cast<unsigned long long*>(hkeys + h), kEmptyKey, id);
          if (old == kEmptyKey || old == id) {
            ins = old == kEmptyKey;
            break;
          }
        }
        h = (h + 1) & mask;
      }
      e = static_cast<uint32_t>(h);
    }
    if (!ins) hmul[e] = 1;
    hidx[i] = e | (ins ? kInserter : 0u);
  }
}

// Owner rank per listing; for inserters the id's index inside its owner's segment of
// send_ids; for ids listed once in the batch (their only listing is the inserter) the
// pair's index among the owner's single pairs (spair, else kNoPair). Block-aggregated
// counters: one global atomic per owner per block iteration.
__global__ void __launch_bounds__(kXBlock)
    x_number_kernel(const uint64_t* __restrict__ ids, uint64_t n, uint32_t S, uint32_t G,
                    const uint32_t* __restrict__ hidx, const uint8_t* __restrict__ hmul,
                    uint32_t* __restrict__ hval, uint8_t* __restrict__ dest,
                    uint32_t* __restrict__ spair, uint32_t* cnt) {
  __shared__ uint32_t bc[32], gb[32], sc[32], sb[32];
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < G) bc[threadIdx.x] = 0, sc[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t i = base + threadIdx.x;
    uint32_t d = 0, r = 0, q = 0, code = 0;
    bool single = false;
    const bool valid = i < n;
    if (valid) {
      code = hidx[i];
      d = route_shard(ids[i], S) % G;
      dest[i] = static_cast<uint8_t>(d);
      if (code & kInserter) {
        r = atomicAdd(&bc[d], 1u);
        single = hmul[code & ~kInserter] == 0;
        if (single) q = atomicAdd(&sc[d], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x < G) {
      gb[threadIdx.x] = bc[threadIdx.x] ? atomicAdd(&cnt[threadIdx.x], bc[threadIdx.x]) : 0;
      sb[threadIdx.x] =
          sc[threadIdx.x] ? atomicAdd(&cnt[kCntSingle + threadIdx.x], sc[threadIdx.x]) : 0;
    }
    __syncthreads();
    if (valid) {
      if (code & kInserter) hval[code & ~kInserter] = gb[d] + r;
      spair[i] = single ? sb[d] + q : kNoPair;
    }
    __syncthreads();
  }
}

// Segment starts from the per-owner counts (G <= 32), kept on the device for later calls.
__device__ __forceinline__ void load_seg(const uint32_t* cnt, uint32_t G, uint32_t* seg) {
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (uint32_t d = 0; d < G; ++d) {
      seg[d] = run;
      run += cnt[d];
    }
    seg[G] = run;
  }
  __syncthreads();
}

// Send position per listing, send_ids, and the composite keys (pos << lbits | listing)
// of listings whose id is listed more than once (while they fit the small sort).
__global__ void __launch_bounds__(kXBlock)
    x_scatter_kernel(const uint64_t* __restrict__ ids, uint64_t n, uint32_t G,
                     const uint32_t* __restrict__ hidx, const uint32_t* __restrict__ hval,
                     const uint8_t* __restrict__ dest, const uint32_t* __restrict__ spair,
                     uint32_t* cnt, int lbits, uint32_t* __restrict__ sendpos,
                     uint64_t* __restrict__ send_ids, uint32_t* __restrict__ seg_out,
                     unsigned long long* __restrict__ mkeys) {
  __shared__ uint32_t seg[33];
  __shared__ uint32_t s_n, s_base;
  load_seg(cnt, G, seg);
  if (blockIdx.x == 0 && threadIdx.x <= G) seg_out[threadIdx.x] = seg[threadIdx.x];
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const uint64_t i = base + threadIdx.x;
    uint32_t pos = 0, r = 0;
    bool multi = false;
    if (i < n) {
      const uint32_t code = hidx[i];
      pos = seg[dest[i]] + hval[code & ~kInserter];
      sendpos[i] = pos;
      if (code & kInserter) send_ids[pos] = ids[i];
      multi = spair[i] == kNoPair;
      if (multi) r = atomicAdd(&s_n, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(&cnt[kCntMulti], s_n) : 0;
    __syncthreads();
    if (multi && s_base + r < radix::kSmallN)
      mkeys[s_base + r] = (static_cast<unsigned long long>(pos) << lbits) | i;
    __syncthreads();
  }
}

// Pair heads over the sorted multi listings: a new (id, sample). n_host bounds the list;
// its live length is *n_multi on the small path, n_host on the large path (which sorts
// every listing -- single-pair listings are then skipped here).
__global__ void x_pair_flags_kernel(const uint32_t* __restrict__ spos,
                                    const uint32_t* __restrict__ slist,
                                    const uint32_t* __restrict__ lgrp,
                                    const uint32_t* __restrict__ spair, uint32_t F,
                                    uint64_t n_host, const uint32_t* __restrict__ n_multi,
                                    uint32_t* __restrict__ head) {
  const bool large = *n_multi > radix::kSmallN;
  const uint64_t n = large ? n_host : *n_multi;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n_host;
       p += (uint64_t)gridDim.x * blockDim.x) {
    bool h = false;
    if (p < n && spair[slist[p]] == kNoPair)
      h = p == 0 || spos[p] != spos[p - 1] || lgrp[slist[p]] / F != lgrp[slist[p - 1]] / F;
    head[p] = h ? 1u : 0u;
  }
}

// Multi pairs per owner and the owners' pair offsets: pair_off[d] = sum over d' < d of
// (single pairs + multi pairs of d'); mstart[d] = index of d's first multi pair. The
// multi pairs are sorted by send position and owner segments are contiguous, so owner
// d's multi pairs start at the first listing whose position >= seg[d].
__global__ void x_pair_bounds_kernel(const uint32_t* __restrict__ spos,
                                     const uint32_t* __restrict__ ex,
                                     const uint32_t* __restrict__ head, uint64_t n_host,
                                     const uint32_t* __restrict__ cnt,
                                     const uint32_t* __restrict__ seg, uint32_t G,
                                     uint64_t* __restrict__ pair_off,
                                     uint32_t* __restrict__ mstart) {
  __shared__ uint32_t ms[33];
  const uint32_t nm = cnt[kCntMulti];
  const uint64_t n = nm > radix::kSmallN ? n_host : nm;
  const uint32_t total = n ? ex[n - 1] + head[n - 1] : 0;
  const uint32_t d = threadIdx.x;
  if (d < G) {
    uint64_t lo = 0, hi = n;  // first p with spos[p] >= seg[d]
    while (lo < hi) {
      uint64_t mid = (lo + hi) / 2;
      if (spos[mid] < seg[d]) lo = mid + 1;
      else hi = mid;
    }
    ms[d] = lo < n ? ex[lo] : total;
  } else if (d == G) {
    ms[G] = total;
  }
  __syncthreads();
  if (d == 0) {
    uint64_t run = 0;
    for (uint32_t k = 0; k < G; ++k) {
      pair_off[k] = run;
      mstart[k] = ms[k];
      run += cnt[kCntSingle + k] + (ms[k + 1] - ms[k]);
    }
    pair_off[G] = run;
    mstart[G] = ms[G];
  }
}

template <int V, bool GEN>
__device__ __forceinline__ void put_row(float* dst, const float (&o)[V]) {
  if constexpr (GEN) {
    dst[0] = o[0];
  } else {
    store_vec<V>(dst, o);
  }
}

// Single pairs (an id listed once in the batch): streamed in listing order, the pair is
// the listing itself, c = (float)(0.0 + (double)g * scale), placed at pair_off[d] + its
// index among d's single pairs.
template <int V, int L, bool GEN>
__global__ void __launch_bounds__(kXBlock)
    x_single_emit_kernel(const uint32_t* __restrict__ spair, const uint8_t* __restrict__ dest,
                         const uint32_t* __restrict__ sendpos, const uint32_t* __restrict__ lgrp,
                         const uint32_t* __restrict__ offsets, uint64_t n, uint32_t D, int mean,
                         const float* __restrict__ grads, const uint32_t* __restrict__ seg,
                         const uint64_t* __restrict__ pair_off, uint32_t* __restrict__ pair_pos,
                         float* __restrict__ contrib) {
  const uint32_t lane = threadIdx.x % L;
  const uint64_t groups = (uint64_t)gridDim.x * (kXBlock / L);
  for (uint64_t i = blockIdx.x * (uint64_t)(kXBlock / L) + threadIdx.x / L; i < n;
       i += groups) {
    const uint32_t sp = spair[i];
    if (sp == kNoPair) continue;
    const uint32_t d = dest[i];
    const uint64_t out = pair_off[d] + sp;
    const uint32_t g = lgrp[i];
    if (lane == 0) pair_pos[out] = sendpos[i] - seg[d];
    const double scale = mean ? 1.0 / static_cast<double>(offsets[g + 1] - offsets[g]) : 1.0;
    for (uint32_t d0 = lane * V; d0 < D; d0 += L * V) {
      const float* src = grads + static_cast<uint64_t>(g) * D + d0;
      float x[V], o[V];
      if constexpr (GEN) {
        x[0] = src[0];
      } else {
        load_vec<V>(src, x);
      }
#pragma unroll
      for (int v = 0; v < V; ++v)
        o[v] = __double2float_rn(__dadd_rn(0.0, __dmul_rn(static_cast<double>(x[v]), scale)));
      put_row<V, GEN>(contrib + out * D + d0, o);
    }
  }
}

// Multi pairs: c = (float)(0.0 + sum over the pair's listings, ascending listing order =
// group then position order, of (double)g * scale) -- push_to_shards
// (embedding_worker.hpp:743-760); placed after owner d's single pairs.
template <int V, int L, bool GEN>
__global__ void __launch_bounds__(kXBlock)
    x_multi_emit_kernel(const uint32_t* __restrict__ spos, const uint32_t* __restrict__ slist,
                        const uint32_t* __restrict__ head, const uint32_t* __restrict__ ex,
                        const uint32_t* __restrict__ lgrp, const uint32_t* __restrict__ offsets,
                        uint32_t F, uint64_t n_host, const uint32_t* __restrict__ cnt,
                        uint32_t D, int mean, const float* __restrict__ grads,
                        const uint8_t* __restrict__ dest_of_pos,
                        const uint32_t* __restrict__ seg, const uint64_t* __restrict__ pair_off,
                        const uint32_t* __restrict__ mstart, uint32_t* __restrict__ pair_pos,
                        float* __restrict__ contrib) {
  const uint32_t nm = cnt[kCntMulti];
  const uint64_t n = nm > radix::kSmallN ? n_host : nm;
  const uint32_t lane = threadIdx.x % L;
  const uint64_t groups = (uint64_t)gridDim.x * (kXBlock / L);
  for (uint64_t p = blockIdx.x * (uint64_t)(kXBlock / L) + threadIdx.x / L; p < n;
       p += groups) {
    if (!head[p]) continue;
    const uint32_t pos = spos[p];
    const uint32_t sample = lgrp[slist[p]] / F;
    const uint32_t d = dest_of_pos[pos];
    const uint64_t out = pair_off[d] + cnt[kCntSingle + d] + (ex[p] - mstart[d]);
    if (lane == 0) pair_pos[out] = pos - seg[d];
    for (uint32_t d0 = lane * V; d0 < D; d0 += L * V) {
      double acc[V];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = 0.0;
      for (uint64_t q = p; q < n; ++q) {
        if (q != p && (spos[q] != pos || lgrp[slist[q]] / F != sample)) break;
        const uint32_t g = lgrp[slist[q]];
        const double scale =
            mean ? 1.0 / static_cast<double>(offsets[g + 1] - offsets[g]) : 1.0;
        const float* src = grads + static_cast<uint64_t>(g) * D + d0;
        float x[V];
        if constexpr (GEN) {
          x[0] = src[0];
        } else {
          load_vec<V>(src, x);
        }
#pragma unroll
        for (int v = 0; v < V; ++v)
          acc[v] = __dadd_rn(acc[v], __dmul_rn(static_cast<double>(x[v]), scale));
      }
      float o[V];
#pragma unroll
      for (int v = 0; v < V; ++v) o[v] = __double2float_rn(acc[v]);
      put_row<V, GEN>(contrib + out * D + d0, o);
    }
  }
}

// dest per send position (the owner of send_ids[pos]) from the segment table; U = seg[G]
// is device-side, the grid covers the host bound n >= U.
__global__ void x_dest_of_pos_kernel(const uint32_t* __restrict__ seg, uint32_t G, uint64_t n,
                                     uint8_t* __restrict__ out) {
  const uint64_t U = seg[G];
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < U && u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t d = 0;
    while (d + 1 < G && seg[d + 1] <= u) ++d;
    out[u] = static_cast<uint8_t>(d);
  }
}

// Per-owner counts as u64 into a device array (no host round trip).
__global__ void x_counts_kernel(const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ off,
                                uint32_t G, uint64_t* __restrict__ out) {
  const uint32_t d = threadIdx.x;
  if (d < G) out[d] = cnt ? cnt[d] : off[d + 1] - off[d];
}

// Small path: the rank-sorted multi listings become the head of the sorted list the
// downstream kernels read (the large path's output buffers, unused on this path).
__global__ void x_pick_small_kernel(const uint32_t* __restrict__ n_multi,
                                    const uint32_t* __restrict__ sm_pos,
                                    const uint32_t* __restrict__ sm_list,
                                    uint32_t* __restrict__ spos, uint32_t* __restrict__ slist) {
  const uint32_t nm = *n_multi;
  if (nm > radix::kSmallN) return;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nm) {
    spos[i] = sm_pos[i];
    slist[i] = sm_list[i];
  }
}

struct Offs {
  uint64_t v[kMaxWorld + 1];
};

// Owner side: pair k (received from source r) names entry id_off[r] + pair_pos[k] of
// the ids this rank received (and looked up) in the forward exchange. The pairs become a
// batch of P one-listing samples (offsets = 0..P) in arrival order.
__global__ void x_owner_kernel(const uint64_t* __restrict__ recv_ids,
                               const uint64_t* __restrict__ recv_versions, Offs id_off,
                               Offs pair_off, uint32_t G, const uint32_t* __restrict__ pair_pos,
                               uint64_t P, uint64_t* __restrict__ out_ids,
                               uint64_t* __restrict__ out_rv, uint32_t* __restrict__ out_off,
                               unsigned long long* protocol) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k <= P;
       k += (uint64_t)gridDim.x * blockDim.x) {
    out_off[k] = static_cast<uint32_t>(k);
    if (k == P) break;
    uint32_t r = 0;
    while (r + 1 < G && pair_off.v[r + 1] <= k) ++r;
    uint64_t idx = id_off.v[r] + pair_pos[k];
    if (idx >= id_off.v[r + 1]) {
      atomicOr(protocol, 1ull);  // gates every update kernel; reported by check_flags
      idx = id_off.v[r];
    }
    out_ids[k] = idx < id_off.v[G] ? recv_ids[idx] : 0;
    out_rv[k] = (recv_versions && idx < id_off.v[G]) ? recv_versions[idx] : 0;
  }
}

uint32_t grid_n(uint64_t n, int sms) {
  return static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n, kXBlock), uint64_t(sms) * 8)));
}

// Grows with 25% slack so per-step size jitter does not reallocate (and synchronise).
template <typename T>
void grow(T*& p, uint64_t& cap, uint64_t want) {
  if (want <= cap && p) return;
  want = want + want / 4 + 1024;
  if (p) HPS_CUDA(cudaFree(p));
  p = nullptr;
  HPS_CUDA(cudaMalloc(&p, std::max<uint64_t>(want, 1) * sizeof(T)));
  cap = want;
}

}  // namespace

XBatch::~XBatch() {
  DeviceGuard g(device);
  void* ps[] = {hkeys,  hidx,   hval,   hmul,    dest,    sendpos, spair, offsets, lgrp,
                keys_a, vals_a, keys_b, vals_b,  scratch, head,    ex,    tsum,    cnt,
                seg,    dest_of_pos,    pair_off, mkeys,  mstart,  sm_pos, sm_list};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (h_buf) cudaFreeHost(h_buf);
}

void xbatch_init(XBatch& x) {
  DeviceGuard g(x.device);
  HPS_CUDA(cudaMalloc(&x.cnt, kCntWords * sizeof(uint32_t)));
  HPS_CUDA(cudaMalloc(&x.seg, 33 * sizeof(uint32_t)));
  HPS_CUDA(cudaMalloc(&x.pair_off, 33 * sizeof(uint64_t)));
  HPS_CUDA(cudaMalloc(&x.mstart, 33 * sizeof(uint32_t)));
  HPS_CUDA(cudaMalloc(&x.mkeys, radix::kSmallN * sizeof(unsigned long long)));
  HPS_CUDA(cudaMalloc(&x.sm_pos, radix::kSmallN * sizeof(uint32_t)));
  HPS_CUDA(cudaMalloc(&x.sm_list, radix::kSmallN * sizeof(uint32_t)));
  HPS_CUDA(cudaMallocHost(&x.h_buf, 128 * sizeof(uint64_t)));
  int dev = 0;
  HPS_CUDA(cudaGetDevice(&dev));
  HPS_CUDA(cudaDeviceGetAttribute(&x.sms, cudaDevAttrMultiProcessorCount, dev));
}

static void require_device(const void* p, const char* what) {
  if (p && !is_device_ptr(p))
    throw Error(HPS_E_PRECONDITION, std::string(what) + ": device pointer required");
}

void xbatch_route(XBatch& x, const uint64_t* ids, uint64_t n, const uint32_t* offsets, uint32_t B,
                  uint32_t F, uint64_t* out_send_ids, uint64_t* out_counts, cudaStream_t st) {
  require_device(ids, "hps_exchange_route ids");
  require_device(offsets, "hps_exchange_route offsets");
  require_device(out_send_ids, "hps_exchange_route send_ids");
  if (n >= (1ull << 31)) throw Error(HPS_E_PRECONDITION, "hps_exchange_route: too many ids");
  const uint64_t BF = static_cast<uint64_t>(B) * F;
  x.N = n;
  x.B = B;
  x.F = F;
  x.lbits = bits_for(n ? n - 1 : 0);
  uint64_t H = 1024;
  int lg = 10;
  while (H < 2 * n) H <<= 1, ++lg;
  grow(x.hkeys, x.cap_H, H + 1);
  grow(x.hidx, x.cap_hidx, n);
  grow(x.hval, x.cap_hval, H + 1);
  grow(x.hmul, x.cap_hmul, H + 1);
  grow(x.dest, x.cap_dest, n);
  grow(x.sendpos, x.cap_sendpos, n);
  grow(x.spair, x.cap_spair, n);
  grow(x.lgrp, x.cap_lgrp, n);
  grow(x.offsets, x.cap_off, BF + 1);
  HPS_CUDA(cudaMemcpyAsync(x.offsets, offsets, (BF + 1) * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, st));
  HPS_CUDA(cudaMemsetAsync(x.cnt, 0, kCntWords * sizeof(uint32_t), st));
  if (n) {
    HPS_CUDA(cudaMemsetAsync(x.hkeys, 0xff, H * sizeof(uint64_t), st));
    HPS_CUDA(cudaMemsetAsync(x.hmul, 0, H + 1, st));
    x_insert_kernel<<<grid_n(n, x.sms), kXBlock, 0, st>>>(ids, n, x.hkeys, H - 1, 64 - lg,
                                                          x.cnt + kCntSpecial, x.hidx, x.hmul);
    x_number_kernel<<<grid_n(n, x.sms), kXBlock, 0, st>>>(ids, n, x.S, x.G, x.hidx, x.hmul,
                                                          x.hval, x.dest, x.spair, x.cnt);
    HPS_LAUNCH_CHECK_N(2);
  }
  x_scatter_kernel<<<grid_n(std::max<uint64_t>(n, 1), x.sms), kXBlock, 0, st>>>(
      ids, n, x.G, x.hidx, x.hval, x.dest, x.spair, x.cnt, x.lbits, x.sendpos, out_send_ids,
      x.seg, x.mkeys);
  HPS_LAUNCH_CHECK();
  launch_expand_groups(x.offsets, static_cast<uint32_t>(BF), x.lgrp, st);
  if (is_device_ptr(out_counts)) {  // stays on the device: no host round trip
    x_counts_kernel<<<1, 32, 0, st>>>(x.cnt, nullptr, x.G, out_counts);
    HPS_LAUNCH_CHECK();
    return;
  }
  uint32_t* h = reinterpret_cast<uint32_t*>(x.h_buf);
  HPS_CUDA(cudaMemcpyAsync(h, x.cnt, x.G * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
  for (uint32_t d = 0; d < x.G; ++d) out_counts[d] = h[d];
}

void xbatch_pool(XBatch& x, const float* rows, uint32_t D, float* out_pooled, cudaStream_t st) {
  require_device(rows, "hps_exchange_pool rows");
  require_device(out_pooled, "hps_exchange_pool out");
  if (!D) throw Error(HPS_E_PRECONDITION, "hps_exchange_pool: dim must be positive");
  DevTable view{};
  view.rows = const_cast<float*>(rows);
  view.D = D;
  view.stride = D;
  view.capacity = static_cast<uint32_t>(x.N);  // U <= N (U itself may be device-side)
  const uint64_t BF = static_cast<uint64_t>(x.B) * x.F;
  launch_pool(view, x.offsets, x.sendpos, static_cast<uint32_t>(BF), x.N,
              x.agg == HPS_MEAN ? 1 : 0, out_pooled, nullptr, nullptr, st);
}

// Pairs = one per (sample, distinct id). Ids listed once in the batch (one-hot: nearly
// all) are their own pair and stream through x_single_emit_kernel; the listings of ids
// listed more than once are ordered by (send position, listing) -- a rank sort of their
// composite keys when they are few, else (device-gated) a radix sort of every listing --
// and reduced per (id, sample) run by x_multi_emit_kernel.
void xbatch_pairs(XBatch& x, const float* grads, uint32_t D, uint32_t* out_pair_pos,
                  float* out_contrib, uint64_t* out_pair_counts, cudaStream_t st) {
  require_device(grads, "hps_exchange_pairs grads");
  require_device(out_pair_pos, "hps_exchange_pairs pair_pos");
  require_device(out_contrib, "hps_exchange_pairs contrib");
  if (!D) throw Error(HPS_E_PRECONDITION, "hps_exchange_pairs: dim must be positive");
  const uint64_t n = x.N;
  if (n == 0) {
    if (is_device_ptr(out_pair_counts)) {
      HPS_CUDA(cudaMemsetAsync(out_pair_counts, 0, x.G * sizeof(uint64_t), st));
    } else {
      for (uint32_t d = 0; d < x.G; ++d) out_pair_counts[d] = 0;
    }
    return;
  }
  grow(x.keys_a, x.cap_ka, n);
  grow(x.vals_a, x.cap_va, n);
  grow(x.keys_b, x.cap_kb, n);
  grow(x.vals_b, x.cap_vb, n);
  grow(x.scratch, x.cap_scratch, radix::scratch_words<uint32_t>(n));
  grow(x.head, x.cap_head, n);
  grow(x.ex, x.cap_ex, n);
  grow(x.tsum, x.cap_tsum, ceil_div(n, 4096) + 2);
  grow(x.dest_of_pos, x.cap_dop, n);
  const uint32_t* n_multi = x.cnt + kCntMulti;
  // small path: rank sort of the multi listings' composite keys (no-op when large)
  radix::sort_composite_small(x.mkeys, n_multi, x.lbits, x.sm_pos, x.sm_list, st);
  // large path: stable radix sort of every listing by send position (no-op when small)
  const bool in_b = radix::sort_pairs<uint32_t>(x.keys_a, x.vals_a, x.keys_b, x.vals_b, n,
                                                x.lbits, x.scratch, st, x.sms, n_multi,
                                                x.sendpos, true);
  // Both paths write the same buffers downstream; the kernels pick by the device count.
  // The small path's results are copied over the large path's output buffers' heads.
  uint32_t* spos = in_b ? x.keys_b : x.keys_a;
  uint32_t* slist = in_b ? x.vals_b : x.vals_a;
  x_pick_small_kernel<<<ceil_div(radix::kSmallN, kXBlock), kXBlock, 0, st>>>(
      n_multi, x.sm_pos, x.sm_list, spos, slist);
  const uint64_t nh = n;  // host bound of the live list
  x_pair_flags_kernel<<<grid_n(nh, x.sms), kXBlock, 0, st>>>(spos, slist, x.lgrp, x.spair, x.F,
                                                             nh, n_multi, x.head);
  exclusive_scan(x.head, x.ex, nh, x.tsum, x.tsum + ceil_div(nh, 4096), st);
  x_dest_of_pos_kernel<<<grid_n(n, x.sms), kXBlock, 0, st>>>(x.seg, x.G, n, x.dest_of_pos);
  x_pair_bounds_kernel<<<1, 64, 0, st>>>(spos, x.ex, x.head, nh, x.cnt, x.seg, x.G, x.pair_off,
                                         x.mstart);
  HPS_LAUNCH_CHECK_N(4);
  const int mean = x.agg == HPS_MEAN ? 1 : 0;
  HPS_DISPATCH_DIM(D, {
    const uint32_t blocks = static_cast<uint32_t>(std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div(n, kXBlock / L), uint64_t(x.sms) * 16)));
    x_single_emit_kernel<V, L, G><<<blocks, kXBlock, 0, st>>>(
        x.spair, x.dest, x.sendpos, x.lgrp, x.offsets, n, D, mean, grads, x.seg, x.pair_off,
        out_pair_pos, out_contrib);
    x_multi_emit_kernel<V, L, G><<<blocks, kXBlock, 0, st>>>(
        spos, slist, x.head, x.ex, x.lgrp, x.offsets, x.F, nh, x.cnt, D, mean, grads,
        x.dest_of_pos, x.seg, x.pair_off, x.mstart, out_pair_pos, out_contrib);
  });
  HPS_LAUNCH_CHECK_N(2);
  if (is_device_ptr(out_pair_counts)) {
    x_counts_kernel<<<1, 32, 0, st>>>(nullptr, x.pair_off, x.G, out_pair_counts);
    HPS_LAUNCH_CHECK();
    return;
  }
  HPS_CUDA(cudaMemcpyAsync(x.h_buf, x.pair_off, (x.G + 1) * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
  for (uint32_t d = 0; d < x.G; ++d) out_pair_counts[d] = x.h_buf[d + 1] - x.h_buf[d];
}

void table_apply_pairs(Table* t, const uint64_t* recv_ids, const uint64_t* recv_versions,
                       const uint64_t* id_counts, const uint32_t* pair_pos, const float* contrib,
                       const uint64_t* pair_counts, uint32_t G, float lr, uint32_t step_tag,
                       uint32_t epoch, int* accepted, uint32_t flags, cudaStream_t st) {
  require_device(recv_ids, "hps_table_apply_pairs recv_ids");
  require_device(recv_versions, "hps_table_apply_pairs recv_versions");
  require_device(pair_pos, "hps_table_apply_pairs pair_pos");
  require_device(contrib, "hps_table_apply_pairs contrib");
  if (G == 0 || G > kMaxWorld) throw Error(HPS_E_PRECONDITION, "apply_pairs: bad world size");
  Offs io{}, po{};
  for (uint32_t r = 0; r < G; ++r) {
    io.v[r + 1] = io.v[r] + id_counts[r];
    po.v[r + 1] = po.v[r] + pair_counts[r];
  }
  const uint64_t P = po.v[G];
  if (P >= 0xffffffffull) throw Error(HPS_E_PRECONDITION, "apply_pairs: too many pairs");
  XScratch& xs = t->xs;
  grow(xs.ids, xs.cap_ids, P);
  grow(xs.rv, xs.cap_rv, P);
  grow(xs.off, xs.cap_off, P + 1);
  x_owner_kernel<<<grid_n(P + 1, t->sm_count), kXBlock, 0, st>>>(
      recv_ids, recv_versions, io, po, G, pair_pos, P, xs.ids, xs.rv, xs.off,
      t->d.ctr + kCtrProtocol);
  HPS_LAUNCH_CHECK();
  // The pairs as a batch of P one-listing samples, sum aggregation: each contribution is
  // applied as is (the source's fan-out already produced (float)(0.0 + sum), never -0.0),
  // per row in arrival order = (source rank, sample) order, through the batch plan
  // (rows hit once skip the ordering sort).
  Batch& b = t->scratch;
  b.agg = HPS_SUM;
  batch_register(b, xs.ids, P, xs.off, static_cast<uint32_t>(P), 1, nullptr, st);
  batch_push(b, HPS_SUM, contrib, lr, step_tag, epoch, recv_versions ? 0 : 1,
             recv_versions ? xs.rv : nullptr, accepted, flags, st);
}

}  // namespace hps
