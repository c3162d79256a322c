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
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>

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
// [33] listings of multi-listed ids, [34] groups left for the requester's own pooling
// (glist), [64,96) ids listed once per owner (= single pairs), [96,128) multi-listed ids
// per owner. Within an owner's segment the ids listed once come first, numbered like
// their pairs, so a single pair's position needs no word of its own on the peer path.
constexpr int kCntSpecial = 32, kCntMulti = 33, kCntGlist = 34, kCntSingle = 64,
              kCntMultiIds = 96, kCntWords = 128;
// hval of an id listed more than once: its index among its owner's multi-listed ids
constexpr uint32_t kMultiIdx = 0x80000000u;

// Distinct ids: a transient open-addressing set (keys only). The entry index of each
// listing's id is recorded; the thread whose CAS claimed the entry is its inserter and
// every other listing of the id marks the entry "multi". Entry H is the side entry of
// id ~0 (the empty marker).
__global__ void __launch_bounds__(kXBlock)
    x_insert_kernel(const uint64_t* __restrict__ ids, uint64_t n, uint64_t* hkeys,
                    uint64_t mask, int shift, uint32_t* special, uint32_t* __restrict__ hidx,
                    uint8_t* __restrict__ hmul) {
  pdl_entry();
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
  pdl_entry();
  __shared__ uint32_t bc[32], mc[32], mb[32], sc[32], sb[32];
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < G) bc[threadIdx.x] = 0, sc[threadIdx.x] = 0, mc[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t i = base + threadIdx.x;
    uint32_t d = 0, q = 0, code = 0;
    bool single = false;
    const bool valid = i < n;
    if (valid) {
      code = hidx[i];
      d = route_shard(ids[i], S) % G;
      dest[i] = static_cast<uint8_t>(d);
      if (code & kInserter) {
        atomicAdd(&bc[d], 1u);
        single = hmul[code & ~kInserter] == 0;
        q = single ? atomicAdd(&sc[d], 1u) : atomicAdd(&mc[d], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x < G) {
      if (bc[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], bc[threadIdx.x]);
      sb[threadIdx.x] =
          sc[threadIdx.x] ? atomicAdd(&cnt[kCntSingle + threadIdx.x], sc[threadIdx.x]) : 0;
      mb[threadIdx.x] =
          mc[threadIdx.x] ? atomicAdd(&cnt[kCntMultiIds + threadIdx.x], mc[threadIdx.x]) : 0;
    }
    __syncthreads();
    if (valid) {
      // ids listed once: index = their pair index; multi-listed: placed after all of
      // the owner's ids listed once (x_scatter resolves kMultiIdx)
      if (code & kInserter)
        hval[code & ~kInserter] = single ? sb[d] + q : (kMultiIdx | (mb[d] + q));
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

// Id regions of the owners (peer path): p[d] = owner d's region for this source rank.
struct PeerIds {
  uint64_t* p[kMaxWorld];
  uint32_t* tg[kMaxWorld];  // (direct pooling) per id: the requester's group to write, or ~0
};

// Send position per listing, send_ids, and the composite keys (pos << lbits | listing)
// of listings whose id is listed more than once (while they fit the small sort).
__global__ void __launch_bounds__(kXBlock)
    x_scatter_kernel(const uint64_t* __restrict__ ids, uint64_t n, uint32_t G,
                     const uint32_t* __restrict__ hidx, const uint32_t* __restrict__ hval,
                     const uint8_t* __restrict__ dest, const uint32_t* __restrict__ spair,
                     uint32_t* cnt, int lbits, uint32_t* __restrict__ sendpos,
                     uint64_t* __restrict__ send_ids, uint32_t* __restrict__ seg_out,
                     unsigned long long* __restrict__ mkeys, PeerIds pid,
                     const uint32_t* __restrict__ lgrp, const uint32_t* __restrict__ offsets,
                     uint8_t* __restrict__ gdirect) {
  pdl_entry();
  __shared__ uint32_t seg[33], s_single[32];
  __shared__ uint32_t s_n, s_base;
  load_seg(cnt, G, seg);
  if (threadIdx.x < G) s_single[threadIdx.x] = cnt[kCntSingle + threadIdx.x];
  __syncthreads();
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
      const uint32_t d = dest[i], hv = hval[code & ~kInserter];
      const uint32_t j = (hv & kMultiIdx) ? s_single[d] + (hv & ~kMultiIdx) : hv;
      pos = seg[d] + j;
      sendpos[i] = pos;
      if (code & kInserter) {
        if (send_ids) {
          send_ids[pos] = ids[i];
        } else {
          pid.p[d][j] = ids[i];  // straight into owner d's id region for this rank
          if (gdirect) {
            // an id listed once, alone in its group: its pooled value is the row itself,
            // which the owner writes straight into this rank's pooled output
            const uint32_t lg = lgrp[i];
            const bool direct = spair[i] != kNoPair && offsets[lg + 1] - offsets[lg] == 1;
            pid.tg[d][j] = direct ? lg : 0xffffffffu;
            if (direct) gdirect[lg] = 1;
          }
        }
      }
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

// Groups the owners did not pool (gdirect == 0: empty groups, several listings, or an id
// listed more than once) -> glist, warp-aggregated appends; the requester pools only those.
__global__ void x_glist_kernel(const uint8_t* __restrict__ gdirect, uint64_t BF,
                               uint32_t* __restrict__ glist, uint32_t* cnt) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < BF;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = base + threadIdx.x;
    const bool want = g < BF && !gdirect[g];
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) continue;
    uint32_t b = 0;
    if (lane == __ffs(m) - 1) b = atomicAdd(&cnt[kCntGlist], __popc(m));
    b = __shfl_sync(0xffffffffu, b, __ffs(m) - 1);
    if (want) glist[b + __popc(m & ((1u << lane) - 1))] = static_cast<uint32_t>(g);
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
  pdl_entry();
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
  pdl_entry();
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

// Where owner d's pairs go: contribution rows c[d][k * D ...] and positions p[d][k] for
// k = base[d] + index -- one local buffer for all owners (NCCL path) or each owner's
// peer-mapped receive arena (NVLink path).
struct PairOut {
  float* c[kMaxWorld];
  uint32_t* p[kMaxWorld];
  // peer path: owner d's XHdr::bad word for this source, and the barrier epoch of this
  // emit (the validation PsShard::apply_gradients does before mutating, :146-153, done
  // here while the contributions are formed; the owner reads the words after the barrier)
  uint32_t* bad[kMaxWorld];
  const unsigned long long* epoch;
  // write single pairs' positions (NCCL path); the peer path's owners derive them (a
  // single pair's index is its id's index in the owner segment)
  int single_pos;
  // value codec (kappa > 0, peer path): each contribution row travels as a kappa-scaled
  // binary16 payload at (uint16_t*)c[d] + k * D and its f32 scale at c[d][scale_off + k]
  float kappa;
  uint64_t scale_off;
};

// compress_values (codec.hpp:222-244) of one row held by an L-lane group (V floats per
// lane): scale = kappa / max|v| (1 for an all-zero row), payload = binary16(v * scale)
// rounded to nearest (float_to_half_bits); the group's lane 0 writes the scale.
template <int V, int L>
__device__ __forceinline__ void put_coded(float* base, uint64_t rec, uint64_t scale_off,
                                          uint32_t D, uint32_t d0, const float (&o)[V],
                                          float kappa) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(L - 1u)));
  float m = 0.0f;
#pragma unroll
  for (int v = 0; v < V; ++v) m = fmaxf(m, fabsf(o[v]));
#pragma unroll
  for (int off = L / 2; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(mask, m, off, L));
  const float scale = m == 0.0f ? 1.0f : __fdiv_rn(kappa, m);
  uint16_t h[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const float x = m == 0.0f ? 0.0f : __fmul_rn(o[v], scale);
    h[v] = __half_as_ushort(__float2half_rn(x));
  }
  uint16_t* dst = reinterpret_cast<uint16_t*>(base) + rec * D + d0;
  if constexpr (V == 4) {
    uint2 w;
    w.x = h[0] | (static_cast<uint32_t>(h[1]) << 16);
    w.y = h[2] | (static_cast<uint32_t>(h[3]) << 16);
    *reinterpret_cast<uint2*>(dst) = w;
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) dst[v] = h[v];
  }
  if ((lane & (L - 1u)) == 0) base[scale_off + rec] = scale;
}

template <int V>
__device__ __forceinline__ void flag_nonfinite(const PairOut& po, uint32_t d, const float (&o)[V]) {
  if (!po.epoch) return;
  bool bad = false;
#pragma unroll
  for (int v = 0; v < V; ++v) bad |= !isfinite(o[v]);
  if (bad) *reinterpret_cast<volatile uint32_t*>(po.bad[d]) = static_cast<uint32_t>(*po.epoch);
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
                         const uint64_t* __restrict__ base, PairOut po) {
  pdl_entry();
  const uint32_t lane = threadIdx.x % L;
  const uint64_t groups = (uint64_t)gridDim.x * (kXBlock / L);
  if constexpr (!GEN) {
    // kEmitILP pairs in flight per lane group (metadata loads, gradient loads, then the
    // mostly remote stores), as in the owner gather
    constexpr int kEmitILP = 4;
    for (uint64_t i0 = blockIdx.x * (uint64_t)(kXBlock / L) + threadIdx.x / L; i0 < n;
         i0 += groups * kEmitILP) {
      uint32_t sp[kEmitILP], dd[kEmitILP], gg[kEmitILP], cntg[kEmitILP];
#pragma unroll
      for (int u = 0; u < kEmitILP; ++u) {
        const uint64_t i = i0 + u * groups;
        sp[u] = i < n ? spair[i] : kNoPair;
        dd[u] = sp[u] != kNoPair ? dest[i] : 0u;
        gg[u] = sp[u] != kNoPair ? lgrp[i] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kEmitILP; ++u)
        cntg[u] = (sp[u] != kNoPair && mean) ? offsets[gg[u] + 1] - offsets[gg[u]] : 1u;
      for (uint32_t d0 = lane * V; d0 < D; d0 += L * V) {
        float x[kEmitILP][V];
#pragma unroll
        for (int u = 0; u < kEmitILP; ++u) {
          if (sp[u] != kNoPair) load_vec<V>(grads + static_cast<uint64_t>(gg[u]) * D + d0, x[u]);
        }
#pragma unroll
        for (int u = 0; u < kEmitILP; ++u) {
          if (sp[u] == kNoPair) continue;
          const uint32_t d = dd[u];
          const uint64_t out = base[d] + sp[u];
          if (po.single_pos && lane == 0 && d0 == lane * V)
            po.p[d][out] = sendpos[i0 + u * groups] - seg[d];
          const double scale = mean ? 1.0 / static_cast<double>(cntg[u]) : 1.0;
          float o[V];
#pragma unroll
          for (int v = 0; v < V; ++v)
            o[v] = __double2float_rn(__dadd_rn(0.0, __dmul_rn(static_cast<double>(x[u][v]), scale)));
          if (po.kappa > 0.0f) put_coded<V, L>(po.c[d], out, po.scale_off, D, d0, o, po.kappa);
          else put_row<V, GEN>(po.c[d] + out * D + d0, o);
          flag_nonfinite<V>(po, d, o);
        }
      }
    }
    return;
  }
  for (uint64_t i = blockIdx.x * (uint64_t)(kXBlock / L) + threadIdx.x / L; i < n;
       i += groups) {
    const uint32_t sp = spair[i];
    if (sp == kNoPair) continue;
    const uint32_t d = dest[i];
    const uint64_t out = base[d] + sp;
    const uint32_t g = lgrp[i];
    if (po.single_pos && lane == 0) po.p[d][out] = sendpos[i] - seg[d];
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
      put_row<V, GEN>(po.c[d] + out * D + d0, o);
      flag_nonfinite<V>(po, d, o);
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
                        const uint32_t* __restrict__ seg, const uint64_t* __restrict__ base,
                        const uint32_t* __restrict__ mstart, PairOut po) {
  pdl_entry();
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
    const uint64_t out = base[d] + cnt[kCntSingle + d] + (ex[p] - mstart[d]);
    if (lane == 0) po.p[d][out] = pos - seg[d];
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
      if constexpr (!GEN) {
        if (po.kappa > 0.0f) put_coded<V, L>(po.c[d], out, po.scale_off, D, d0, o, po.kappa);
        else put_row<V, GEN>(po.c[d] + out * D + d0, o);
      } else {
        put_row<V, GEN>(po.c[d] + out * D + d0, o);
      }
      flag_nonfinite<V>(po, d, o);
    }
  }
}

// dest per send position (the owner of send_ids[pos]) from the segment table; U = seg[G]
// is device-side, the grid covers the host bound n >= U.
__global__ void x_dest_of_pos_kernel(const uint32_t* __restrict__ seg, uint32_t G, uint64_t n,
                                     uint8_t* __restrict__ out) {
  pdl_entry();
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
  pdl_entry();
  const uint32_t d = threadIdx.x;
  if (d < G) out[d] = cnt ? cnt[d] : off[d + 1] - off[d];
}

// Small path: the rank-sorted multi listings become the head of the sorted list the
// downstream kernels read (the large path's output buffers, unused on this path).
__global__ void x_pick_small_kernel(const uint32_t* __restrict__ n_multi,
                                    const uint32_t* __restrict__ sm_pos,
                                    const uint32_t* __restrict__ sm_list,
                                    uint32_t* __restrict__ spos, uint32_t* __restrict__ slist) {
  pdl_entry();
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
                               Offs id_end, Offs pair_off, uint32_t G,
                               const uint32_t* __restrict__ pair_pos,
                               uint64_t P, uint64_t* __restrict__ out_ids,
                               uint64_t* __restrict__ out_rv, uint32_t* __restrict__ out_off,
                               unsigned long long* protocol) {
  pdl_entry();
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k <= P;
       k += (uint64_t)gridDim.x * blockDim.x) {
    out_off[k] = static_cast<uint32_t>(k);
    if (k == P) break;
    uint32_t r = 0;
    while (r + 1 < G && pair_off.v[r + 1] <= k) ++r;
    uint64_t idx = id_off.v[r] + pair_pos[k];
    if (idx >= id_end.v[r]) {
      atomicOr(protocol, 1ull);  // gates every update kernel; reported by check_flags
      idx = id_off.v[r];
    }
    out_ids[k] = idx < id_end.v[r] ? recv_ids[idx] : 0;
    out_rv[k] = (recv_versions && idx < id_end.v[r]) ? recv_versions[idx] : 0;
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
  cudaDeviceSynchronize();
  for (uint32_t r = 0; r < G && r < kMaxWorld; ++r)
    if (peer[r] && peer[r] != arena) cudaIpcCloseMemHandle(peer[r]);
  if (arena) cudaFree(arena);
  if (gdirect) cudaFree(gdirect);
  if (glist) cudaFree(glist);
  if (pnew) cudaFree(pnew);
  if (dec_contrib) cudaFree(dec_contrib);
  if (side) cudaStreamDestroy(side);
  if (aux) cudaStreamDestroy(aux);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (xbase) cudaFree(xbase);
  if (dev_epoch) cudaFree(dev_epoch);
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

// ---- shared cores of the two transports ---------------------------------------------------

// Distinct ids grouped by owner: send positions, segment table, and the ids themselves
// either into send_ids (NCCL path) or straight into each owner's id region (peer path).
static void route_core(XBatch& x, const uint64_t* ids, uint64_t n, const uint32_t* offsets,
                       uint32_t B, uint32_t F, uint64_t* send_ids, const PeerIds& pid,
                       cudaStream_t st) {
  require_device(ids, "exchange ids");
  require_device(offsets, "exchange offsets");
  if (n >= (1ull << 31)) throw Error(HPS_E_PRECONDITION, "exchange: too many ids");
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
    launch(x_insert_kernel, grid_n(n, x.sms), kXBlock, 0, st, ids, n, x.hkeys, H - 1, 64 - lg,
                                                          x.cnt + kCntSpecial, x.hidx, x.hmul);
    launch(x_number_kernel, grid_n(n, x.sms), kXBlock, 0, st, ids, n, x.S, x.G, x.hidx, x.hmul,
                                                          x.hval, x.dest, x.spair, x.cnt);
    HPS_LAUNCH_CHECK_N(2);
  }
  launch_expand_groups(x.offsets, static_cast<uint32_t>(BF), x.lgrp, st);
  uint8_t* gdirect = nullptr;
  if (!send_ids && x.direct_ok) {
    gdirect = x.gdirect;
    HPS_CUDA(cudaMemsetAsync(gdirect, 0, BF, st));
  }
  launch(x_scatter_kernel, grid_n(std::max<uint64_t>(n, 1), x.sms), kXBlock, 0, st, 
      ids, n, x.G, x.hidx, x.hval, x.dest, x.spair, x.cnt, x.lbits, x.sendpos, send_ids, x.seg,
      x.mkeys, pid, x.lgrp, x.offsets, gdirect);
  HPS_LAUNCH_CHECK();
  if (gdirect) {
    launch(x_glist_kernel, grid_n(std::max<uint64_t>(BF, 1), x.sms), kXBlock, 0, st, gdirect, BF,
           x.glist, x.cnt);
    HPS_LAUNCH_CHECK();
  }
}

// Pair ordering and counts up to (not including) the emit kernels: x.pair_off = owners'
// pair offsets in a concatenated layout. Returns the sorted list (spos, slist).
static void pairs_core(XBatch& x, const uint32_t** spos_out, const uint32_t** slist_out,
                       cudaStream_t st) {
  const uint64_t n = x.N;
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
  // large path: stable radix sort of every listing by send position, only when the
  // device count says so (its kernels exit at once otherwise)
  const bool in_b = ((x.lbits + radix::kBits - 1) / radix::kBits) & 1;
  radix::sort_scratch_zero(x.scratch, st);
  radix::sort_pairs<uint32_t>(x.keys_a, x.vals_a, x.keys_b, x.vals_b, n, x.lbits, x.scratch, st,
                              x.sms, n_multi, x.sendpos, true, false);
  uint32_t* spos = in_b ? x.keys_b : x.keys_a;
  uint32_t* slist = in_b ? x.vals_b : x.vals_a;
  launch(x_pick_small_kernel, ceil_div(radix::kSmallN, kXBlock), kXBlock, 0, st, 
      n_multi, x.sm_pos, x.sm_list, spos, slist);
  launch(x_pair_flags_kernel, grid_n(n, x.sms), kXBlock, 0, st, spos, slist, x.lgrp, x.spair, x.F,
                                                            n, n_multi, x.head);
  exclusive_scan(x.head, x.ex, n, x.tsum, x.tsum + ceil_div(n, 4096), st);
  launch(x_dest_of_pos_kernel, grid_n(n, x.sms), kXBlock, 0, st, x.seg, x.G, n, x.dest_of_pos);
  launch(x_pair_bounds_kernel, 1, 64, 0, st, spos, x.ex, x.head, n, x.cnt, x.seg, x.G, x.pair_off,
                                         x.mstart);
  HPS_LAUNCH_CHECK_N(4);
  *spos_out = spos;
  *slist_out = slist;
}

static void emit_pairs(XBatch& x, const float* grads, uint32_t D, const uint32_t* spos,
                       const uint32_t* slist, const uint64_t* base, const PairOut& po,
                       cudaStream_t st) {
  const uint64_t n = x.N;
  const int mean = x.agg == HPS_MEAN ? 1 : 0;
  HPS_DISPATCH_DIM(D, {
    const uint32_t blocks = static_cast<uint32_t>(std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div(n, kXBlock / L), uint64_t(x.sms) * 16)));
    launch(x_single_emit_kernel<V, L, G>, blocks, kXBlock, 0, st, 
        x.spair, x.dest, x.sendpos, x.lgrp, x.offsets, n, D, mean, grads, x.seg, base, po);
    launch(x_multi_emit_kernel<V, L, G>, blocks, kXBlock, 0, st, 
        spos, slist, x.head, x.ex, x.lgrp, x.offsets, x.F, n, x.cnt, D, mean, grads,
        x.dest_of_pos, x.seg, base, x.mstart, po);
  });
  HPS_LAUNCH_CHECK_N(2);
}

// ---- NCCL transport (the caller moves the buffers) -------------------------------------

void xbatch_route(XBatch& x, const uint64_t* ids, uint64_t n, const uint32_t* offsets, uint32_t B,
                  uint32_t F, uint64_t* out_send_ids, uint64_t* out_counts, cudaStream_t st) {
  require_device(out_send_ids, "hps_exchange_route send_ids");
  if (n && !out_send_ids) throw Error(HPS_E_PRECONDITION, "hps_exchange_route: null send_ids");
  route_core(x, ids, n, offsets, B, F, out_send_ids, PeerIds{}, st);
  if (is_device_ptr(out_counts)) {  // stays on the device: no host round trip
    launch(x_counts_kernel, 1, 32, 0, st, x.cnt, nullptr, x.G, out_counts);
    HPS_LAUNCH_CHECK();
    return;
  }
  uint32_t* h = reinterpret_cast<uint32_t*>(x.h_buf);
  HPS_CUDA(cudaMemcpyAsync(h, x.cnt, x.G * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
  for (uint32_t d = 0; d < x.G; ++d) out_counts[d] = h[d];
}

// decompress_values (codec.hpp:246-261) of n compressed rows (payload (uint16_t*)rec +
// k * D, scale rec[scale_off + k]): out = (float)half / scale, one rounded division. n is
// *n_dev when given (device-side counts), else n_host.
// decompress_values (codec.hpp:246-261): v = (float)h / scale, one rounded divide per
// element. D is a power of two >= 4 (xbatch_arena checks it): four elements per thread,
// an 8-byte load and a 16-byte store, the record index by shift.
__global__ void x_decode_kernel(const float* __restrict__ rec, uint64_t scale_off, uint32_t log2d,
                                uint64_t n_host, const uint32_t* __restrict__ n_dev,
                                float* __restrict__ out) {
  pdl_entry();
  const uint64_t n = n_dev ? min(n_host, static_cast<uint64_t>(*n_dev)) : n_host;
  const uint2* __restrict__ pay = reinterpret_cast<const uint2*>(rec);
  const uint64_t quads = (n << log2d) >> 2;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < quads;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const float s = __ldg(rec + scale_off + ((e << 2) >> log2d));
    const uint2 w = __ldcs(pay + e);
    float4 v;
    v.x = __fdiv_rn(__half2float(__ushort_as_half(static_cast<unsigned short>(w.x & 0xffffu))), s);
    v.y = __fdiv_rn(__half2float(__ushort_as_half(static_cast<unsigned short>(w.x >> 16))), s);
    v.z = __fdiv_rn(__half2float(__ushort_as_half(static_cast<unsigned short>(w.y & 0xffffu))), s);
    v.w = __fdiv_rn(__half2float(__ushort_as_half(static_cast<unsigned short>(w.y >> 16))), s);
    reinterpret_cast<float4*>(out)[e] = v;
  }
}

static void decode(const float* rec, uint64_t scale_off, uint32_t D, uint64_t n_host,
                   const uint32_t* n_dev, float* out, int sms, cudaStream_t st) {
  if (!n_host) return;
  uint32_t log2d = 0;
  while ((1u << log2d) < D) ++log2d;
  launch(x_decode_kernel,
         std::max<uint64_t>(1, std::min<uint64_t>(ceil_div((n_host * D) / 4, 256), uint64_t(sms) * 8)),
         256, 0, st, rec, scale_off, log2d, n_host, n_dev, out);
  HPS_LAUNCH_CHECK();
}

// serve_pull over compressed rows (codec mode): the requester pools straight from the
// delivered binary16 records -- each element decoded as decompress_values does it
// (one rounded divide by the record's scale, codec.hpp:246-261), then pooled exactly as
// pool_kernel pools (fp64 sum in listing order, (float)(acc * scale), empty -> 0) --
// without materialising the decoded rows. L = D / 4 lanes per group, 4 dims per lane.
template <int L>
__global__ void __launch_bounds__(256)
    x_pool_coded_kernel(const float* __restrict__ rec, uint64_t scale_off,
                        const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ sendpos,
                        uint64_t BF, int mean, float* __restrict__ out) {
  pdl_entry();
  constexpr uint32_t D = 4 * L;
  const uint2* __restrict__ pay = reinterpret_cast<const uint2*>(rec);
  const uint32_t ln = threadIdx.x % L;
  const uint64_t groups = static_cast<uint64_t>(gridDim.x) * blockDim.x / L;
  for (uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L; g < BF;
       g += groups) {
    const uint32_t a = offsets[g], e = offsets[g + 1];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t l = a; l < e; ++l) {
      const uint32_t r = sendpos[l];
      const float sc = __ldg(rec + scale_off + r);
      const uint2 w = pay[static_cast<uint64_t>(r) * L + ln];
      const uint32_t hs[4] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = __fdiv_rn(__half2float(__ushort_as_half(static_cast<unsigned short>(hs[k]))), sc);
        acc[k] = __dadd_rn(acc[k], static_cast<double>(x));
      }
    }
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e > a) {
      const double scale = mean ? __drcp_rn(static_cast<double>(e - a)) : 1.0;
      v.x = __double2float_rn(__dmul_rn(acc[0], scale));
      v.y = __double2float_rn(__dmul_rn(acc[1], scale));
      v.z = __double2float_rn(__dmul_rn(acc[2], scale));
      v.w = __double2float_rn(__dmul_rn(acc[3], scale));
    }
    reinterpret_cast<float4*>(out + g * D)[ln] = v;
  }
}

void xbatch_pool(XBatch& x, const float* rows, uint32_t D, float* out_pooled, cudaStream_t st) {
  const bool peer = !rows;
  if (peer) {  // peer path: the owners delivered into the arena
    rows = x.arena_rows;
    if (!x.connected) throw Error(HPS_E_PRECONDITION, "hps_exchange_pool: no rows");
    // pool into the arena's pooled buffer (where the owners wrote the one-listing groups),
    // then hand it over (zero-copy when the caller asks for the arena buffer itself)
    const uint64_t BF = static_cast<uint64_t>(x.B) * x.F;
    float* arena_pooled = reinterpret_cast<float*>(x.arena + x.off_pooled);
    if (x.kappa > 0.0f) {  // the delivered rows are compressed: pool them as they are
      float* dst = out_pooled ? out_pooled : arena_pooled;
      require_device(dst, "hps_exchange_pool out");
      const uint64_t blocks = std::max<uint64_t>(
          1, std::min<uint64_t>(ceil_div(BF * (D / 4), 256), uint64_t(x.sms) * 8));
      switch (D) {
        case 4: launch(x_pool_coded_kernel<1>, blocks, 256, 0, st, x.arena_rows, x.max_ids * D / 2, x.offsets, x.sendpos, BF, x.agg == HPS_MEAN ? 1 : 0, dst); break;
        case 8: launch(x_pool_coded_kernel<2>, blocks, 256, 0, st, x.arena_rows, x.max_ids * D / 2, x.offsets, x.sendpos, BF, x.agg == HPS_MEAN ? 1 : 0, dst); break;
        case 16: launch(x_pool_coded_kernel<4>, blocks, 256, 0, st, x.arena_rows, x.max_ids * D / 2, x.offsets, x.sendpos, BF, x.agg == HPS_MEAN ? 1 : 0, dst); break;
        case 32: launch(x_pool_coded_kernel<8>, blocks, 256, 0, st, x.arena_rows, x.max_ids * D / 2, x.offsets, x.sendpos, BF, x.agg == HPS_MEAN ? 1 : 0, dst); break;
        case 64: launch(x_pool_coded_kernel<16>, blocks, 256, 0, st, x.arena_rows, x.max_ids * D / 2, x.offsets, x.sendpos, BF, x.agg == HPS_MEAN ? 1 : 0, dst); break;
        default: launch(x_pool_coded_kernel<32>, blocks, 256, 0, st, x.arena_rows, x.max_ids * D / 2, x.offsets, x.sendpos, BF, x.agg == HPS_MEAN ? 1 : 0, dst); break;
      }
      HPS_LAUNCH_CHECK();
      return;
    }
    if (x.direct_ok) {
      DevTable view{};
      view.rows = const_cast<float*>(rows);
      view.D = D;
      view.stride = D;
      view.capacity = static_cast<uint32_t>(x.N);
      launch_pool(view, x.offsets, x.sendpos, static_cast<uint32_t>(BF), x.N,
                  x.agg == HPS_MEAN ? 1 : 0, arena_pooled, nullptr, nullptr, st, x.glist,
                  x.cnt + kCntGlist);
      if (out_pooled && out_pooled != arena_pooled) {
        require_device(out_pooled, "hps_exchange_pool out");
        HPS_CUDA(cudaMemcpyAsync(out_pooled, arena_pooled, BF * D * sizeof(float),
                                 cudaMemcpyDeviceToDevice, st));
      }
      return;
    }
    if (!out_pooled) out_pooled = arena_pooled;
  }
  require_device(rows, "hps_exchange_pool rows");
  require_device(out_pooled, "hps_exchange_pool out");
  if (!D) throw Error(HPS_E_PRECONDITION, "hps_exchange_pool: dim must be positive");
  if (x.N && !rows) throw Error(HPS_E_PRECONDITION, "hps_exchange_pool: no rows");
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
  if (x.N == 0) {
    if (is_device_ptr(out_pair_counts)) {
      HPS_CUDA(cudaMemsetAsync(out_pair_counts, 0, x.G * sizeof(uint64_t), st));
    } else {
      for (uint32_t d = 0; d < x.G; ++d) out_pair_counts[d] = 0;
    }
    return;
  }
  const uint32_t *spos, *slist;
  pairs_core(x, &spos, &slist, st);
  PairOut po{};
  po.single_pos = 1;
  for (uint32_t d = 0; d < x.G; ++d) po.c[d] = out_contrib, po.p[d] = out_pair_pos;
  emit_pairs(x, grads, D, spos, slist, x.pair_off, po, st);
  if (is_device_ptr(out_pair_counts)) {
    launch(x_counts_kernel, 1, 32, 0, st, nullptr, x.pair_off, x.G, out_pair_counts);
    HPS_LAUNCH_CHECK();
    return;
  }
  HPS_CUDA(cudaMemcpyAsync(x.h_buf, x.pair_off, (x.G + 1) * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
  for (uint32_t d = 0; d < x.G; ++d) out_pair_counts[d] = x.h_buf[d + 1] - x.h_buf[d];
}

// Owner side, shared by both transports: pairs (source-rank major) -> a batch of P
// one-listing samples applied through the batch plan.
static void owner_apply(Table* t, const uint64_t* recv_ids, const uint64_t* recv_versions,
                        const Offs& io, const Offs& ie, const Offs& po, uint32_t G,
                        const uint32_t* pair_pos, const float* contrib, float lr,
                        uint32_t step_tag, uint32_t epoch, int* accepted, uint32_t flags,
                        cudaStream_t st) {
  const uint64_t P = po.v[G];
  if (P >= 0xffffffffull) throw Error(HPS_E_PRECONDITION, "apply_pairs: too many pairs");
  XScratch& xs = t->xs;
  grow(xs.ids, xs.cap_ids, P);
  grow(xs.rv, xs.cap_rv, P);
  grow(xs.off, xs.cap_off, P + 1);
  launch(x_owner_kernel, grid_n(P + 1, t->sm_count), kXBlock, 0, st, 
      recv_ids, recv_versions, io, ie, po, G, pair_pos, P, xs.ids, xs.rv, xs.off,
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

void table_apply_pairs(Table* t, const uint64_t* recv_ids, const uint64_t* recv_versions,
                       const uint64_t* id_counts, const uint32_t* pair_pos, const float* contrib,
                       const uint64_t* pair_counts, uint32_t G, float lr, uint32_t step_tag,
                       uint32_t epoch, int* accepted, uint32_t flags, cudaStream_t st) {
  require_device(recv_ids, "hps_table_apply_pairs recv_ids");
  require_device(recv_versions, "hps_table_apply_pairs recv_versions");
  require_device(pair_pos, "hps_table_apply_pairs pair_pos");
  require_device(contrib, "hps_table_apply_pairs contrib");
  if (G == 0 || G > kMaxWorld) throw Error(HPS_E_PRECONDITION, "apply_pairs: bad world size");
  Offs io{}, ie{}, po{};
  for (uint32_t r = 0; r < G; ++r) {
    io.v[r + 1] = io.v[r] + id_counts[r];
    ie.v[r] = io.v[r + 1];
    po.v[r + 1] = po.v[r] + pair_counts[r];
  }
  owner_apply(t, recv_ids, recv_versions, io, ie, po, G, pair_pos, contrib, lr, step_tag, epoch,
              accepted, flags, st);
}

// ---- NVLink peer transport -------------------------------------------------------------
// Every rank owns one arena (cudaMalloc, exported by CUDA IPC, opened by every peer):
//   hdr      XHdr: barrier arrivals + per-source counts (written by peers)
//   ids      [W][Nmax] u64   region r: the distinct ids source r asks this rank for
//   rows     [Nmax][D] f32   this rank's rows, in its send order (written by the owners)
//   ppos     [W*Nmax]  u32   pairs this rank owns, source-rank major (written by sources)
//   contrib  [W*Nmax][D] f32
//   oslot    [W][Nmax] u32   owner-local: slot of each received id
//   oids     [W][Nmax] u64   owner-local copy of the id regions (sources may overwrite the
//   ocnt     [W] u32         regions and counts with the next step once this one's last
//                            barrier is passed, while the owner still applies)
//   tgt      [W][Nmax] u32   per received id: the source's one-listing group to write
//                            the row into directly, or ~0 (written by sources)
//   pooled   [max_groups][D] f32  this rank's pooled batch (owners write the one-listing
//                            groups, hps_exchange_pool the rest)
// A step writes every payload once, directly into the consumer's HBM over NVLink; the
// only synchronisation is a device-side barrier through the hdr flags.

struct PeerHdrs {
  XHdr* h[kMaxWorld];
};

// Owner (peer path): the pairs that arrived -- source-rank major, counts bwd_cnt[r] --
// become a batch of device-counted one-listing samples: ids / read versions of the ids
// each pair names, offsets[k] = min(k, P) for k <= cap (samples past P are empty).
__global__ void x_owner_dyn_kernel(const XHdr* __restrict__ hdr,
                                   const uint32_t* __restrict__ ocnt, uint32_t W,
                                   uint64_t stride, const uint64_t* __restrict__ oids,
                                   const uint64_t* __restrict__ orv,
                                   const uint32_t* __restrict__ pair_pos, uint64_t cap,
                                   uint64_t* __restrict__ out_ids, uint64_t* __restrict__ out_rv,
                                   uint32_t* __restrict__ out_off,
                                   unsigned long long* protocol, DevTable t,
                                   const uint32_t* __restrict__ oslot,
                                   uint32_t* __restrict__ out_slot,
                                   const unsigned long long* epoch, uint32_t* cflags) {
  pdl_entry();
  __shared__ uint64_t po[kMaxWorld + 1];
  __shared__ uint32_t ps[kMaxWorld];
  if (epoch && blockIdx.x == 0 && threadIdx.x == 0) {
    // the sources validated the contributions while emitting them (one barrier ago)
    const uint32_t e = static_cast<uint32_t>(*epoch - 1);
    bool bad = false;
    for (uint32_t r = 0; r < W; ++r) bad |= ld_volatile(&hdr->bad[r]) == e;
    // the owner batch's call flags (its register keeps them); a finite contribution
    // applies as is, so no exact check is needed
    cflags[kCflagReject] = bad ? 1u : 0u;
    cflags[kCflagNeedExact] = 0u;
    if (bad) t.ctr[kCtrDivergence] = 1ull;  // sticky until reported
  }
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (uint32_t r = 0; r < W; ++r) {
      po[r] = run;
      run += ld_volatile(&hdr->bwd_cnt[r]);
      ps[r] = ld_volatile(&hdr->bwd_single[r]);
    }
    po[W] = run;
  }
  __syncthreads();
  const uint64_t P = min(po[W], cap);
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k <= cap;
       k += (uint64_t)gridDim.x * blockDim.x) {
    out_off[k] = static_cast<uint32_t>(min(k, P));
    if (k >= P) {
      if (out_slot && k < cap) out_slot[k] = kInvalidSlot;
      continue;
    }
    uint32_t r = 0;
    while (r + 1 < W && po[r + 1] <= k) ++r;
    // a source's first ps[r] pairs are its ids listed once, numbered like those ids
    const uint64_t kk = k - po[r];
    uint32_t j = kk < ps[r] ? static_cast<uint32_t>(kk) : pair_pos[k];
    if (j >= ocnt[r]) {
      atomicOr(protocol, 1ull);
      j = 0;
    }
    out_ids[k] = oids[r * stride + j];
    if (orv) out_rv[k] = orv[r * stride + j];
    if (out_slot) {
      // the forward already found (or created) the row: reuse its slot instead of a
      // second hash probe, and mark the batch-plan bits the probe would have (plan.cu)
      const uint32_t s = oslot[r * stride + j];
      out_slot[k] = s;
      if (slot_ok(t, s)) {
        const uint32_t bit = 1u << (s & 31);
        if (atomicOr(&t.seen[s >> 5], bit) & bit) atomicOr(&t.multi[s >> 5], bit);
      }
    }
  }
}
struct PeerRows {
  float* p[kMaxWorld];
};

constexpr unsigned long long kBarrierTimeoutNs = 4'000'000'000ull;  // 4 s: never hang the GPU

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// All ranks: arrive (release, system scope) at every peer, then wait (acquire) for
// every peer's arrival at this rank. A peer that never arrives trips the timeout, which
// flags the table (updates are gated off) and surfaces as HPS_E_SYNC_FAILURE.
__global__ void x_barrier_kernel(PeerHdrs ph, uint32_t W, uint32_t rank,
                                 unsigned long long* epoch_ctr, unsigned long long* fail) {
  pdl_entry();
  __shared__ unsigned long long s_epoch;
  const uint32_t t = threadIdx.x;
  // The epoch lives on the device, so a barrier captured in a CUDA graph advances it on
  // every replay (every rank runs the same sequence of barriers).
  if (t == 0) s_epoch = ++*epoch_ctr;
  __threadfence_system();
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  if (t < W) {
    unsigned long long* f = &ph.h[t]->bar[rank];
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
  }
  if (t < W) {
    const unsigned long long* f = &ph.h[rank]->bar[t];
    const unsigned long long t0 = global_ns();  // wall-clock, not SM-clock, timeout
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= epoch) break;
      if (global_ns() - t0 > kBarrierTimeoutNs) {
        atomicExch(&ph.h[rank]->err, 1u);
        atomicOr(fail, 1ull);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
}

__global__ void x_fwd_hdr_kernel(PeerHdrs ph, uint32_t W, uint32_t rank,
                                 const uint32_t* __restrict__ cnt,
                                 const uint32_t* __restrict__ seg) {
  pdl_entry();
  const uint32_t d = threadIdx.x;
  if (d < W) {
    ph.h[d]->fwd_cnt[rank] = cnt[d];
    ph.h[d]->fwd_seg[rank] = seg[d];
  }
}

__global__ void x_bwd_hdr_kernel(PeerHdrs ph, uint32_t W, uint32_t rank,
                                 const uint64_t* __restrict__ pair_off,
                                 const uint32_t* __restrict__ cnt) {
  pdl_entry();
  const uint32_t d = threadIdx.x;
  if (d < W) {
    ph.h[d]->bwd_cnt[rank] = static_cast<uint32_t>(pair_off[d + 1] - pair_off[d]);
    ph.h[d]->bwd_single[rank] = cnt[kCntSingle + d];  // its first pairs: no position word
  }
}

// Where this rank's pairs start in each owner's (source-rank major) pair arrays.
__global__ void x_bwd_base_kernel(PeerHdrs ph, uint32_t W, uint32_t rank,
                                  uint64_t* __restrict__ base) {
  pdl_entry();
  const uint32_t d = threadIdx.x;
  if (d < W) {
    uint64_t b = 0;
    for (uint32_t r = 0; r < rank; ++r) b += ld_volatile(&ph.h[d]->bwd_cnt[r]);
    base[d] = b;
  }
}

// Owner: the rows (and versions) of the ids source r asked for, written straight into
// source r's rows buffer at its segment for this owner.
template <int V, int L, bool kGuard>
__global__ void __launch_bounds__(256)
    x_owner_gather_kernel(DevTable t, const uint32_t* __restrict__ oslot, uint64_t stride,
                          const XHdr* __restrict__ hdr, PeerRows pr,
                          uint64_t* __restrict__ orv, PeerRows pooled,
                          const uint32_t* __restrict__ tgt, float kappa, uint64_t scale_off) {
  pdl_entry();
  using Gm = Geo<V, L, kGuard>;
  const uint32_t r = blockIdx.y;
  const uint64_t n = ld_volatile(&hdr->fwd_cnt[r]);
  const uint64_t seg = ld_volatile(&hdr->fwd_seg[r]);
  const uint32_t D = t.D;
  const int ln = Gm::lane();
  const uint64_t gid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  const uint64_t groups = static_cast<uint64_t>(gridDim.x) * blockDim.x / L;
  float* dst_base = pr.p[r] + seg * D;
  if constexpr (!kGuard) {
    // kGatherILP rows in flight per lane group: the slot / target loads, then the row
    // loads, then the (mostly remote, NVLink) stores -- independent chains, so the
    // random-row latency overlaps instead of serialising per row
    constexpr int kGatherILP = 4;
    for (uint64_t j0 = gid; j0 < n; j0 += groups * kGatherILP) {
      uint32_t s[kGatherILP], g[kGatherILP];
      bool live[kGatherILP];
#pragma unroll
      for (int u = 0; u < kGatherILP; ++u) {
        const uint64_t j = j0 + u * groups;
        live[u] = j < n;
        s[u] = live[u] ? oslot[r * stride + j] : 0u;
        g[u] = (live[u] && pooled.p[r]) ? tgt[r * stride + j] : 0xffffffffu;
      }
      float v[kGatherILP][V];
#pragma unroll
      for (int u = 0; u < kGatherILP; ++u) {
        if (live[u] && slot_ok(t, s[u]))
          load_vec<V>(t.rows + static_cast<uint64_t>(s[u]) * t.stride + ln * V, v[u]);
        else
          for (int k = 0; k < V; ++k) v[u][k] = 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kGatherILP; ++u) {
        if (!live[u]) continue;
        const uint64_t j = j0 + u * groups;
        // a one-listing group of the requester: its pooled value float(0.0 + (double)row),
        // i.e. row + 0.0f, goes straight into the requester's pooled output
        if (kappa > 0.0f) {  // the row as a compressed PS pull reply (codec.hpp:222-244)
          put_coded<V, L>(pr.p[r], seg + j, scale_off, D, ln * V, v[u], kappa);
          if (ln == 0 && orv) orv[r * stride + j] = slot_ok(t, s[u]) ? vt_read(t, s[u]).x : 0;
          continue;
        }
        float* dst = g[u] != 0xffffffffu ? pooled.p[r] + static_cast<uint64_t>(g[u]) * D
                                         : dst_base + j * D;
        if (g[u] != 0xffffffffu)
          for (int k = 0; k < V; ++k) v[u][k] = __fadd_rn(v[u][k], 0.0f);
        store_vec<V>(dst + ln * V, v[u]);
        if (ln == 0 && orv) orv[r * stride + j] = slot_ok(t, s[u]) ? vt_read(t, s[u]).x : 0;
      }
    }
    return;
  }
  for (uint64_t j = gid; j < n; j += groups) {
    const uint32_t s = oslot[r * stride + j];
    const bool ok = slot_ok(t, s);
    const float* row = t.rows + static_cast<uint64_t>(ok ? s : 0) * t.stride;
    // a one-listing group of the requester: its pooled value float(0.0 + (double)row),
    // i.e. row + 0.0f, goes straight into the requester's pooled output
    const uint32_t g = pooled.p[r] ? tgt[r * stride + j] : 0xffffffffu;
    float* dst = g != 0xffffffffu ? pooled.p[r] + static_cast<uint64_t>(g) * D
                                  : dst_base + j * D;
    if constexpr (!kGuard) {
      float v[V];
      if (ok) load_vec<V>(row + ln * V, v);
      else for (int k = 0; k < V; ++k) v[k] = 0.0f;
      if (g != 0xffffffffu)
        for (int k = 0; k < V; ++k) v[k] = __fadd_rn(v[k], 0.0f);
      store_vec<V>(dst + ln * V, v);
    } else {
      for (uint32_t d = ln; d < D; d += L) {
        const float v = ok ? row[d] : 0.0f;
        dst[d] = g != 0xffffffffu ? __fadd_rn(v, 0.0f) : v;
      }
    }
    if (ln == 0 && orv) orv[r * stride + j] = ok ? vt_read(t, s).x : 0;
  }
}

static size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

void xbatch_arena(XBatch& x, uint64_t max_ids, uint64_t max_groups, uint32_t D, void* out_handle) {
  if (x.arena) throw Error(HPS_E_PRECONDITION, "exchange arena already created");
  if (!max_ids || !D) throw Error(HPS_E_PRECONDITION, "exchange arena: empty");
  if (x.kappa > 0.0f && (D % 4 != 0 || D > 128 || (D & (D - 1)) != 0))
    throw Error(HPS_E_PRECONDITION, "exchange codec: dim must be a power of two in [4, 128]");
  const uint64_t W = x.G, M = max_ids;
  size_t o = al256(sizeof(XHdr));
  x.off_ids = o;     o += al256(W * M * 8);
  x.off_rows = o;    o += al256(M * D * 4);
  x.off_ppos = o;    o += al256(W * M * 4);
  x.off_contrib = o; o += al256(W * M * D * 4);
  x.off_oslot = o;   o += al256(W * M * 4);
  x.off_oids = o;    o += al256(W * M * 8);
  x.off_ocnt = o;    o += al256(kMaxWorld * 4);
  x.off_tgt = o;     o += al256(W * M * 4);
  x.off_pooled = o;  o += al256(static_cast<size_t>(max_groups) * D * 4);
  x.arena_bytes = o;
  x.max_groups = max_groups;
  HPS_CUDA(cudaMalloc(&x.gdirect, std::max<uint64_t>(max_groups, 1)));
  HPS_CUDA(cudaMalloc(&x.glist, std::max<uint64_t>(max_groups, 1) * sizeof(uint32_t)));
  x.max_ids = M;
  x.arena_dim = D;
  HPS_CUDA(cudaMalloc(&x.arena, o));
  HPS_CUDA(cudaMemset(x.arena, 0, al256(sizeof(XHdr))));
  HPS_CUDA(cudaMalloc(&x.xbase, 33 * sizeof(uint64_t)));
  HPS_CUDA(cudaMalloc(&x.dev_epoch, sizeof(unsigned long long)));
  HPS_CUDA(cudaMemset(x.dev_epoch, 0, sizeof(unsigned long long)));
  x.arena_rows = reinterpret_cast<float*>(x.arena + x.off_rows);
  if (x.kappa > 0.0f) {
    HPS_CUDA(cudaMalloc(&x.dec_contrib, W * M * D * sizeof(float)));
  }
  cudaIpcMemHandle_t h;
  HPS_CUDA(cudaIpcGetMemHandle(&h, x.arena));
  memcpy(out_handle, &h, sizeof(h));
}

void xbatch_set_codec(XBatch& x, float kappa) {
  if (x.arena) throw Error(HPS_E_PRECONDITION, "exchange codec: set it before the arena");
  if (!(kappa >= 0.0f) || !std::isfinite(kappa))
    throw Error(HPS_E_PRECONDITION, "compress_values: kappa must be positive (0 = off)");
  x.kappa = kappa;
}

void xbatch_connect(XBatch& x, uint32_t rank, const void* handles) {
  if (!x.arena) throw Error(HPS_E_PRECONDITION, "exchange connect: create the arena first");
  if (rank >= x.G) throw Error(HPS_E_PRECONDITION, "exchange connect: bad rank");
  x.rank = rank;
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (uint32_t r = 0; r < x.G; ++r) {
    if (r == rank) {
      x.peer[r] = x.arena;
      continue;
    }
    void* p = nullptr;
    HPS_CUDA(cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess));
    x.peer[r] = static_cast<uint8_t*>(p);
  }
  x.connected = true;
}

static PeerHdrs peer_hdrs(const XBatch& x) {
  PeerHdrs ph{};
  for (uint32_t r = 0; r < x.G; ++r) ph.h[r] = reinterpret_cast<XHdr*>(x.peer[r]);
  return ph;
}

// A timeout flags the table (kCtrProtocol): the step's updates are gated off and the
// failure surfaces from the next synchronising call.
static void barrier(XBatch& x, Table* t, cudaStream_t st) {
  ProfScope p(t, "x_barrier", st);
  launch(x_barrier_kernel, 1, 32, 0, st, peer_hdrs(x), x.G, x.rank, x.dev_epoch,
                                     t->d.ctr + kCtrProtocol);
  HPS_LAUNCH_CHECK();
}

static void require_connected(const XBatch& x, uint32_t D, uint64_t n) {
  if (!x.connected) throw Error(HPS_E_PRECONDITION, "exchange: peer transport not connected");
  if (D != x.arena_dim) throw Error(HPS_E_PRECONDITION, "exchange: dim differs from the arena's");
  if (n > x.max_ids) throw Error(HPS_E_PRECONDITION, "exchange: batch exceeds the arena size");
}

// Forward, phase 1 (no barrier, no table access): route the batch -- distinct ids straight
// into their owners' id regions, counts into their headers -- and plan the backward's
// pairs. fork_pairs: the pair plan on the exchange's aux stream (joined by phase 2),
// else on `st` itself (a prefetch stream already beside the critical path).
static void fwd_route_phase(XBatch& x, Table* t, const uint64_t* ids, uint64_t n,
                            const uint32_t* offsets, uint32_t B, uint32_t F, cudaStream_t st,
                            bool fork_pairs) {
  require_connected(x, t->cfg.embedding_dim, n);
  if (t->d.lru)
    throw Error(HPS_E_PRECONDITION, "exchange: tables with HPS_TABLE_LRU serve the PS surface only");
  const uint64_t M = x.max_ids;
  PeerIds pid{};
  for (uint32_t d = 0; d < x.G; ++d) {
    pid.p[d] = reinterpret_cast<uint64_t*>(x.peer[d] + x.off_ids) + x.rank * M;
    pid.tg[d] = reinterpret_cast<uint32_t*>(x.peer[d] + x.off_tgt) + x.rank * M;
  }
  // one-listing groups are pooled by their rows' owners when the arena's pooled buffer
  // holds the batch (every rank takes the same decision: same batch shapes)
  x.direct_ok = static_cast<uint64_t>(B) * F <= x.max_groups && x.kappa == 0.0f;
  const PeerHdrs ph = peer_hdrs(x);
  {
    ProfScope p(t, "x_route", st);
    route_core(x, ids, n, offsets, B, F, nullptr, pid, st);
    launch(x_fwd_hdr_kernel, 1, 32, 0, st, ph, x.G, x.rank, x.cnt, x.seg);
    HPS_LAUNCH_CHECK();
  }
  // The pair plan of the backward (push_to_shards' per-sample dedup) depends only on the
  // routed batch: it runs on a second stream beside the owner lookup and the row
  // delivery (latency-bound sorts overlapping an NVLink-bound gather), joined before the
  // forward returns.
  x.pairs_ready = false;
  x.pairs_forked = false;
  if (n && !fork_pairs) {
    ProfScope p(t, "x_pairs", st);
    pairs_core(x, &x.pairs_spos, &x.pairs_slist, st);
    x.pairs_ready = true;
  } else if (n) {
    if (!x.aux) {
      HPS_CUDA(cudaStreamCreateWithFlags(&x.aux, cudaStreamNonBlocking));
      HPS_CUDA(cudaEventCreateWithFlags(&x.ev_fork, cudaEventDisableTiming));
      HPS_CUDA(cudaEventCreateWithFlags(&x.ev_join, cudaEventDisableTiming));
    }
    HPS_CUDA(cudaEventRecord(x.ev_fork, st));
    HPS_CUDA(cudaStreamWaitEvent(x.aux, x.ev_fork, 0));
    {
      ProfScope p(t, "x_pairs", x.aux);
      pairs_core(x, &x.pairs_spos, &x.pairs_slist, x.aux);
    }
    HPS_CUDA(cudaEventRecord(x.ev_join, x.aux));
    x.pairs_ready = true;
    x.pairs_forked = true;
  }
}

// Forward, phase 2: the first barrier (ids and counts landed), owner lookup of what every
// source asked for, rows (and one-listing groups' pooled values) straight back to the
// sources, the pair counts, the second barrier.
// Forward, phase 1b: the first barrier (every source's ids and counts landed), then the
// owner's find-or-init of what every source asked for (hash probe + lazy init of new
// rows: no existing row is read or written, so it may run beside another batch's
// apply). The new-row list is the exchange's own (not the table's scratch batch).
static void fwd_probe_phase(XBatch& x, Table* t, cudaStream_t st) {
  const uint64_t M = x.max_ids;
  const PeerHdrs ph = peer_hdrs(x);
  barrier(x, t, st);  // every id region and count has landed
  XHdr* mine = ph.h[x.rank];
  uint32_t* oslot = reinterpret_cast<uint32_t*>(x.arena + x.off_oslot);
  grow(x.pnew, x.cap_pnew, x.G * M + 1);
  HPS_CUDA(cudaMemsetAsync(x.pnew, 0, sizeof(uint32_t), st));  // [0] = new-row count
  {
    ProfScope p(t, "x_owner_probe", st);
    launch_probe_regions(t->d, reinterpret_cast<const uint64_t*>(x.arena + x.off_ids), M, x.G,
                         mine, oslot, reinterpret_cast<uint64_t*>(x.arena + x.off_oids),
                         reinterpret_cast<uint32_t*>(x.arena + x.off_ocnt), x.pnew + 1,
                         x.pnew, t->sm_count, st);
    launch_lazy_init(t->d, x.pnew + 1, x.pnew, x.G * M, t->sm_count, st);
  }
}

// Forward, phase 2: rows (and one-listing groups' pooled values) straight back to the
// sources -- after this rank's previous apply -- the pair counts, the second barrier.
static void fwd_finish_phase(XBatch& x, Table* t, cudaStream_t st) {
  const uint64_t M = x.max_ids;
  const PeerHdrs ph = peer_hdrs(x);
  XHdr* mine = ph.h[x.rank];
  uint32_t* oslot = reinterpret_cast<uint32_t*>(x.arena + x.off_oslot);
  PeerRows pr{}, pp{};
  for (uint32_t r = 0; r < x.G; ++r) {
    pr.p[r] = reinterpret_cast<float*>(x.peer[r] + x.off_rows);
    pp.p[r] = reinterpret_cast<float*>(x.peer[r] + x.off_pooled);
  }
  {
    ProfScope p(t, "x_owner_gather", st);
    HPS_DISPATCH_DIM(t->d.D, {
      const uint32_t bx = static_cast<uint32_t>(std::max<uint64_t>(
          1, std::min<uint64_t>(ceil_div(M, 256 / L), uint64_t(t->sm_count) * 16 / x.G + 1)));
      // (no read versions: the owner applies in fresh mode, see xbatch_bwd)
      launch(x_owner_gather_kernel<V, L, G>, dim3(bx, x.G), 256, 0, st, 
          t->d, oslot, M, mine, pr, nullptr, x.direct_ok ? pp : PeerRows{},
          reinterpret_cast<const uint32_t*>(x.arena + x.off_tgt), x.kappa, M * t->d.D / 2);
    });
    HPS_LAUNCH_CHECK();
  }
  // The backward's pair counts are known once the pair plan has finished: they ride on
  // this barrier instead of one of their own. (Safe against the next step: a source
  // writes step s+1's counts only after the first barrier of s+1, which every owner
  // reaches after its step-s apply has read them.)
  if (x.pairs_ready && x.pairs_forked) HPS_CUDA(cudaStreamWaitEvent(st, x.ev_join, 0));
  else if (!x.pairs_ready) HPS_CUDA(cudaMemsetAsync(x.pair_off, 0, 33 * sizeof(uint64_t), st));
  if (!x.pairs_ready) HPS_CUDA(cudaMemsetAsync(x.cnt + kCntSingle, 0, 32 * sizeof(uint32_t), st));
  launch(x_bwd_hdr_kernel, 1, 32, 0, st, ph, x.G, x.rank, x.pair_off, x.cnt);
  HPS_LAUNCH_CHECK();
  x.counts_sent = true;
  barrier(x, t, st);  // every owner's rows have landed in this rank's rows buffer
}

void xbatch_fwd(XBatch& x, Table* t, const uint64_t* ids, uint64_t n, const uint32_t* offsets,
                uint32_t B, uint32_t F, cudaStream_t st) {
  require_connected(x, t->cfg.embedding_dim, n);
  x.prefetched = false;
  fwd_route_phase(x, t, ids, n, offsets, B, F, st, /*fork_pairs=*/true);
  fwd_probe_phase(x, t, st);
  x.generation = t->generation;
  fwd_finish_phase(x, t, st);
}

void xbatch_prefetch(XBatch& x, Table* t, const uint64_t* ids, uint64_t n,
                     const uint32_t* offsets, uint32_t B, uint32_t F, cudaStream_t st) {
  require_connected(x, t->cfg.embedding_dim, n);
  fwd_route_phase(x, t, ids, n, offsets, B, F, st, /*fork_pairs=*/false);
  fwd_probe_phase(x, t, st);
  x.generation = t->generation;
  x.prefetched = true;
}

void xbatch_fwd_prefetched(XBatch& x, Table* t, cudaStream_t st) {
  if (!x.prefetched) throw Error(HPS_E_PRECONDITION, "exchange: no prefetched batch");
  x.prefetched = false;
  fwd_finish_phase(x, t, st);
}

void xbatch_bwd(XBatch& x, Table* t, const float* grads, float lr, uint32_t step_tag,
                uint32_t epoch, int* accepted, uint32_t flags, cudaStream_t st) {
  const uint32_t D = t->cfg.embedding_dim;
  require_connected(x, D, x.N);
  require_device(grads, "hps_exchange_bwd grads");
  const uint64_t M = x.max_ids;
  const PeerHdrs ph = peer_hdrs(x);
  // the pair plan ran beside the forward, whose last barrier also delivered the counts
  if (!x.counts_sent) throw Error(HPS_E_PRECONDITION, "exchange backward: no forward for this batch");
  // the owner applies through the slots its forward probe found: a reset / restore of the
  // table since then voids them (every rank must run the step again)
  if (x.generation != t->generation)
    throw Error(HPS_E_STALE_SAMPLE, "exchange backward: the table was reset or restored since "
                                    "this batch's forward");
  x.counts_sent = false;
  const uint32_t* spos = x.pairs_spos;
  const uint32_t* slist = x.pairs_slist;
  x.pairs_ready = false;
  launch(x_bwd_base_kernel, 1, 32, 0, st, ph, x.G, x.rank, x.xbase);
  HPS_LAUNCH_CHECK();
  if (x.N) {
    PairOut po{};
    for (uint32_t d = 0; d < x.G; ++d) {
      po.c[d] = reinterpret_cast<float*>(x.peer[d] + x.off_contrib);
      po.p[d] = reinterpret_cast<uint32_t*>(x.peer[d] + x.off_ppos);
      po.bad[d] = &ph.h[d]->bad[x.rank];
    }
    po.epoch = x.dev_epoch;
    po.kappa = x.kappa;
    po.scale_off = static_cast<uint64_t>(x.G) * M * D / 2;
    ProfScope p(t, "x_emit", st);
    emit_pairs(x, grads, D, spos, slist, x.xbase, po, st);
  }
  barrier(x, t, st);  // every pair has landed at its owner
  ProfScope p_apply(t, "x_owner_apply", st);
  // owner: a device-counted batch of the pairs that arrived (no host round trip: the
  // whole step stays stream-ordered and capturable in a CUDA graph)
  XHdr* mine = ph.h[x.rank];
  const uint64_t cap = x.G * M;
  XScratch& xs = t->xs;
  grow(xs.ids, xs.cap_ids, cap);
  grow(xs.rv, xs.cap_rv, cap);
  grow(xs.off, xs.cap_off, cap + 1);
  Batch& b = t->scratch;
  b.agg = HPS_SUM;
  batch_reserve(b, cap, cap, cap);
  launch(x_owner_dyn_kernel, grid_n(cap + 1, t->sm_count), kXBlock, 0, st, 
      mine, reinterpret_cast<const uint32_t*>(x.arena + x.off_ocnt), x.G, M,
      reinterpret_cast<const uint64_t*>(x.arena + x.off_oids), nullptr,
      reinterpret_cast<const uint32_t*>(x.arena + x.off_ppos), cap, xs.ids, xs.rv, xs.off,
      t->d.ctr + kCtrProtocol, batch_plan_view(b), reinterpret_cast<const uint32_t*>(x.arena + x.off_oslot),
      b.slot, x.dev_epoch, b.small + kSmallFlags);
  HPS_LAUNCH_CHECK();
  batch_register(b, xs.ids, cap, xs.off, static_cast<uint32_t>(cap), 1, nullptr, st, true,
                 /*slots_ready=*/true);
  // Fresh mode: every pair's read version is the row's version before this apply. The
  // forward read the rows at their current versions and nothing mutates this table
  // between a step's forward and its apply (one batch in flight per exchange), so this
  // is the version the forward read -- without carrying it through the arena.
  b.pulled = true;
  b.rv_valid = false;
  const float* contrib = reinterpret_cast<const float*>(x.arena + x.off_contrib);
  if (x.kappa > 0.0f) {  // compressed pushes (codec.hpp:246-261), P = offsets[cap]
    decode(contrib, cap * D / 2, D, cap, xs.off + cap, x.dec_contrib, t->sm_count, st);
    contrib = x.dec_contrib;
  }
  batch_push(b, HPS_SUM, contrib, lr, step_tag, epoch, 0, nullptr, accepted,
             flags | kPushPrechecked, st);
}

}  // namespace hps
