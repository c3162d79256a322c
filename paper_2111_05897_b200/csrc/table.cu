// Host-side orchestration of the hot path: table lifecycle, the PS surface
// (lookup / apply / peek) and the embedding-worker batch surface (register /
// pull / push). Every public entry point is in capi.cu; this file throws
// hps::Error and never returns status codes itself.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "radix_sort.cuh"
#include "table.cuh"
#include "table_impl.h"

namespace hps {

// ---- pointer staging --------------------------------------------------------------------

PtrKind ptr_kind(const void* p) {
  if (!p) return PtrKind::kDevice;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return PtrKind::kPageable;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return PtrKind::kDevice;
  if (at.type == cudaMemoryTypeHost) return PtrKind::kPinned;
  return PtrKind::kPageable;
}

DeviceGuard::DeviceGuard(int dev) {
  HPS_CUDA(cudaGetDevice(&prev_));
  changed_ = dev >= 0 && dev != prev_;
  if (changed_) HPS_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
  if (changed_) cudaSetDevice(prev_);
}

template <typename T>
static void ensure(T*& p, uint64_t& cap, uint64_t need) {
  if (need <= cap && p) return;
  if (p) HPS_CUDA(cudaFree(p));
  p = nullptr;
  uint64_t n = std::max<uint64_t>(need, 1);
  HPS_CUDA(cudaMalloc(&p, n * sizeof(T)));
  cap = n;
}

void StagePool::free_all() {
  for (Buf& b : bufs) {
    if (b.dev) cudaFree(b.dev);
    if (b.pinned) cudaFreeHost(b.pinned);
  }
  bufs.clear();
}

StagePool::Buf& Stager::next(size_t bytes, bool need_pinned) {
  if (used_ == pool_.bufs.size()) pool_.bufs.emplace_back();
  StagePool::Buf& b = pool_.bufs[used_++];
  bytes = std::max<size_t>(bytes, 16);
  if (b.dev_cap < bytes) {
    if (b.dev) HPS_CUDA(cudaFree(b.dev));
    b.dev = nullptr;
    HPS_CUDA(cudaMalloc(&b.dev, bytes));
    b.dev_cap = bytes;
  }
  if (need_pinned && b.pinned_cap < bytes) {
    if (b.pinned) HPS_CUDA(cudaFreeHost(b.pinned));
    b.pinned = nullptr;
    HPS_CUDA(cudaMallocHost(&b.pinned, bytes));
    b.pinned_cap = bytes;
  }
  return b;
}

const void* Stager::in(const void* p, size_t bytes, cudaStream_t st) {
  if (!p) return p;
  PtrKind k = ptr_kind(p);
  if (k == PtrKind::kDevice) return p;
  sync_needed_ = true;
  StagePool::Buf& b = next(bytes, k == PtrKind::kPageable);
  if (!bytes) return b.dev;
  if (k == PtrKind::kPageable) {
    memcpy(b.pinned, p, bytes);
    HPS_CUDA(cudaMemcpyAsync(b.dev, b.pinned, bytes, cudaMemcpyHostToDevice, st));
  } else {
    HPS_CUDA(cudaMemcpyAsync(b.dev, p, bytes, cudaMemcpyHostToDevice, st));
  }
  return b.dev;
}

void* Stager::out(void* p, size_t bytes) {
  if (!p) return p;
  PtrKind k = ptr_kind(p);
  if (k == PtrKind::kDevice) return p;
  sync_needed_ = true;
  StagePool::Buf& b = next(bytes, k == PtrKind::kPageable);
  outs_.push_back(Out{p, b.dev, k == PtrKind::kPageable ? b.pinned : nullptr, bytes});
  return b.dev;
}

void Stager::finish(cudaStream_t st) {
  for (Out& o : outs_)
    if (o.bytes)
      HPS_CUDA(cudaMemcpyAsync(o.pinned ? o.pinned : o.host, o.dev, o.bytes,
                               cudaMemcpyDeviceToHost, st));
  if (sync_needed_) HPS_CUDA(cudaStreamSynchronize(st));
  for (Out& o : outs_)
    if (o.pinned && o.bytes) memcpy(o.host, o.pinned, o.bytes);
  outs_.clear();
}

// ---- profiling ------------------------------------------------------------------------------

cudaEvent_t Profiler::next() {
  if (used == pool.size()) {
    cudaEvent_t e;
    HPS_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}

void Profiler::reset() {
  recs.clear();
  used = 0;
}

void Profiler::destroy() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
  pool.clear();
  reset();
}

ProfScope::ProfScope(Table* tb, const char* n, cudaStream_t s) : t(tb), name(n), st(s) {
  if (t->prof.enabled) {
    a = t->prof.next();
    HPS_CUDA(cudaEventRecord(a, st));
  }
}

ProfScope::~ProfScope() {
  if (a) {
    cudaEvent_t b = t->prof.next();
    cudaEventRecord(b, st);
    t->prof.recs.push_back({name, a, b});
  }
}

void profile_enable(Table* t, bool on) {
  t->prof.reset();
  t->prof.enabled = on;
}

// Sum of elapsed ms and record count of one region since profile_enable().
void profile_get(Table* t, const char* name, double* ms, uint64_t* count) {
  HPS_CUDA(cudaDeviceSynchronize());
  double total = 0;
  uint64_t n = 0;
  for (auto& r : t->prof.recs) {
    if (strcmp(r.name, name) != 0) continue;
    float x = 0;
    HPS_CUDA(cudaEventElapsedTime(&x, r.a, r.b));
    total += x;
    ++n;
  }
  *ms = total;
  *count = n;
}

// ---- table lifecycle -----------------------------------------------------------------------

Table* table_create(const hps_table_cfg& cfg) {
  if (cfg.shard_count == 0) throw Error(HPS_E_CONFIG, "hps_table_create: shard_count must be positive");
  if (!cfg.shard_salts) throw Error(HPS_E_CONFIG, "hps_table_create: shard_salts required");
  if (cfg.embedding_dim == 0) throw Error(HPS_E_CONFIG, "hps_table_create: embedding_dim must be positive");
  const bool lru = (cfg.flags & HPS_TABLE_LRU) != 0;
  if (lru && (cfg.shard_capacity == 0 ||
              cfg.shard_capacity * static_cast<uint64_t>(cfg.shard_count) >= (1ull << 31)))
    throw Error(HPS_E_CONFIG, "hps_table_create: HPS_TABLE_LRU needs shard_capacity in [1, 2^31 / S)");
  // < 2^31 rows keeps every hash-entry index (H <= 2^32) in 32 bits.
  if (!lru && (cfg.capacity == 0 || cfg.capacity >= (1ull << 31)))
    throw Error(HPS_E_CONFIG, "hps_table_create: capacity must be in [1, 2^31)");
  if (cfg.optimizer != HPS_ADAGRAD && cfg.optimizer != HPS_SGD)
    throw Error(HPS_E_CONFIG, "hps_table_create: unknown optimizer");
  if (cfg.world_size == 0 || cfg.owner_rank >= cfg.world_size)
    throw Error(HPS_E_CONFIG, "hps_table_create: owner_rank must be < world_size");
  if (cfg.flags & ~(HPS_TABLE_TAG_RING | HPS_TABLE_LRU))
    throw Error(HPS_E_CONFIG, "hps_table_create: unknown flags");
  auto t = new Table();
  try {
    t->cfg = cfg;
    if (lru) t->cfg.capacity = cfg.shard_capacity * cfg.shard_count;
    t->salts.assign(cfg.shard_salts, cfg.shard_salts + cfg.shard_count);
    t->cfg.shard_salts = t->salts.data();
    if (cfg.device >= 0) {
      t->device = cfg.device;
    } else {
      HPS_CUDA(cudaGetDevice(&t->device));
    }
    DeviceGuard g(t->device);
    cudaDeviceProp prop{};
    HPS_CUDA(cudaGetDeviceProperties(&prop, t->device));
    t->sm_count = prop.multiProcessorCount;

    const uint64_t C = t->cfg.capacity;
    uint64_t H = 1024;
    int lg = 10;
    while (H < 2 * C) H <<= 1, ++lg;
    t->ht_size = H;
    DevTable& d = t->d;
    d.ht_mask = H - 1;
    d.ht_shift = 64 - lg;
    d.D = cfg.embedding_dim;
    d.svt = uses_svt(cfg.embedding_dim, cfg.optimizer);
    d.stride = row_stride_floats(cfg.embedding_dim, d.svt);
    d.capacity = static_cast<uint32_t>(C);
    d.S = cfg.shard_count;
    d.opt = cfg.optimizer;
    HPS_CUDA(cudaMalloc(&d.ht, H * sizeof(HashEntry)));
    HPS_CUDA(cudaMalloc(&d.rows, C * d.stride * sizeof(float)));
    d.vt = VtView{d.rows, d.stride, 2 * d.D};
    HPS_CUDA(cudaMalloc(&d.seen, (C / 32 + 1) * sizeof(uint32_t)));
    HPS_CUDA(cudaMalloc(&d.multi, (C / 32 + 1) * sizeof(uint32_t)));
    HPS_CUDA(cudaMalloc(&d.slot_id, C * sizeof(uint64_t)));
    if (cfg.flags & HPS_TABLE_TAG_RING)
      HPS_CUDA(cudaMalloc(&d.ring, C * kTagRing * sizeof(uint32_t)));
    if (lru) {
      d.lru = 1;
      d.shard_cap = static_cast<uint32_t>(cfg.shard_capacity);
      HPS_CUDA(cudaMalloc(&d.shard_hwm, cfg.shard_count * sizeof(uint32_t)));
      HPS_CUDA(cudaMalloc(&d.shard_evict, cfg.shard_count * sizeof(unsigned long long)));
      HPS_CUDA(cudaMalloc(&d.stamp, C * sizeof(unsigned long long)));
    }
    HPS_CUDA(cudaMalloc(&d.special, sizeof(uint32_t)));
    HPS_CUDA(cudaMalloc(&d.hwm, sizeof(uint32_t)));
    HPS_CUDA(cudaMalloc(&d.ctr, kCtrCount * sizeof(unsigned long long)));
    HPS_CUDA(cudaMalloc(&t->d_salts, cfg.shard_count * sizeof(uint64_t)));
    HPS_CUDA(cudaMemcpy(t->d_salts, t->salts.data(), cfg.shard_count * sizeof(uint64_t),
                        cudaMemcpyHostToDevice));
    d.salts = t->d_salts;
    HPS_CUDA(cudaMallocHost(&t->h_ctr, kCtrCount * sizeof(unsigned long long)));
    HPS_CUDA(cudaMemset(d.ctr, 0, kCtrCount * sizeof(unsigned long long)));
    table_clear(t, nullptr);
    HPS_CUDA(cudaDeviceSynchronize());
    t->scratch.table = t;
    return t;
  } catch (...) {
    table_destroy(t);
    throw;
  }
}

// Empties the index and the row store (LruStore::clear + PsShard state reset).
void table_clear(Table* t, cudaStream_t st) {
  DevTable& d = t->d;
  ++t->generation;
  t->max_tag = 0;  // every row's bump tags are gone (kNoStep), like the reference's rings
  t->disordered = false;
  t->untracked_seen = false;
  launch_ht_clear(d, st);
  HPS_CUDA(cudaMemsetAsync(d.seen, 0, (d.capacity / 32 + 1) * sizeof(uint32_t), st));
  HPS_CUDA(cudaMemsetAsync(d.multi, 0, (d.capacity / 32 + 1) * sizeof(uint32_t), st));
  HPS_CUDA(cudaMemsetAsync(d.special, 0xff, sizeof(uint32_t), st));
  HPS_CUDA(cudaMemsetAsync(d.hwm, 0, sizeof(uint32_t), st));
  if (d.lru) {
    HPS_CUDA(cudaMemsetAsync(d.shard_hwm, 0, d.S * sizeof(uint32_t), st));
    HPS_CUDA(cudaMemsetAsync(d.shard_evict, 0, d.S * sizeof(unsigned long long), st));
    HPS_CUDA(cudaMemsetAsync(d.stamp, 0, d.capacity * sizeof(unsigned long long), st));
    t->clock = 1;
  }
  HPS_CUDA(cudaMemsetAsync(d.ctr + kCtrOverflow, 0, sizeof(unsigned long long), st));
}

static void ensure_aux(Table* t) {
  if (t->aux) return;
  // The registers' sorts (gated: a few no-op launches for one-hot batches) at the highest
  // priority, so they slot in beside the previous push instead of queueing behind its
  // waves; the push's multi-row stream keeps the default (highest measured slower,
  // profiles/r2_sched_ab.txt).
  int lo = 0, hi = 0;
  HPS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  HPS_CUDA(cudaStreamCreateWithPriority(&t->aux, cudaStreamNonBlocking, hi));
  HPS_CUDA(cudaStreamCreateWithFlags(&t->aux_lo, cudaStreamNonBlocking));
  HPS_CUDA(cudaStreamCreateWithFlags(&t->aux_push, cudaStreamNonBlocking));
  HPS_CUDA(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
  HPS_CUDA(cudaEventCreateWithFlags(&t->ev_join, cudaEventDisableTiming));
  HPS_CUDA(cudaEventCreateWithFlags(&t->ev_runs, cudaEventDisableTiming));
  HPS_CUDA(cudaEventCreateWithFlags(&t->ev_sort, cudaEventDisableTiming));
}

// The batch's large-plan sort (forked by batch_register) has finished before `st` goes on
// (the batch's own event: another batch may be registered -- and sorted -- meanwhile).
// A batch registered eagerly and pulled inside a CUDA-graph capture: its sort is work
// from before the capture (completed before the graph is launched, as any capture's
// inputs must be) and cannot be a dependency of the graph.
static void join_sort(Batch& b, cudaStream_t st) {
  if (!b.sort_pending) return;
  b.sort_pending = false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  HPS_CUDA(cudaStreamIsCapturing(st, &cs));
  // (a captured register rejoined its fork itself -- unless its batch defers the join)
  if (cs == cudaStreamCaptureStatusActive && !b.sort_in_capture) return;
  b.sort_in_capture = false;
  HPS_CUDA(cudaStreamWaitEvent(st, b.ev_sort, 0));
}

void batch_join_plan(Batch& b, cudaStream_t st) { join_sort(b, st); }

DevTable batch_plan_view(Batch& b) {
  Table* t = b.table;
  if (!b.seen) {
    const size_t words = t->d.capacity / 32 + 1;
    HPS_CUDA(cudaMalloc(&b.seen, 2 * words * sizeof(uint32_t)));
    b.multi = b.seen + words;
    HPS_CUDA(cudaMemset(b.seen, 0, 2 * words * sizeof(uint32_t)));
  }
  DevTable d = t->d;
  d.seen = b.seen;
  d.multi = b.multi;
  return d;
}

static void forget_outstanding(Batch& b) {
  if (!b.table) return;
  auto& v = b.table->outstanding;
  v.erase(std::remove(v.begin(), v.end(), &b), v.end());
}

// Copy-on-write of read versions: before any mutation of the table, every batch that
// was pulled but not yet pushed (other than `except`) materialises its pull-time
// versions, so its own push can still count staleness delays exactly. In the sync
// step (pull, push, pull, ...) nothing is ever outstanding and this costs nothing.
static void protect_reads(Table* t, const Batch* except, cudaStream_t st) {
  for (Batch* y : t->outstanding) {
    if (y == except || y->rv_valid || !y->registered) continue;
    launch_snapshot_rv(t->d, y->slot, y->N, y->rv, st);
    y->rv_valid = true;
  }
}

void batch_free(Batch& b) {
  forget_outstanding(b);
  if (b.ev_sort) cudaEventDestroy(b.ev_sort);
  if (b.seen) cudaFree(b.seen);  // (multi shares the allocation)
  b.seen = b.multi = nullptr;
  void* ptrs[] = {b.offsets, b.lgrp,  b.slot,   b.keys_a,  b.vals_a,
                  b.keys_b,  b.vals_b, b.rv,  b.new_slots, b.kind,  b.hist,
                  b.mkeys,   b.slist, b.hot, b.mlist, b.meta, b.small_slot, b.small_listing,
                  b.small,   b.skeys_a, b.skeys_b, b.sperm_a, b.sperm_b, b.sstart};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  Table* t = b.table;
  int agg = b.agg;
  b = Batch{};
  b.table = t;
  b.agg = agg;
}

void table_destroy(Table* t) {
  if (!t) return;
  {
    DeviceGuard g(t->device);
    cudaDeviceSynchronize();
    batch_free(t->scratch);
    t->stage.free_all();
    t->prof.destroy();
    DevTable& d = t->d;
    void* ptrs[] = {d.ht, d.rows, d.seen, d.multi, d.slot_id, d.ring, d.shard_hwm, d.stamp,
                    d.shard_evict,
                    t->lru_scratch, t->lru_keys, t->lru_keys2, d.special,
                    d.hwm, d.ctr,  t->d_salts, t->xs.ids, t->xs.rv,  t->xs.off};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (t->h_ctr) cudaFreeHost(t->h_ctr);
    if (t->side) cudaStreamDestroy(t->side);
    if (t->aux) cudaStreamDestroy(t->aux);
    if (t->aux_lo) cudaStreamDestroy(t->aux_lo);
    if (t->aux_push) cudaStreamDestroy(t->aux_push);
    if (t->ev_fork) cudaEventDestroy(t->ev_fork);
    if (t->ev_join) cudaEventDestroy(t->ev_join);
    if (t->ev_runs) cudaEventDestroy(t->ev_runs);
    if (t->aux_hot) cudaStreamDestroy(t->aux_hot);
    if (t->ev_hot0) cudaEventDestroy(t->ev_hot0);
    if (t->ev_hot1) cudaEventDestroy(t->ev_hot1);
    if (t->ev_sort) cudaEventDestroy(t->ev_sort);
  }
  delete t;
}

void read_counters(Table* t, cudaStream_t st) {
  HPS_CUDA(cudaMemcpyAsync(t->h_ctr, t->d.ctr, kCtrCount * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
}

void table_counters(Table* t, hps_counters* out) {
  DeviceGuard g(t->device);
  HPS_CUDA(cudaDeviceSynchronize());
  read_counters(t, nullptr);
  uint32_t hwm = 0;
  HPS_CUDA(cudaMemcpy(&hwm, t->d.hwm, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof(*out));
  const unsigned long long* c = t->h_ctr;
  out->misses = c[kCtrMisses];
  out->clock_resets = c[kCtrClockResets];
  out->stale_epoch_drops = c[kCtrStaleDrops];
  out->size = std::min<uint64_t>(hwm, t->cfg.capacity);
  if (t->d.lru) {
    std::vector<uint32_t> sh(t->d.S);
    HPS_CUDA(cudaMemcpy(sh.data(), t->d.shard_hwm, t->d.S * sizeof(uint32_t),
                        cudaMemcpyDeviceToHost));
    out->size = 0;
    for (uint32_t v : sh) out->size += std::min(v, t->d.shard_cap);
  }
  out->evictions = c[kCtrEvictions];
  out->capacity = t->cfg.capacity;
  out->epoch = t->epoch;
  out->max_delay = static_cast<uint32_t>(c[kCtrMaxDelay]);
  for (int i = 0; i < 17; ++i) out->delay_hist[i] = c[kCtrDelayHist + i];
}

// The divergence flag belongs to the push that raised it: it is reported once (by
// that push, or by the next table sync for an HPS_ASYNC push) and then cleared.
void check_flags(Table* t, cudaStream_t st, bool divergence) {
  read_counters(t, st);
  if (t->h_ctr[kCtrOverflow])
    throw Error(HPS_E_CONFIG,
                "embedding table capacity exhausted (" + std::to_string(t->cfg.capacity) +
                    " rows); device tables do not evict -- raise capacity");
  if (t->h_ctr[kCtrProtocol]) {
    HPS_CUDA(cudaMemsetAsync(t->d.ctr + kCtrProtocol, 0, sizeof(unsigned long long), st));
    HPS_CUDA(cudaStreamSynchronize(st));
    throw Error(HPS_E_PROTOCOL,
                "exchange failed (a pair named an id outside its source's segment, or a peer "
                "missed a barrier); the step's updates were not applied");
  }
  if (divergence && t->h_ctr[kCtrDivergence]) {
    HPS_CUDA(cudaMemsetAsync(t->d.ctr + kCtrDivergence, 0, sizeof(unsigned long long), st));
    HPS_CUDA(cudaStreamSynchronize(st));
    throw Error(HPS_E_DIVERGENCE, "non-finite gradient contribution; nothing was applied");
  }
}

void table_sync(Table* t) {
  DeviceGuard g(t->device);
  HPS_CUDA(cudaDeviceSynchronize());
  check_flags(t, nullptr);
}

void table_reset(Table* t) {
  DeviceGuard g(t->device);
  HPS_CUDA(cudaDeviceSynchronize());
  table_clear(t, nullptr);
  HPS_CUDA(cudaDeviceSynchronize());
  t->epoch++;
}

// ---- batch workspace --------------------------------------------------------------------

// Buffers grow with 25% slack: batch sizes that vary from call to call (exchange
// receive sides) must not reallocate -- and synchronise the device -- every step.
static inline uint64_t with_slack(uint64_t n) { return n + n / 4 + 1024; }

void batch_reserve(Batch& b, uint64_t N, uint64_t BF, uint64_t B) {
  uint64_t n = std::max<uint64_t>(N, 1);
  if (n > b.cap_N) {
    n = with_slack(n);
    uint64_t c = 0;
    uint32_t** bufs[] = {&b.lgrp, &b.slot,   &b.keys_a,   &b.vals_a,
                         &b.keys_b, &b.vals_b, &b.rv,   &b.new_slots};
    for (uint32_t** p : bufs) {
      c = 0;
      ensure(*p, c, n);
    }
    c = 0;
    ensure(b.kind, c, n);
    c = 0;
    ensure(b.mkeys, c, n);
    c = 0;
    ensure(b.slist, c, n);
    c = 0;
    ensure(b.hot, c, n / kHotRun + 1);
    c = 0;
    ensure(b.mlist, c, n + 1);
    c = 0;
    ensure(b.meta, c, n);
    size_t hw = radix::scratch_words<uint32_t>(n);
    if (hw > b.hist_cap) {
      c = 0;
      ensure(b.hist, c, hw);
      b.hist_cap = hw;
    }
    b.cap_N = n;
  }
  if (BF + 1 > b.cap_BF) {
    uint64_t c = 0;
    BF = with_slack(BF);
    ensure(b.offsets, c, BF + 1);
    b.cap_BF = BF + 1;
  }
  if (B > b.cap_B) {
    B = with_slack(B);
    uint64_t c = 0;
    ensure(b.skeys_a, c, B);
    c = 0;
    ensure(b.skeys_b, c, B);
    c = 0;
    ensure(b.sperm_a, c, B);
    c = 0;
    ensure(b.sperm_b, c, B);
    c = 0;
    ensure(b.sstart, c, B + 1);
    size_t hw = radix::scratch_words<uint64_t>(B);
    if (hw > b.hist_cap) {
      c = 0;
      ensure(b.hist, c, hw);
      b.hist_cap = hw;
    }
    b.cap_B = B;
  }
  if (!b.small) {
    uint64_t c = 0;
    ensure(b.small, c, kSmallWords);
    c = 0;
    ensure(b.small_slot, c, radix::kSmallN);
    c = 0;
    ensure(b.small_listing, c, radix::kSmallN);
  }
}

// The update arguments describing a registered batch's plan.
static UpdateArgs plan_args(const Batch& b) {
  UpdateArgs a{};
  a.sorted_slot = b.sorted_slot;
  a.sorted_listing = b.sorted_listing;
  a.small_slot = b.small_slot;
  a.small_listing = b.small_listing;
  a.n = b.N;
  a.n_dev = b.all_multi ? nullptr : &b.small[0];
  a.kind = b.kind;
  a.slots = b.slot;
  // (classify's single-listing list: multi-hot plan batches only)
  const bool listed = !b.all_multi && b.N > 2ull * b.B * b.F;
  a.slist = listed ? b.slist : nullptr;
  a.n_single = listed ? &b.small[12] : nullptr;
  a.lgrp = b.lgrp;
  a.offsets = b.offsets;
  a.F = b.F;
  a.meta = b.meta_ok ? b.meta : nullptr;
  a.n_live = b.n_live;
  return a;
}

static int slot_key_bits(const Table* t) {
  return std::max(1, bits_for(static_cast<uint64_t>(t->cfg.capacity) - 1));
}

// Stable sort of (slot, listing) pairs by slot: every row's listings become one
// contiguous run in apply order. keys_in0 = slots to sort (else keys_a); iota: the
// listings are the positions 0..N-1 (else vals_a); gate = device-side condition
// (radix_sort.cuh): the sort's kernels exit at once when *gate <= kSmallN.
static void sort_slots(Batch& b, const uint32_t* keys_in0, bool iota, const uint32_t* gate,
                       cudaStream_t st, bool plan_meta = false) {
  Table* t = b.table;
  ProfScope p(t, "sort", st);
  const int kb = slot_key_bits(t);
  const int passes = (kb + radix::kBits - 1) / radix::kBits;
  b.sorted_slot = (passes & 1) ? b.keys_b : b.keys_a;
  b.sorted_listing = (passes & 1) ? b.vals_b : b.vals_a;
  radix::SortMeta meta;
  // batch plans (not the direct apply): per-position metadata, produced by the large
  // path's final pass (the single-CTA small sort does not)
  b.meta_ok = plan_meta && (gate || b.N > radix::kSmallN);
  if (b.meta_ok) {
    meta.lgrp = b.lgrp;
    meta.offsets = b.offsets;
    meta.out = b.meta;
  }
  auto sort = [&](cudaStream_t s, bool zero) {
    bool in_b = radix::sort_pairs<uint32_t>(b.keys_a, b.vals_a, b.keys_b, b.vals_b, b.N, kb,
                                            b.hist, s, t->sm_count, gate, keys_in0, iota, zero,
                                            meta);
    b.sorted_slot = in_b ? b.keys_b : b.keys_a;
    b.sorted_listing = in_b ? b.vals_b : b.vals_a;
  };
  if (!gate) {
    sort(st, true);
    return;
  }
  // gated large path (device count of multi listings > kSmallN)
  radix::sort_scratch_zero(b.hist, st);
  sort(st, false);
}

// EmbeddingWorker::register_sample for a whole batch + the route/dedup/probe half of
// serve_pull: after this, every listing has its slot (rows lazily initialised) and the
// listings are grouped per row in apply order.
void batch_register(Batch& b, const uint64_t* ids, uint64_t N, const uint32_t* offsets, uint32_t B,
                    uint32_t F, const uint64_t* sample_keys, cudaStream_t st, bool dynamic,
                    bool slots_ready) {
  Table* t = b.table;
  if (N >= 0xffffffffull) throw Error(HPS_E_PRECONDITION, "batch too large (>= 2^32 listings)");
  const uint64_t BF = static_cast<uint64_t>(B) * F;
  if (BF >= 0xffffffffull) throw Error(HPS_E_PRECONDITION, "batch too large (B*F >= 2^32)");
  if (F == 0) throw Error(HPS_E_PRECONDITION, "register: feature group count must be positive");
  if (t->d.lru)
    throw Error(HPS_E_PRECONDITION, "register: the batch surface needs a table without "
                                    "HPS_TABLE_LRU (use hps_lookup / hps_apply)");
  join_sort(b, st);
  forget_outstanding(b);
  b.rv_valid = false;
  batch_reserve(b, N, BF, B);
  const DevTable pv = batch_plan_view(b);
  Stager stg(t->stage);
  const uint64_t* d_ids =
      slots_ready ? nullptr : static_cast<const uint64_t*>(stg.in(ids, N * sizeof(uint64_t), st));
  if (!is_device_ptr(offsets)) {
    if (offsets[BF] != N || offsets[0] != 0)
      throw Error(HPS_E_PRECONDITION, "register: offsets[B*F] must equal n_ids and offsets[0] 0");
    for (uint64_t i = 0; i < BF; ++i)
      if (offsets[i] > offsets[i + 1])
        throw Error(HPS_E_PRECONDITION, "register: offsets must be non-decreasing");
  }
  const uint32_t* d_off =
      static_cast<const uint32_t*>(stg.in(offsets, (BF + 1) * sizeof(uint32_t), st));
  const uint64_t* d_sk =
      static_cast<const uint64_t*>(stg.in(sample_keys, B * sizeof(uint64_t), st));
  b.B = B;
  b.F = F;
  b.N = N;
  b.n_live = dynamic ? b.offsets + BF : nullptr;
  // Keep our own copy of the offsets so later pull/push calls do not depend on caller
  // buffers (ids are consumed here: everything after register works on slots), and clear
  // the batch's device scalars (plan counts, hot-row lists, the push's call flags; an
  // exchange owner's assembly (slots_ready) has already written the call flags) -- all
  // in the launch that expands the groups.
  launch_expand_groups(d_off, static_cast<uint32_t>(BF), b.lgrp, st, b.kind, b.offsets, b.small,
                       slots_ready ? kSmallFlags : kSmallWords);
  // Sample keys that reorder the batch: every listing takes the sorted (multi) path.
  const bool permute = d_sk && B > 1;
  b.all_multi = permute;
  if (!slots_ready) {
    {
      ProfScope p(t, "probe", st);
      // dynamic: N is only a bound; the live listing count is offsets[B*F] on the device
      // (new rows are initialised by the probe itself: no lazy-init launch per batch)
      launch_probe(pv, d_ids, N, b.slot, nullptr, nullptr, nullptr, &b.small[2], !permute, st,
                   dynamic ? b.offsets + BF : nullptr);
    }
  }
  if (permute) {
    // Apply order = ascending sample key: enumerate listings sample by sample in key
    // order before the stable slot sort.
    launch_sample_order(d_sk, B, b.skeys_a, b.sperm_a, st);
    bool in_b = radix::sort_pairs<uint64_t>(b.skeys_a, b.sperm_a, b.skeys_b, b.sperm_b, B, 64,
                                            b.hist, st, t->sm_count);
    const uint32_t* perm = in_b ? b.sperm_b : b.sperm_a;
    launch_sample_lengths(perm, b.offsets, B, F, b.sstart, st);
    launch_scan_inplace(b.sstart, B, b.sstart + B, st);
    launch_permuted_listing(perm, b.sstart, b.offsets, b.slot, B, F, b.keys_a, b.vals_a, st);
    sort_slots(b, nullptr, false, nullptr, st, true);
  } else {
    // Plan (plan.cu): rows listed once apply directly; the multi listings are ordered
    // by the small composite sort, or -- past kSmallN of them -- the whole batch is
    // slot-sorted instead. Both sorts are launched; the device count picks one.
    const int lbits = std::max(1, bits_for(N ? N - 1 : 0));
    {
      ProfScope p(t, "plan", st);
      // (multi-hot batches also list their single listings for update_single)
      const bool list_singles = N > 2ull * BF;
      launch_classify(pv, b.slot, N, lbits, b.kind, b.mkeys, &b.small[0],
                      list_singles ? b.slist : nullptr, &b.small[12], t->sm_count, st,
                      b.n_live);
    }
    {
      ProfScope p(t, "sort_small", st);
      radix::sort_composite_small(b.mkeys, &b.small[0], lbits, b.small_slot, b.small_listing,
                                  st);
    }
    // The gated large sort (a no-op unless the device count of multi listings exceeds
    // kSmallN) needs only the slots; the pooling does not need it. It runs on the aux
    // stream beside the pull and is joined by the pull / push (join_sort; measured
    // 0.2691 -> 0.2660 ms per C2 step against in line, profiles/r1_sort_fork_ab.txt).
    // (a multi-hot batch's sort is real work: at normal priority it yields to the
    // previous batch's hot-row walk, 6.60 -> 6.52 ms at C3; a one-hot batch's gated no-op
    // launches stay at the highest priority, profiles/r2_c3_sched_ab.txt)
    ensure_aux(t);
    cudaStream_t sst = N > 2ull * BF ? t->aux_lo : t->aux;
    HPS_CUDA(cudaEventRecord(t->ev_fork, st));
    HPS_CUDA(cudaStreamWaitEvent(sst, t->ev_fork, 0));
    sort_slots(b, b.slot, true, &b.small[0], sst, true);
    if (!b.ev_sort) HPS_CUDA(cudaEventCreateWithFlags(&b.ev_sort, cudaEventDisableTiming));
    HPS_CUDA(cudaEventRecord(b.ev_sort, sst));
    // Under CUDA-graph capture the fork rejoins the register's own stream (a captured
    // branch must end inside its capture, and a later capture may not wait on it);
    // eagerly, the pull / push of this batch joins it (join_sort).
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    HPS_CUDA(cudaStreamIsCapturing(st, &cs));
    const bool capturing = cs == cudaStreamCaptureStatusActive;
    if (capturing && !b.defer_join) HPS_CUDA(cudaStreamWaitEvent(st, b.ev_sort, 0));
    b.sort_pending = !capturing || b.defer_join;
    b.sort_in_capture = capturing && b.defer_join;
  }
  b.registered = true;
  b.generation = t->generation;
  b.pulled = false;
  stg.finish(st);
}

// Step tags of tracked applies (Table::max_tag). With the tag ring any order counts
// exactly (the kernels walk the ring once the table saw an out-of-order tag or an
// untracked write); without it a tracked apply the latest-bump-tag rule could miscount
// is refused before anything mutates (HPS_TABLE_TAG_RING, hps_c.h). HPS_DEVICE_STEP
// pushes take monotone tags from the device counter.
static void note_tag(Table* t, uint32_t step_tag) {
  if (!t->d.ring) {
    if (step_tag < t->max_tag)
      throw Error(HPS_E_CLOCK, "step tag " + std::to_string(step_tag) + " is older than " +
                                   std::to_string(t->max_tag) +
                                   ", which this table already applied; out-of-order step "
                                   "tags need a table with HPS_TABLE_TAG_RING");
    if (t->untracked_seen)
      throw Error(HPS_E_CLOCK, "tracked apply after an untracked write: exact delays need a "
                               "table with HPS_TABLE_TAG_RING");
  }
  if (step_tag < t->max_tag) t->disordered = true;
  else t->max_tag = step_tag;
}

// A batch whose slots predate a table clear / reset / checkpoint load must not read or
// write through them (the reference resolves ids at apply time, find_or_init).
static void require_current(const Batch& b, const char* what) {
  if (b.generation != b.table->generation)
    throw Error(HPS_E_STALE_SAMPLE, std::string(what) +
                                        ": batch registered before the table was reset or "
                                        "restored from a checkpoint; register it again");
}

void batch_pull(Batch& b, int agg, float* out_pooled, uint64_t* out_rv, cudaStream_t st) {
  if (!b.registered) throw Error(HPS_E_STALE_SAMPLE, "pull: batch not registered");
  require_current(b, "pull");
  Table* t = b.table;
  const uint64_t BF = static_cast<uint64_t>(b.B) * b.F;
  Stager stg(t->stage);
  float* d_out = static_cast<float*>(stg.out(out_pooled, BF * t->cfg.embedding_dim * sizeof(float)));
  uint64_t* d_rv = static_cast<uint64_t*>(stg.out(out_rv, b.N * sizeof(uint64_t)));
  // Read versions are produced only when the caller asks for them; otherwise the push
  // takes them from the table (nothing mutated since) or from a snapshot that a
  // mutation in between forces (protect_reads).
  {
    ProfScope p(t, "pool", st);
    launch_pool(t->d, b.offsets, b.slot, static_cast<uint32_t>(BF), b.N, agg == HPS_MEAN ? 1 : 0,
                d_out, d_rv, d_rv ? b.rv : nullptr, st);
  }
  b.rv_valid = d_rv != nullptr;
  if (!b.pulled) t->outstanding.push_back(&b);
  b.pulled = true;
  // the forward is self-contained (capturable on its own) -- unless the batch defers the
  // plan's join to its push: the pooling does not need the sort
  if (!b.defer_join) join_sort(b, st);
  stg.finish(st);
}

void batch_push(Batch& b, int agg, const float* grads, float lr, uint32_t step_tag,
                uint32_t epoch, int untracked, const uint64_t* rv64, int* accepted,
                uint32_t flags, cudaStream_t st) {
  if (!b.registered) throw Error(HPS_E_STALE_SAMPLE, "push: batch not registered");
  Table* t = b.table;
  join_sort(b, st);
  if (epoch != t->epoch) {
    // PsShard::apply_gradients epoch fence (embedding_ps.hpp:142-145): drop every
    // (sample, unique id) entry of the batch, count them.
    launch_count_pairs(plan_args(b), t->d.ctr + kCtrStaleDrops, st);
    if (!(flags & HPS_ASYNC)) HPS_CUDA(cudaStreamSynchronize(st));
    if (accepted) *accepted = 0;
    return;
  }
  require_current(b, "push");
  if ((rv64 || (!untracked && b.pulled)) && !(flags & HPS_DEVICE_STEP)) note_tag(t, step_tag);
  const uint64_t BF = static_cast<uint64_t>(b.B) * b.F;
  const uint32_t D = t->cfg.embedding_dim;
  protect_reads(t, &b, st);
  Stager stg(t->stage);
  const float* d_g = static_cast<const float*>(stg.in(grads, BF * D * sizeof(float), st));
  const uint64_t* d_rv = static_cast<const uint64_t*>(stg.in(rv64, b.N * sizeof(uint64_t), st));
  // kPushPrechecked (exchange owners): the call's reject flag was set by the owner's
  // batch assembly from what the sources found while emitting
  const bool prechecked = (flags & kPushPrechecked) != 0;
  const bool device_step = (flags & HPS_DEVICE_STEP) != 0;
  const int mean = agg == HPS_MEAN ? 1 : 0;
  UpdateArgs a = plan_args(b);
  const DevTable pv = batch_plan_view(b);
  a.mean = mean;
  a.grads = d_g;
  a.lr = lr;
  a.step_tag = step_tag;
  a.cflags = b.small + kSmallFlags;
  if (device_step) a.step_dev = reinterpret_cast<const uint32_t*>(t->d.ctr + kCtrStep);
  if (!prechecked) {
    // validation (with, for HPS_DEVICE_STEP, the step counter advanced by its last block)
    ProfScope p(t, "check", st);
    launch_check_batch(pv, a, b.B, device_step ? t->d.ctr + kCtrStep : nullptr, st);
  } else if (device_step) {
    launch_add_counter_const(t->d.ctr, kCtrStep, 1, st);
  }
  if (d_rv) {
    a.rv64 = d_rv;
    a.tracked = 1;
  } else if (!untracked && b.pulled) {
    a.tracked = 1;
    if (b.rv_valid) a.rv32 = b.rv;
    else a.fresh = 1;  // no mutation since the pull: read version == current version
  }
  if (!a.tracked) t->untracked_seen = true;
  a.exact = t->d.ring && (t->disordered || t->untracked_seen);

  if (b.meta_ok) {
    // sorted (large) plans: runs_kernel lists the rows listed more than once -- hot
    // (>= kHotRun listings) and very hot ones in b.hot, the others in b.mlist -- for
    // update_runs. Counters b.small[6..11] (zeroed by the register): [6] multi-list
    // rows, [8] hot rows, [10] very hot rows (listed from the end), [9] / [11] claims.
    a.hot = b.hot;
    a.n_hot = &b.small[8];
    a.hot_cap = static_cast<uint32_t>(b.N / kHotRun + 1);
    a.mlist = b.mlist;
    a.n_mlist = &b.small[6];
    a.mlist_cap = static_cast<uint32_t>(b.N + 1);  // (sample-key plans list singles too)
  }
  // Multi-hot batches (more listings than groups): the short runs of the multi list go to
  // update_short, on the main stream after the single pass, beside update_runs' hot rows.
  // (A host-side shape test: a one-hot batch's plan is small, its multi list empty.)
  const bool use_short = !b.all_multi && b.meta_ok && b.N > 2ull * b.B * b.F &&
                         update_short_fits(t->d, a);
  a.short_multi = use_short ? 1 : 0;
  if (!b.all_multi) {
    // Rows listed more than once (ordered chains, latency-bound, few) and rows listed
    // once are disjoint: the multi chains run on a second stream beside the single pass
    // (fork/join events; under graph capture two parallel branches).
    // (its own stream: the next batch's register may be sorting on t->aux meanwhile)
    ensure_aux(t);
    HPS_CUDA(cudaEventRecord(t->ev_fork, st));
    HPS_CUDA(cudaStreamWaitEvent(t->aux_push, t->ev_fork, 0));
    {
      ProfScope p(t, "update_multi", t->aux_push);
      launch_runs(a, t->sm_count, t->aux_push);
      if (use_short) HPS_CUDA(cudaEventRecord(t->ev_runs, t->aux_push));
      launch_update(pv, a, false, t->sm_count, t->aux_push);
      // Multi-hot batches: the hot-row walk (the step's long pole) on a high-priority
      // stream, and the single-row pass only after the runs are listed, so update_runs'
      // blocks are placed first and the single pass fills the SMs its tail leaves
      // (6.75 -> 6.60-6.67 ms at C3, profiles/r2_c3_sched_ab.txt).
      if (use_short) {
        if (!t->aux_hot) {
          int lo = 0, hi = 0;
          HPS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
          HPS_CUDA(cudaStreamCreateWithPriority(&t->aux_hot, cudaStreamNonBlocking, hi));
          HPS_CUDA(cudaEventCreateWithFlags(&t->ev_hot0, cudaEventDisableTiming));
          HPS_CUDA(cudaEventCreateWithFlags(&t->ev_hot1, cudaEventDisableTiming));
        }
        HPS_CUDA(cudaEventRecord(t->ev_hot0, t->aux_push));
        HPS_CUDA(cudaStreamWaitEvent(t->aux_hot, t->ev_hot0, 0));
        launch_update_runs(pv, a, t->sm_count, t->aux_hot);
        HPS_CUDA(cudaEventRecord(t->ev_hot1, t->aux_hot));
        HPS_CUDA(cudaStreamWaitEvent(t->aux_push, t->ev_hot1, 0));
      } else {
        launch_update_runs(pv, a, t->sm_count, t->aux_push);
      }
    }
    {
      ProfScope p(t, "update", st);
      if (use_short) HPS_CUDA(cudaStreamWaitEvent(st, t->ev_runs, 0));
      launch_update_single(pv, a, t->sm_count, st);
      if (use_short) {
        HPS_CUDA(cudaStreamWaitEvent(st, t->ev_runs, 0));  // the multi list is listed
        launch_update_short(pv, a, t->sm_count, st);
      }
    }
    HPS_CUDA(cudaEventRecord(t->ev_join, t->aux_push));
    HPS_CUDA(cudaStreamWaitEvent(st, t->ev_join, 0));
  } else {
    ProfScope p(t, "update_multi", st);
    launch_runs(a, t->sm_count, st);
    launch_update(pv, a, false, t->sm_count, st);
    launch_update_runs(pv, a, t->sm_count, st);
  }
  forget_outstanding(b);
  b.pulled = false;
  b.rv_valid = false;
  if (accepted) *accepted = 1;
  stg.finish(st);
  if (!(flags & HPS_ASYNC)) check_flags(t, st);
}

// (sample, unique id) pairs of the registered batch = optimizer applications a push
// performs (= delays it records).
uint64_t batch_pairs(Batch& b) {
  if (!b.registered) return 0;
  Table* t = b.table;
  join_sort(b, nullptr);
  HPS_CUDA(cudaMemset(t->d.ctr + kCtrScratch, 0, sizeof(unsigned long long)));
  launch_count_pairs(plan_args(b), t->d.ctr + kCtrScratch, nullptr);
  unsigned long long p = 0;
  HPS_CUDA(cudaMemcpy(&p, t->d.ctr + kCtrScratch, sizeof(p), cudaMemcpyDeviceToHost));
  return p;
}

// ---- PS surface ------------------------------------------------------------------------

void table_lookup(Table* t, const uint64_t* ids, uint64_t n, float* out_values,
                  uint64_t* out_versions, cudaStream_t st, uint32_t flags) {
  Batch& b = t->scratch;
  batch_reserve(b, n, 0, 0);
  Stager stg(t->stage);
  const uint64_t* d_ids = static_cast<const uint64_t*>(stg.in(ids, n * sizeof(uint64_t), st));
  float* d_out = static_cast<float*>(stg.out(out_values, n * t->cfg.embedding_dim * sizeof(float)));
  uint64_t* d_ver = static_cast<uint64_t*>(stg.out(out_versions, n * sizeof(uint64_t)));
  if (t->d.lru && lru_needs_eviction(t, d_ids, n, st)) {
    lru_sequential(t, 0, d_ids, n, nullptr, nullptr, 0.0f, 0, 0, d_out, d_ver, nullptr, st);
    b.registered = false;
    stg.finish(st);
    if (!(flags & HPS_ASYNC)) check_flags(t, st, false);
    return;
  }
  HPS_CUDA(cudaMemsetAsync(b.small, 0, 8 * sizeof(uint32_t), st));
  launch_probe(t->d, d_ids, n, b.slot, nullptr, nullptr, b.new_slots, &b.small[2], false, st);
  launch_lazy_init(t->d, b.new_slots, &b.small[2], n, t->sm_count, st);
  launch_gather(t->d, b.slot, n, d_out, d_ver, st);
  if (t->d.lru) lru_stamp(t, b.slot, n, st);
  b.registered = false;
  stg.finish(st);
  if (!(flags & HPS_ASYNC)) check_flags(t, st, false);
}

void table_peek(Table* t, const uint64_t* ids, uint64_t n, float* out_w, float* out_acc,
                uint64_t* out_versions, uint8_t* out_present, cudaStream_t st) {
  const uint32_t D = t->cfg.embedding_dim;
  Stager stg(t->stage);
  const uint64_t* d_ids = static_cast<const uint64_t*>(stg.in(ids, n * sizeof(uint64_t), st));
  float* w = static_cast<float*>(stg.out(out_w, n * D * sizeof(float)));
  float* a = static_cast<float*>(stg.out(out_acc, n * D * sizeof(float)));
  uint64_t* v = static_cast<uint64_t*>(stg.out(out_versions, n * sizeof(uint64_t)));
  uint8_t* p = static_cast<uint8_t*>(stg.out(out_present, n));
  launch_peek(t->d, d_ids, n, w, a, v, p, st);
  stg.finish(st);
}

// PsShard::apply_gradients, array-shaped (embedding_ps.hpp:139-189).
void table_apply(Table* t, const uint64_t* ids, const float* grads, const uint64_t* rv, uint64_t n,
                 float lr, uint32_t step_tag, uint32_t epoch, uint32_t* out_delays,
                 int* accepted, uint32_t flags, cudaStream_t st) {
  Batch& b = t->scratch;
  batch_reserve(b, n, 0, 0);
  if (epoch != t->epoch) {
    uint32_t n32 = static_cast<uint32_t>(n);
    HPS_CUDA(cudaMemcpyAsync(b.small + 1, &n32, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    launch_add_counter_from(t->d.ctr, kCtrStaleDrops, b.small + 1, st);
    HPS_CUDA(cudaStreamSynchronize(st));
    if (accepted) *accepted = 0;
    return;
  }
  if (n >= 0xffffffffull) throw Error(HPS_E_PRECONDITION, "apply: too many entries");
  const uint32_t D = t->cfg.embedding_dim;
  Stager stg(t->stage);
  const uint64_t* d_ids = static_cast<const uint64_t*>(stg.in(ids, n * sizeof(uint64_t), st));
  const float* d_g = static_cast<const float*>(stg.in(grads, n * D * sizeof(float), st));
  const uint64_t* d_rv = static_cast<const uint64_t*>(stg.in(rv, n * sizeof(uint64_t), st));
  uint32_t* d_dl = static_cast<uint32_t*>(stg.out(out_delays, n * sizeof(uint32_t)));
  HPS_CUDA(cudaMemsetAsync(b.small, 0, kSmallWords * sizeof(uint32_t), st));
  // Validate before anything mutates -- including lazy inserts (embedding_ps.hpp:146-156).
  launch_check_direct(d_g, n * D, b.small + kSmallFlags + kCflagReject, st);
  uint32_t bad = 0;
  HPS_CUDA(cudaMemcpyAsync(&bad, b.small + kSmallFlags + kCflagReject, sizeof(bad),
                           cudaMemcpyDeviceToHost, st));
  HPS_CUDA(cudaStreamSynchronize(st));
  if (bad) {
    stg.finish(st);
    throw Error(HPS_E_DIVERGENCE, "PsShard::apply_gradients: non-finite gradient");
  }
  if (t->d.lru) {
    if (d_rv) note_tag(t, step_tag);
    if (!d_rv) t->untracked_seen = true;
    if (lru_needs_eviction(t, d_ids, n, st)) {
      protect_reads(t, nullptr, st);
      lru_sequential(t, d_rv ? 1 : 2, d_ids, n, d_g, d_rv, lr, step_tag,
                     t->d.ring && (t->disordered || t->untracked_seen), nullptr, nullptr, d_dl,
                     st);
      if (accepted) *accepted = 1;
      stg.finish(st);
      if (!(flags & HPS_ASYNC)) check_flags(t, st);
      return;
    }
  }
  if (!d_dl && !t->d.lru) {
    // No per-entry delays wanted: the entries as a batch of one-listing samples (sum
    // aggregation: each contribution applied as given) through the batch plan -- rows
    // listed once skip the ordering sort; repeated ids apply in array order.
    XScratch& xs = t->xs;
    if (n + 1 > xs.cap_off) {
      if (xs.off) HPS_CUDA(cudaFree(xs.off));
      xs.off = nullptr;
      HPS_CUDA(cudaMalloc(&xs.off, (n + 1 + n / 4 + 1024) * sizeof(uint32_t)));
      xs.cap_off = n + 1 + n / 4 + 1024;
    }
    launch_iota(xs.off, n + 1, st);
    b.agg = HPS_SUM;
    batch_register(b, d_ids, n, xs.off, static_cast<uint32_t>(n), 1, nullptr, st);
    batch_push(b, HPS_SUM, d_g, lr, step_tag, epoch, d_rv ? 0 : 1, d_rv, accepted, flags, st);
    b.registered = false;
    stg.finish(st);
    return;
  }
  if (d_rv && !t->d.lru) note_tag(t, step_tag);
  protect_reads(t, nullptr, st);
  forget_outstanding(b);
  b.pulled = false;
  b.N = n;
  b.B = static_cast<uint32_t>(n);
  b.F = 1;
  launch_probe(t->d, d_ids, n, b.slot, b.keys_a, b.vals_a, b.new_slots, &b.small[2], false, st);
  launch_lazy_init(t->d, b.new_slots, &b.small[2], n, t->sm_count, st);
  sort_slots(b, nullptr, false, nullptr, st);
  b.all_multi = true;
  UpdateArgs a{};
  a.sorted_slot = b.sorted_slot;
  a.sorted_listing = b.sorted_listing;
  a.n = n;
  a.grads = d_g;
  a.rv64 = d_rv;
  a.tracked = d_rv ? 1 : 0;
  if (!d_rv) t->untracked_seen = true;
  a.exact = t->d.ring && (t->disordered || t->untracked_seen);
  a.out_delays = d_dl;
  a.lr = lr;
  a.step_tag = step_tag;
  launch_update(t->d, a, true, t->sm_count, st);
  if (t->d.lru) lru_stamp(t, b.slot, n, st);
  b.registered = false;
  if (accepted) *accepted = 1;
  stg.finish(st);
  if (!(flags & HPS_ASYNC)) check_flags(t, st);
}

void route(const uint64_t* ids, uint64_t n, uint32_t S, uint32_t* out, cudaStream_t st) {
  StagePool pool;
  Stager stg(pool);
  const uint64_t* d_ids = static_cast<const uint64_t*>(stg.in(ids, n * sizeof(uint64_t), st));
  uint32_t* d_out = static_cast<uint32_t*>(stg.out(out, n * sizeof(uint32_t)));
  launch_route(d_ids, n, S, d_out, st);
  stg.finish(st);
}

}  // namespace hps
