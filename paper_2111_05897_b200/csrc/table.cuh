// Device-resident embedding table and per-batch plan (host-side objects).
//
// HBM layout of one table:
//   ht[H]        16 B  open-addressing id index {u64 key, u32 slot}, H = pow2 >= 2*capacity
//                      (load <= 0.5); one probe = one 32-byte sector
//   rows[C][2D+4] f32  [w D | acc D | header] per slot -- the reference row
//                      (embedding_ps.hpp:64) plus a 16-byte header {version (# distinct
//                      steps that wrote the row, embedding_ps.hpp:482), step tag of the
//                      latest version bump (replaces the 16-deep ring), 0, 0}; one
//                      contiguous segment, read-modify-written by the update
//   slot_id[C]   u64   id held by a slot (init seed, export)
// Slots are handed out densely from a device high-water mark (lru_store.hpp:98).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <vector>

#include "common.cuh"

namespace hps {

// Device counter words (u64).
enum CounterIdx : int {
  kCtrMisses = 0,
  kCtrClockResets = 1,
  kCtrStaleDrops = 2,
  kCtrOverflow = 3,    // sticky: capacity exhausted (no LRU eviction on device)
  kCtrDivergence = 4,  // sticky until reported: some push was rejected (non-finite /
                       //   overflowing contribution); its own gate is the call flag
  kCtrUnused5 = 5,
  kCtrMaxDelay = 6,
  kCtrDelayHist = 7,   // 17 words: delays 0..15, >=16
  kCtrProtocol = 24,   // sticky until reported: malformed exchange input (exchange.cu)
  kCtrEvictions = 25,  // LRU mode: rows evicted (PsShard::eviction_count embedding_ps.hpp:75)
  kCtrStep = 30,       // HPS_DEVICE_STEP counter (low 32 bits used)
  kCtrScratch = 31,    // per-call scratch (pair counts)
  kCtrCount = 32
};

// One 16-byte index entry: a probe touches a single 32-byte sector.
struct __align__(16) HashEntry {
  unsigned long long key;  // kEmptyKey when free
  uint32_t slot;           // kPending while the inserting thread publishes it
  uint32_t pad;
};

// The {version, latest bump tag} word of a row lives in the row's own 16-byte header
// right after [w | acc]: the update's version read-modify-write then falls in the row's
// DRAM page instead of costing a separate random access (tools/microbench2.cu: a
// separate 8-byte version array added ~30% to the update).
struct VtView {
  float* rows;
  uint32_t stride;
  uint32_t off;  // 2D
  __host__ __device__ uint2& operator[](uint64_t s) const {
    return *reinterpret_cast<uint2*>(rows + s * stride + off);
  }
};

// Row pitch: [w D | acc D | header 16 B] padded to whole 128-byte lines (or to a power of
// two below one line), so a row never straddles more lines than it fills: a D=64 row is
// 5 lines (640 B) and its weight vector exactly lines 0-1. The unpadded 528-byte pitch
// made the pool's 256-byte weight read touch 3 lines (160 MB of DRAM reads for 109 MB
// algorithmic per C2 step, profiles/r1_ncu_full_c2.txt).
// Adagrad tables with D in {64, 128} keep {version, tag} in the sign bits of the first 64
// optimizer-state floats instead of a header (svt): the accumulator is a sum of squares,
// so its sign bit is otherwise always 0, and the update -- which reads and writes every
// accumulator anyway -- saves a whole extra random line per row (23 us of 132 us per C2
// step, measured). Rows are then exactly [w D | acc D] = 512 B (D=64).
inline bool uses_svt(uint32_t D, int opt) { return opt == HPS_ADAGRAD && (D == 64 || D == 128); }

inline uint32_t row_stride_floats(uint32_t D, bool svt = false) {
  if (svt) return 2 * D;
  uint32_t bytes = 8 * D + 16;
  if (bytes >= 128) return ((bytes + 127) / 128) * 32;
  uint32_t p = 16;
  while (p < bytes) p <<= 1;
  return p / 4;
}

struct DevTable {
  HashEntry* ht;
  uint64_t ht_mask;
  int ht_shift;       // 64 - log2(H)
  uint32_t* special;  // slot of id == kEmptyKey (kSpecialAbsent / kSpecialInserting / slot)
  float* rows;
  uint32_t D;
  uint32_t stride;  // floats per row: row_stride_floats(D) ([w D | acc D | header 16 B | pad])
  VtView vt;        // {version, latest bump tag} in each row's header (unless svt)
  bool svt;         // versions in the accumulators' sign bits (uses_svt)
  // Batch-plan bitmaps, one bit per slot (2 x capacity/8 bytes: L2-resident): `seen`
  // = listed by the batch being planned, `multi` = listed more than once (plan.cu).
  uint32_t* seen;
  uint32_t* multi;  // (a batch's two bitmaps are one allocation: seen, then multi)
  uint64_t* slot_id;
  // [C][kTagRing] step tags of each row's latest version bumps (PsShard::tag_ring_
  // embedding_ps.hpp:493-494): written at every bump (one 4-byte store), read only when
  // the delay needs the exact count (UpdateArgs::exact) or an untracked write moves the
  // version onto an older ring entry.
  uint32_t* ring;
  // LRU mode (HPS_TABLE_LRU): logical shard s owns slots [s * shard_cap, (s+1) * shard_cap)
  // (PsShardConfig::capacity per shard, lru_store.hpp), allocated from shard_hwm[s]; each
  // slot's last touch time is stamp[slot] (the LRU order of the shard's rows; lru.cu).
  uint32_t lru;
  uint32_t shard_cap;
  uint32_t* shard_hwm;
  unsigned long long* shard_evict;  // [S] evictions per shard (HPS1 header field)
  unsigned long long* stamp;
  uint32_t capacity;
  uint32_t* hwm;
  unsigned long long* ctr;
  const uint64_t* salts;
  uint32_t S;
  int opt;
};

constexpr uint32_t kSpecialAbsent = 0xffffffffu;
constexpr uint32_t kSpecialInserting = 0xfffffffdu;

struct Table;

// Reusable device + pinned bounce buffers for host-pointer arguments (table.cu).
struct StagePool {
  struct Buf {
    void* dev = nullptr;
    void* pinned = nullptr;
    size_t dev_cap = 0, pinned_cap = 0;
  };
  std::vector<Buf> bufs;
  void free_all();
  ~StagePool() { free_all(); }
};

// Reusable device workspace for one batch (grown on demand, never shrunk).
struct Batch {
  Table* table = nullptr;
  int agg = HPS_MEAN;  // EmbeddingWorkerConfig::aggregation
  uint32_t B = 0, F = 0;
  uint64_t N = 0;
  uint64_t cap_N = 0, cap_BF = 0, cap_B = 0;
  uint32_t* offsets = nullptr;    // [B*F+1] our copy of the CSR offsets
  uint32_t* lgrp = nullptr;       // [N] listing -> b*F+g
  uint32_t* slot = nullptr;       // [N] listing -> table slot
  uint32_t* keys_a = nullptr;     // [N] sort ping-pong (slot keys)
  uint32_t* vals_a = nullptr;     //     (listing values)
  uint32_t* keys_b = nullptr;
  uint32_t* vals_b = nullptr;
  const uint32_t* sorted_slot = nullptr;
  const uint32_t* sorted_listing = nullptr;
  uint32_t* rv = nullptr;         // [N] per-listing read version (u32) from the last pull
  uint32_t* new_slots = nullptr;  // [N] rows inserted by register (lazy-init queue)
  uint8_t* kind = nullptr;        // [N] plan: 1 = row listed once, 2 = multi (sorted path)
  unsigned long long* mkeys = nullptr;  // [N] multi listings as (slot << lbits | listing)
  uint32_t* slist = nullptr;      // [N] multi-hot batches: listings of rows listed once
                                  //   (classify; count small[12])
  uint32_t* hot = nullptr;        // [N / kHotRun + 1] sorted-list starts of hot rows
  uint32_t* mlist = nullptr;      // [N + 1] sorted-list starts of the other listed rows
  uint64_t* meta = nullptr;       // [N] large path: per sorted position, group | size << 32
  bool meta_ok = false;
  // dynamic batches (one listing per live group, live groups first): the live count is
  // offsets[B*F] on the device; kernels bound their loops by it
  const uint32_t* n_live = nullptr;
  uint32_t* small_slot = nullptr;       // [kSmallN] multi listings sorted (small path)
  uint32_t* small_listing = nullptr;
  uint32_t* hist = nullptr;       // sort / plan scratch
  size_t hist_cap = 0;
  // device scalars (kSmallWords, zeroed by register): [0] multi listings, [2] rows
  // inserted, [6] multi-list rows, [8..10] hot lists, [16..18] the push's call flags
  uint32_t* small = nullptr;
  bool all_multi = false;         // plan skipped: every listing on the sorted path
  bool rv_valid = false;          // rv holds the pull-time versions (else: no mutation since)
  // sample-order permutation (sample_keys != NULL)
  uint64_t* skeys_a = nullptr;
  uint64_t* skeys_b = nullptr;
  uint32_t* sperm_a = nullptr;
  uint32_t* sperm_b = nullptr;
  uint32_t* sstart = nullptr;
  bool pulled = false;
  bool registered = false;
  uint64_t generation = 0;        // Table::generation at register (slots valid only then)
  bool sort_pending = false;      // the plan's gated large sort runs on the table's aux
                                  // stream beside the pooling; joined before its use
  cudaEvent_t ev_sort = nullptr;  // recorded after that sort (joined by pull / push)
  // hps_batch_defer_plan_join: the plan's sort is joined by the push (or an explicit
  // hps_batch_join_plan), not by the register / pull -- also inside a graph capture, where
  // the caller then owns the join (the push in the same capture, or join_plan)
  bool defer_join = false;
  bool sort_in_capture = false;
  // Per-batch plan bitmaps (1 bit per slot: listed / listed more than once), so the plan
  // of the next batch can be built while this batch's update runs.
  uint32_t* seen = nullptr;
  uint32_t* multi = nullptr;
};

// Optional per-region CUDA-event timing on the launching stream (hps_profile_*).
struct Profiler {
  bool enabled = false;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t next();
  void reset();
  void destroy();
};

struct ProfScope {
  ProfScope(Table* t, const char* name, cudaStream_t st);
  ~ProfScope();
  Table* t;
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
};

// Owner-side workspace of the multi-GPU exchange (exchange.cu).
constexpr uint32_t kMaxWorld = 32;

// Header of a rank's peer-mapped exchange arena (exchange.cu). Peers write into it over
// NVLink: barrier arrivals, and per source rank the counts of what it delivered.
struct alignas(128) XHdr {
  unsigned long long bar[kMaxWorld];  // bar[r] = last barrier epoch rank r reached
  uint32_t fwd_cnt[kMaxWorld];        // ids source r wrote into my id region r
  uint32_t fwd_seg[kMaxWorld];        // where my rows go in source r's rows buffer
  uint32_t bwd_cnt[kMaxWorld];        // pairs source r sends me
  uint32_t bwd_single[kMaxWorld];     // ... of which its first ones are single pairs
  uint32_t bad[kMaxWorld];            // = the emit's barrier epoch if source r sent me a
                                      //   non-finite contribution in that step
  uint32_t err;                       // barrier timeout seen by this rank
};
struct XScratch {
  uint64_t* ids = nullptr;
  uint64_t* rv = nullptr;
  uint32_t* off = nullptr;
  uint64_t cap_ids = 0, cap_rv = 0, cap_off = 0;
};

struct Table {
  hps_table_cfg cfg{};
  Profiler prof;
  int device = 0;
  DevTable d{};
  uint64_t ht_size = 0;
  uint64_t* d_salts = nullptr;
  std::vector<uint64_t> salts;
  uint32_t epoch = 0;
  uint32_t sm_count = 148;
  std::mutex mu;  // one call at a time per table (PsShard's per-shard lock)
  cudaStream_t side = nullptr;  // captures the bodies of conditional graph nodes
  cudaStream_t aux = nullptr;       // registers' large-plan sorts beside the pooling
  cudaStream_t aux_push = nullptr;  // a push's multi-row updates beside update_single
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_sort = nullptr, ev_runs = nullptr;
  cudaStream_t aux_hot = nullptr, aux_lo = nullptr;
  cudaEvent_t ev_hot0 = nullptr, ev_hot1 = nullptr;
  // Bumped whenever the slot numbering is rebuilt (clear / reset / checkpoint load): a
  // batch registered under an older generation names slots that may now hold other rows.
  uint64_t generation = 0;
  // Newest host step tag a tracked apply used, and whether some tracked apply used an
  // older one since the last clear (out-of-order steps: hybrid stragglers).
  uint32_t max_tag = 0;
  bool disordered = false;
  uint64_t clock = 1;  // LRU mode: touch time of the next access (stamps; 0 = never)
  uint32_t* lru_scratch = nullptr;  // LRU mode: per-shard counts / candidate ranges
  void* lru_keys = nullptr;         // LRU mode: candidate sort keys (ping-pong)
  void* lru_keys2 = nullptr;
  uint64_t lru_cap = 0;
  bool untracked_seen = false;  // some untracked write (version += 1 without a ring entry)
  Batch scratch;  // workspace for the stateless entry points
  StagePool stage;
  // Batches pulled but not yet pushed. Their read versions are only materialised
  // (snapshot) when some other mutation is about to run before their own push.
  std::vector<Batch*> outstanding;
  unsigned long long* h_ctr = nullptr;  // pinned mirror of the counters
  XScratch xs;
};

#ifdef __CUDACC__
// svt encoding: accumulator element 4l + k (l < 16) carries, in its sign bit, bit l of
// k = 0: version low half, 1: version high half, 2: tag low half, 3: tag high half.
__device__ __forceinline__ uint32_t sign_of(float x) { return __float_as_uint(x) >> 31; }
__device__ __forceinline__ float with_sign(float mag, uint32_t bit) {
  return __uint_as_float((__float_as_uint(mag) & 0x7fffffffu) | (bit << 31));
}
// One thread reads a row's {version, tag} (header, or the 64 sign bits).
__device__ __forceinline__ uint2 vt_read(const DevTable& t, uint32_t s) {
  if (!t.svt) return t.vt[s];
  const float4* a = reinterpret_cast<const float4*>(t.rows + static_cast<uint64_t>(s) * t.stride + t.D);
  uint32_t ver = 0, tag = 0;
#pragma unroll
  for (int l = 0; l < 16; ++l) {
    const float4 q = a[l];
    ver |= (sign_of(q.x) << l) | (sign_of(q.y) << (16 + l));
    tag |= (sign_of(q.z) << l) | (sign_of(q.w) << (16 + l));
  }
  return make_uint2(ver, tag);
}
#endif

// ---- kernels / launchers (kernels.cu, update.cu) ---------------------------------------
// Owner side of the peer exchange: slots[r * stride + j] = find_or_insert(ids[r * stride + j])
// for j < hdr->fwd_cnt[r], r < W (counts are device-side); the ids and counts are also
// copied to owner-local memory (peers may overwrite the regions once the step moves on).
void launch_probe_regions(const DevTable& t, const uint64_t* ids, uint64_t stride, uint32_t W,
                          const XHdr* hdr, uint32_t* slots, uint64_t* ids_copy,
                          uint32_t* cnt_copy, uint32_t* new_slots, uint32_t* new_count, int sms,
                          cudaStream_t st);
void launch_route(const uint64_t* ids, uint64_t n, uint32_t S, uint32_t* out, cudaStream_t st);
// Plan kinds per listing: low bits 1 = row listed once in the batch, 2 = more than once,
// 0 = no row; kKindAlone = the listing is alone in its (sample, group).
constexpr uint8_t kKindAlone = 4;
void launch_expand_groups(const uint32_t* offsets, uint32_t BF, uint32_t* lgrp, cudaStream_t st,
                          uint8_t* kind = nullptr, uint32_t* copy = nullptr,
                          uint32_t* zero = nullptr, uint32_t nzero = 0);
// slots[i] = find_or_insert(ids[i]); when sort_keys/sort_vals are given also writes the
// (slot, i) pairs the apply-order sort consumes.
// plan: also mark the rows in the batch-plan bitmaps (plan.cu).
void launch_probe(const DevTable& t, const uint64_t* ids, uint64_t n, uint32_t* slots,
                  uint32_t* sort_keys, uint32_t* sort_vals, uint32_t* new_slots,
                  uint32_t* new_count, bool plan, cudaStream_t st,
                  const uint32_t* n_dev = nullptr);
// plan.cu
void launch_classify(const DevTable& t, const uint32_t* slots, uint64_t n, int lbits,
                     uint8_t* kind, unsigned long long* mkeys, uint32_t* n_multi,
                     uint32_t* slist, uint32_t* n_single, int sms,
                     cudaStream_t st, const uint32_t* n_live = nullptr);
void launch_ht_clear(const DevTable& t, cudaStream_t st);
void launch_lazy_init(const DevTable& t, const uint32_t* new_slots, const uint32_t* new_count,
                      uint64_t max_new, int sms, cudaStream_t st);
void launch_gather(const DevTable& t, const uint32_t* slots, uint64_t n, float* out_values,
                   uint64_t* out_versions, cudaStream_t st);
void launch_peek(const DevTable& t, const uint64_t* ids, uint64_t n, float* out_w, float* out_acc,
                 uint64_t* out_versions, uint8_t* out_present, cudaStream_t st);
// glist/glist_n (optional): pool only the listed groups (device-side count); the others'
// pooled values are already in `out` (one-listing groups the exchange owners wrote).
void launch_pool(const DevTable& t, const uint32_t* offsets, const uint32_t* slots, uint32_t BF,
                 uint64_t N, int mean, float* out, uint64_t* out_rv64, uint32_t* out_rv32,
                 cudaStream_t st, const uint32_t* glist = nullptr,
                 const uint32_t* glist_n = nullptr);
// checkpoint images (kernels.cu): gather [w | acc] + version of slots; adopt rows
void launch_ckpt_gather(const DevTable& t, const uint32_t* slots, uint64_t n, float* rows2d,
                        uint64_t* vers, cudaStream_t st);
void launch_ckpt_restore(const DevTable& t, const uint64_t* ids, const float* rows2d,
                         const uint64_t* vers, uint64_t n, uint32_t* new_slots,
                         uint32_t* new_count, cudaStream_t st, const uint32_t* at = nullptr,
                         const unsigned long long* stamps = nullptr);
void launch_snapshot_rv(const DevTable& t, const uint32_t* slots, uint64_t n, uint32_t* rv,
                        cudaStream_t st);
void launch_check_direct(const float* grads, uint64_t n_floats, uint32_t* flag,
                         cudaStream_t st);
// Per-call flag words of a push (uint32, in the batch's device scalars, zeroed by its
// register): kCflagReject = a contribution is non-finite or overflows -- the call's
// updates are gated off (the table's sticky kCtrDivergence is raised too, so an
// HPS_ASYNC push's rejection surfaces at the next sync); kCflagNeedExact = the
// validation's bound was inconclusive (the exact check ran in the check kernel's last
// block); kCflagDone = block-completion counter of the check kernel.
constexpr int kCflagReject = 0, kCflagNeedExact = 1, kCflagDone = 2;
constexpr int kSmallFlags = 16;  // Batch::small[16..18]: the push's call flags
constexpr int kSmallWords = 32;

struct UpdateArgs {
  // Multi kernel input: either the large-path slot sort of all n listings, or -- when
  // n_dev is given and *n_dev <= kSmallN -- the small sorted multi list of *n_dev
  // entries. Single kernel: skips everything when *n_dev > kSmallN (large path).
  const uint32_t* sorted_slot;
  const uint32_t* sorted_listing;
  const uint32_t* small_slot;
  const uint32_t* small_listing;
  uint64_t n;            // listings of the batch (entries of the direct apply)
  const uint32_t* n_dev; // multi listings of the plan (device), or null
  const uint8_t* kind;   // single kernel: plan kinds per listing
  // single kernel, large plans of multi-hot batches: the listings of rows listed once
  // (count *n_single) -- most of such a batch's listings belong to multi-listed rows
  const uint32_t* slist;
  const uint32_t* n_single;
  const uint32_t* slots; // single kernel: slot per listing
  // batch mode
  const uint32_t* lgrp;
  const uint32_t* offsets;
  uint32_t F;
  int mean;
  // contributions: batch mode -> grads[B*F*D] fanned out; direct mode -> grads[n*D]
  const float* grads;
  // read versions per listing/entry (tracked); exactly one of these or none
  const uint32_t* rv32;
  const uint64_t* rv64;
  uint32_t* out_delays;  // direct mode, per entry
  float lr;
  uint32_t step_tag;
  // HPS_DEVICE_STEP: tag = *step_dev (the table step counter, advanced by this push's
  // check kernel before any update kernel reads it)
  const uint32_t* step_dev;
  uint32_t* cflags;  // this call's flag words (kCflag*), or null
  int tracked;
  int fresh;  // tracked, and no mutation since the pull: read version = current version
  // count delays from the tag ring (count_delay exactly) instead of the latest bump tag:
  // needed once step tags went out of order or untracked writes happened on the table
  int exact;
  // Large (sorted) plans: rows listed more than once, as listed by runs_kernel for
  // update_runs -- hot (>= kHotRun listings, very hot >= kVeryHotRun from the end)
  uint32_t* hot;
  uint32_t* n_hot;
  uint32_t hot_cap;
  // and the other multi rows; null = update_multi scans the sorted positions
  uint32_t* mlist;
  uint32_t* n_mlist;
  uint32_t mlist_cap;
  // large (sorted) path: per sorted position, the listing's group | group size << 32
  const uint64_t* meta;
  // dynamic batches: live listings (= live groups) on the device; null = a.n
  const uint32_t* n_live;
  // the multi list (rows of 2..kHotRun-1 listings) goes to update_short, not update_runs
  int short_multi;
};
constexpr uint32_t kHotRun = 64;
constexpr uint32_t kVeryHotRun = 1024;
// Validation before mutation (embedding_ps.hpp:146-156) of a batch push: every gradient
// finite, and the fan-out's float narrowing bounded (else the exact check of every pair
// contribution runs in the kernel's last block). Reads a.grads [B*F][D] with a.offsets,
// a.F, a.mean, a.n_live; flags into a.cflags (+ the table's sticky kCtrDivergence).
// step_ctr (HPS_DEVICE_STEP): the last block advances the table's step counter, which
// the update kernels then read as their tag.
void launch_check_batch(const DevTable& t, const UpdateArgs& a, uint32_t B,
                        unsigned long long* step_ctr, cudaStream_t st);
// large plan: every row listed more than once (warp per row and 32-dim chunk)
void launch_update_runs(const DevTable& t, const UpdateArgs& a, int sms, cudaStream_t st);
void launch_runs(const UpdateArgs& a, int sms, cudaStream_t st);
void launch_update(const DevTable& t, const UpdateArgs& a, bool direct, int sms, cudaStream_t st);
void launch_update_single(const DevTable& t, const UpdateArgs& a, int sms, cudaStream_t st);
void launch_update_short(const DevTable& t, const UpdateArgs& a, int sms, cudaStream_t st);
bool update_short_fits(const DevTable& t, const UpdateArgs& a);
void launch_count_pairs(const UpdateArgs& a, unsigned long long* ctr, cudaStream_t st);

void launch_sample_order(const uint64_t* sample_keys, uint32_t B, uint64_t* keys_out,
                         uint32_t* perm_out, cudaStream_t st);
void launch_sample_lengths(const uint32_t* perm, const uint32_t* offsets, uint32_t B, uint32_t F,
                           uint32_t* lens, cudaStream_t st);
void launch_scan_inplace(uint32_t* data, uint32_t n, uint32_t* total, cudaStream_t st);
void launch_permuted_listing(const uint32_t* perm, const uint32_t* starts,
                             const uint32_t* offsets, const uint32_t* slots, uint32_t B,
                             uint32_t F, uint32_t* keys_out, uint32_t* vals_out, cudaStream_t st);
void launch_add_counter_from(unsigned long long* ctr, int idx, const uint32_t* src,
                             cudaStream_t st);
void launch_add_counter_const(unsigned long long* ctr, int idx, unsigned long long v,
                              cudaStream_t st);
void launch_iota(uint32_t* out, uint64_t n, cudaStream_t st);

}  // namespace hps
