// Internal host-side declarations shared by table.cu / capi.cu / dedup.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <vector>

#include "table.cuh"

namespace hps {

enum class PtrKind { kDevice, kPinned, kPageable };
PtrKind ptr_kind(const void* p);
inline bool is_device_ptr(const void* p) { return !p || ptr_kind(p) == PtrKind::kDevice; }

struct DeviceGuard {
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
  int prev_ = 0;
  bool changed_ = false;
};

// Per-call staging: inputs that live on the host are copied to device buffers,
// outputs that live on the host are produced in device buffers and copied back by
// finish(), which synchronises the stream when any host buffer was involved.
class Stager {
 public:
  explicit Stager(StagePool& pool) : pool_(pool) {}
  const void* in(const void* p, size_t bytes, cudaStream_t st);
  void* out(void* p, size_t bytes);
  void finish(cudaStream_t st);
  bool any_host() const { return sync_needed_; }

 private:
  struct Out {
    void* host;
    void* dev;
    void* pinned;  // null when host is itself pinned
    size_t bytes;
  };
  StagePool::Buf& next(size_t bytes, bool need_pinned);
  StagePool& pool_;
  size_t used_ = 0;
  std::vector<Out> outs_;
  bool sync_needed_ = false;
};

Table* table_create(const hps_table_cfg& cfg);
void table_destroy(Table* t);
void table_clear(Table* t, cudaStream_t st);
void table_counters(Table* t, hps_counters* out);
void table_sync(Table* t);
void table_reset(Table* t);
// codec.cu: compress_values / decompress_values (codec.hpp:222-261), one block per row
void compress_values(const float* v, uint64_t rows, uint32_t len, float kappa, float* scales,
                     uint16_t* payload, cudaStream_t st);
void decompress_values(const float* scales, const uint16_t* payload, uint64_t rows, uint32_t len,
                       float* out, cudaStream_t st);
// checkpoint.cu: HPS1 image of logical shard `shard` (returns its size; writes it when
// buf holds cap >= size bytes); adopt a set of images (validated first, atomically).
uint64_t table_ckpt_save(Table* t, uint32_t shard, uint32_t shard_capacity, uint8_t* buf,
                         uint64_t cap);
void table_ckpt_load(Table* t, const uint8_t* const* images, const uint64_t* sizes,
                     uint32_t count, int recover);
void read_counters(Table* t, cudaStream_t st);
void profile_enable(Table* t, bool on);
void profile_get(Table* t, const char* name, double* ms, uint64_t* count);
void check_flags(Table* t, cudaStream_t st, bool divergence = true);

void batch_reserve(Batch& b, uint64_t N, uint64_t BF, uint64_t B);
// lru.cu (HPS_TABLE_LRU): does the call need evictions (host round trip); stamps of the
// parallel path; the sequential path (mode 0 lookup, 1 tracked apply, 2 untracked apply)
bool lru_needs_eviction(Table* t, const uint64_t* d_ids, uint64_t n, cudaStream_t st);
void lru_stamp(Table* t, const uint32_t* slots, uint64_t n, cudaStream_t st);
void lru_sequential(Table* t, int mode, const uint64_t* ids, uint64_t n, const float* grads,
                    const uint64_t* rv, float lr, uint32_t step_tag, int exact, float* out_values,
                    uint64_t* out_versions, uint32_t* out_delays, cudaStream_t st);
// The table view a batch's plan kernels use: the table with the batch's own plan bitmaps.
DevTable batch_plan_view(Batch& b);
void batch_free(Batch& b);
// dynamic: N and B are bounds; offsets (device) end at the live count (offsets[B*F]),
// samples past it are empty -- a batch whose size is only known on the device.
// slots_ready: b.slot already holds every listing's slot and the plan bits are marked
// (the exchange owner reuses its forward probe); ids are then not read.
void batch_register(Batch& b, const uint64_t* ids, uint64_t N, const uint32_t* offsets, uint32_t B,
                    uint32_t F, const uint64_t* sample_keys, cudaStream_t st,
                    bool dynamic = false, bool slots_ready = false);
void batch_pull(Batch& b, int agg, float* out_pooled, uint64_t* out_rv, cudaStream_t st);
void batch_join_plan(Batch& b, cudaStream_t st);
// internal push flag (above the public HPS_* bits): contributions already validated
constexpr uint32_t kPushPrechecked = 1u << 16;
void batch_push(Batch& b, int agg, const float* grads, float lr, uint32_t step_tag,
                uint32_t epoch, int untracked, const uint64_t* rv64, int* accepted,
                uint32_t flags, cudaStream_t st);
uint64_t batch_pairs(Batch& b);

void table_lookup(Table* t, const uint64_t* ids, uint64_t n, float* out_values,
                  uint64_t* out_versions, cudaStream_t st, uint32_t flags = 0);
void table_peek(Table* t, const uint64_t* ids, uint64_t n, float* out_w, float* out_acc,
                uint64_t* out_versions, uint8_t* out_present, cudaStream_t st);
void table_apply(Table* t, const uint64_t* ids, const float* grads, const uint64_t* rv, uint64_t n,
                 float lr, uint32_t step_tag, uint32_t epoch, uint32_t* out_delays,
                 int* accepted, uint32_t flags, cudaStream_t st);
void route(const uint64_t* ids, uint64_t n, uint32_t S, uint32_t* out, cudaStream_t st);

// dedup.cu
void exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* tile_sums,
                    uint32_t* total, cudaStream_t st);
void dedup(const uint64_t* ids, uint64_t n, uint64_t* out_unique, uint32_t* out_inverse,
           uint64_t* out_u, cudaStream_t st);
void compress_indices(const uint64_t* ids, uint64_t n, const uint32_t* offsets, uint32_t B,
                      uint32_t G, uint64_t* group_u_off, uint64_t* unique, uint64_t* post_off,
                      uint16_t* postings, cudaStream_t st);

// exchange.cu -- source-side plan of one multi-GPU step (see hps_c.h hps_exchange_*).
struct XBatch {
  int device = 0;
  int sms = 148;
  uint32_t G = 1, S = 1;
  int agg = HPS_MEAN;
  uint32_t B = 0, F = 0;
  uint64_t N = 0;
  int lbits = 1;
  uint64_t* hkeys = nullptr;    // transient distinct-id set [H+1]
  uint32_t* hidx = nullptr;     // [N] listing -> set entry | inserter bit
  uint32_t* hval = nullptr;     // [H+1] entry -> index in its owner's segment
  uint8_t* hmul = nullptr;      // [H+1] entry listed more than once
  uint8_t* dest = nullptr;      // [N] owner rank per listing
  uint32_t* sendpos = nullptr;  // [N] listing -> position in send_ids
  uint32_t* spair = nullptr;    // [N] single pair index within its owner, or ~0
  uint32_t* offsets = nullptr;
  uint32_t* lgrp = nullptr;
  uint32_t *keys_a = nullptr, *vals_a = nullptr, *keys_b = nullptr, *vals_b = nullptr;
  uint32_t* scratch = nullptr;
  uint32_t *head = nullptr, *ex = nullptr, *tsum = nullptr;
  uint32_t* cnt = nullptr;
  uint32_t* seg = nullptr;
  uint8_t* dest_of_pos = nullptr;
  uint64_t* pair_off = nullptr;
  uint32_t* mstart = nullptr;
  unsigned long long* mkeys = nullptr;
  uint32_t *sm_pos = nullptr, *sm_list = nullptr;
  uint64_t* h_buf = nullptr;
  cudaStream_t side = nullptr;  // captures conditional graph bodies
  // peer (NVLink) transport
  uint8_t* arena = nullptr;
  uint8_t* peer[kMaxWorld] = {};
  float* arena_rows = nullptr;
  size_t arena_bytes = 0, off_ids = 0, off_rows = 0, off_ppos = 0, off_contrib = 0,
         off_oslot = 0, off_oids = 0, off_ocnt = 0,
         off_tgt = 0, off_pooled = 0;
  uint64_t max_groups = 0;
  bool direct_ok = false;
  uint8_t* gdirect = nullptr;  // [max_groups] groups the owners pooled this step
  uint32_t* glist = nullptr;   // [max_groups] the other groups (pooled here), count in cnt
  // peer step: the pair plan runs on `aux` beside the owner lookup/gather (fork/join
  // events inside the forward, so a captured forward is self-contained)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool pairs_ready = false;
  bool counts_sent = false;  // the forward delivered this batch's pair counts
  bool pairs_forked = false; // the pair plan ran on `aux` (phase 2 joins it)
  bool prefetched = false;   // phase 1 of the next forward done (hps_exchange_prefetch)
  uint32_t* pnew = nullptr;  // owner probe: [0] new-row count, then the new rows' slots
  // value codec on the NVLink payloads (hps_exchange_set_codec): rows and contributions
  // travel kappa-scaled binary16 (codec.hpp:222-261); decoded here before pooling / apply
  float kappa = 0.0f;
  float* dec_contrib = nullptr;  // [G * max_ids][D]
  uint64_t cap_pnew = 0;
  const uint32_t *pairs_spos = nullptr, *pairs_slist = nullptr;
  uint64_t max_ids = 0;
  uint64_t generation = 0;  // owner table's generation at this batch's forward probe
  uint32_t arena_dim = 0, rank = 0;
  bool connected = false;
  uint64_t* xbase = nullptr;
  unsigned long long* dev_epoch = nullptr;
  uint64_t cap_H = 0, cap_hidx = 0, cap_hval = 0, cap_hmul = 0, cap_dest = 0, cap_sendpos = 0,
           cap_spair = 0, cap_off = 0, cap_lgrp = 0, cap_ka = 0, cap_va = 0, cap_kb = 0,
           cap_vb = 0, cap_scratch = 0, cap_head = 0, cap_ex = 0, cap_tsum = 0, cap_dop = 0;
  ~XBatch();
};
void xbatch_init(XBatch& x);
void xbatch_route(XBatch& x, const uint64_t* ids, uint64_t n, const uint32_t* offsets, uint32_t B,
                  uint32_t F, uint64_t* out_send_ids, uint64_t* out_counts, cudaStream_t st);
void xbatch_pool(XBatch& x, const float* rows, uint32_t D, float* out_pooled, cudaStream_t st);
void xbatch_pairs(XBatch& x, const float* grads, uint32_t D, uint32_t* out_pair_pos,
                  float* out_contrib, uint64_t* out_pair_counts, cudaStream_t st);
void xbatch_arena(XBatch& x, uint64_t max_ids, uint64_t max_groups, uint32_t D, void* out_handle);
void xbatch_connect(XBatch& x, uint32_t rank, const void* handles);
void xbatch_set_codec(XBatch& x, float kappa);
void xbatch_fwd(XBatch& x, Table* t, const uint64_t* ids, uint64_t n, const uint32_t* offsets,
                uint32_t B, uint32_t F, cudaStream_t st);
// the forward in two phases: route + pair plan (no barrier: may run on a stream beside
// the previous batch's backward), then the rest (after that backward on the same rank)
void xbatch_prefetch(XBatch& x, Table* t, const uint64_t* ids, uint64_t n,
                     const uint32_t* offsets, uint32_t B, uint32_t F, cudaStream_t st);
void xbatch_fwd_prefetched(XBatch& x, Table* t, cudaStream_t st);
void xbatch_bwd(XBatch& x, Table* t, const float* grads, float lr, uint32_t step_tag,
                uint32_t epoch, int* accepted, uint32_t flags, cudaStream_t st);
void table_apply_pairs(Table* t, const uint64_t* recv_ids, const uint64_t* recv_versions,
                       const uint64_t* id_counts, const uint32_t* pair_pos, const float* contrib,
                       const uint64_t* pair_counts, uint32_t G, float lr, uint32_t step_tag,
                       uint32_t epoch, int* accepted, uint32_t flags, cudaStream_t st);

}  // namespace hps
