// Internal host-side declarations shared by table.cu / capi.cu / dedup.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
void read_counters(Table* t, cudaStream_t st);
void profile_enable(Table* t, bool on);
void profile_get(Table* t, const char* name, double* ms, uint64_t* count);
void check_flags(Table* t, cudaStream_t st, bool divergence = true);

void batch_reserve(Batch& b, uint64_t N, uint64_t BF, uint64_t B);
void batch_free(Batch& b);
void batch_register(Batch& b, const uint64_t* ids, uint64_t N, const uint32_t* offsets, uint32_t B,
                    uint32_t F, const uint64_t* sample_keys, cudaStream_t st);
void batch_pull(Batch& b, int agg, float* out_pooled, uint64_t* out_rv, cudaStream_t st);
void batch_push(Batch& b, int agg, const float* grads, float lr, uint32_t step_tag,
                uint32_t epoch, int untracked, const uint64_t* rv64, int* accepted,
                uint32_t flags, cudaStream_t st);
uint64_t batch_pairs(Batch& b);

void table_lookup(Table* t, const uint64_t* ids, uint64_t n, float* out_values,
                  uint64_t* out_versions, cudaStream_t st);
void table_peek(Table* t, const uint64_t* ids, uint64_t n, float* out_w, float* out_acc,
                uint64_t* out_versions, uint8_t* out_present, cudaStream_t st);
void table_apply(Table* t, const uint64_t* ids, const float* grads, const uint64_t* rv, uint64_t n,
                 float lr, uint32_t step_tag, uint32_t epoch, uint32_t* out_delays,
                 int* accepted, uint32_t flags, cudaStream_t st);
void route(const uint64_t* ids, uint64_t n, uint32_t S, uint32_t* out, cudaStream_t st);

// dedup.cu
void dedup(const uint64_t* ids, uint64_t n, uint64_t* out_unique, uint32_t* out_inverse,
           uint64_t* out_u, cudaStream_t st);
void compress_indices(const uint64_t* ids, uint64_t n, const uint32_t* offsets, uint32_t B,
                      uint32_t G, uint64_t* group_u_off, uint64_t* unique, uint64_t* post_off,
                      uint16_t* postings, cudaStream_t st);

}  // namespace hps
