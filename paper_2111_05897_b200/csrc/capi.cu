// The C ABI (include/hps_c.h): argument checks, device selection, the per-table
// lock, and mapping of hps::Error / CUDA failures onto hps_status. Nothing here
// throws across the boundary.
#include <cuda_runtime.h>

#include <exception>
#include <mutex>
#include <new>
#include <string>

#include "../../include/hps_c.h"
#include "common.cuh"
#include "table.cuh"
#include "table_impl.h"

struct hps_table {
  hps::Table* impl;
};
struct hps_batch {
  hps::Batch impl;
};
struct hps_exchange {
  hps::XBatch impl;
  std::mutex mu;
};

namespace {

thread_local std::string g_last_error;

template <typename Fn>
hps_status guarded(Fn&& fn) {
  try {
    fn();
    return HPS_OK;
  } catch (const hps::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return HPS_E_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HPS_E_CUDA;
  } catch (...) {
    g_last_error = "unknown failure";
    return HPS_E_CUDA;
  }
}

inline cudaStream_t S(hps_stream s) { return static_cast<cudaStream_t>(s); }

#define REQUIRE(cond, msg) \
  if (!(cond)) throw hps::Error(HPS_E_PRECONDITION, msg)

}  // namespace

extern "C" {

const char* hps_last_error(void) { return g_last_error.c_str(); }
int hps_abi_version(void) { return HPS_ABI_VERSION; }

uint64_t hps_mix64(uint64_t x) { return hps::mix64(x); }

uint32_t hps_route_shard(uint64_t id, uint32_t shard_count) {
  return shard_count ? hps::route_shard(id, shard_count) : 0u;
}

hps_status hps_route(const uint64_t* ids, size_t n, uint32_t shard_count, uint32_t* out_shard,
                     hps_stream stream) {
  return guarded([&] {
    REQUIRE(shard_count > 0, "route_shard: shard_count must be positive");
    REQUIRE(n == 0 || (ids && out_shard), "hps_route: null buffer");
    hps::route(ids, n, shard_count, out_shard, S(stream));
  });
}

hps_status hps_table_create(const hps_table_cfg* cfg, hps_table** out) {
  return guarded([&] {
    REQUIRE(cfg && out, "hps_table_create: null argument");
    *out = nullptr;
    hps::Table* t = hps::table_create(*cfg);
    *out = new hps_table{t};
  });
}

hps_status hps_table_destroy(hps_table* t) {
  return guarded([&] {
    if (!t) return;
    hps::table_destroy(t->impl);
    delete t;
  });
}

hps_status hps_table_counters(hps_table* t, hps_counters* out) {
  return guarded([&] {
    REQUIRE(t && out, "hps_table_counters: null argument");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::table_counters(t->impl, out);
  });
}

hps_status hps_table_sync(hps_table* t) {
  return guarded([&] {
    REQUIRE(t, "hps_table_sync: null table");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::table_sync(t->impl);
  });
}

uint32_t hps_table_epoch(const hps_table* t) { return t ? t->impl->epoch : 0u; }

hps_status hps_table_device_step(hps_table* t, uint32_t* out_step) {
  return guarded([&] {
    REQUIRE(t && out_step, "hps_table_device_step: null argument");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    HPS_CUDA(cudaDeviceSynchronize());
    unsigned long long v = 0;
    HPS_CUDA(cudaMemcpy(&v, t->impl->d.ctr + hps::kCtrStep, sizeof(v), cudaMemcpyDeviceToHost));
    *out_step = static_cast<uint32_t>(v);
  });
}

uint32_t hps_table_advance_epoch(hps_table* t) {
  if (!t) return 0u;
  std::lock_guard<std::mutex> g(t->impl->mu);
  return ++t->impl->epoch;
}

hps_status hps_table_reset(hps_table* t) {
  return guarded([&] {
    REQUIRE(t, "hps_table_reset: null table");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::table_reset(t->impl);
  });
}

hps_status hps_table_checkpoint_save(hps_table* t, uint32_t shard, uint32_t shard_capacity,
                                     void* buf, uint64_t cap, uint64_t* out_bytes) {
  return guarded([&] {
    REQUIRE(t && out_bytes, "hps_table_checkpoint_save: null argument");
    std::lock_guard<std::mutex> g(t->impl->mu);
    *out_bytes = hps::table_ckpt_save(t->impl, shard, shard_capacity,
                                      static_cast<uint8_t*>(buf), cap);
  });
}

hps_status hps_table_checkpoint_load(hps_table* t, const void* const* images,
                                     const uint64_t* sizes, uint32_t count, int recover) {
  return guarded([&] {
    REQUIRE(t && (count == 0 || (images && sizes)), "hps_table_checkpoint_load: null argument");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::table_ckpt_load(t->impl, reinterpret_cast<const uint8_t* const*>(images), sizes, count,
                         recover);
  });
}

hps_status hps_lookup(hps_table* t, const uint64_t* ids, size_t n, float* out_values,
                      uint64_t* out_versions, hps_stream stream) {
  return guarded([&] {
    REQUIRE(t, "hps_lookup: null table");
    REQUIRE(n == 0 || (ids && out_values), "hps_lookup: null buffer");
    if (n == 0) return;
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    hps::table_lookup(t->impl, ids, n, out_values, out_versions, S(stream));
  });
}

hps_status hps_table_gather(hps_table* t, const uint64_t* ids, size_t n, float* out_values,
                            uint64_t* out_versions, uint32_t flags, hps_stream stream) {
  return guarded([&] {
    REQUIRE(t && (n == 0 || (ids && out_values)), "hps_table_gather: null argument");
    if (n == 0) return;
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    hps::table_lookup(t->impl, ids, n, out_values, out_versions, S(stream), flags);
  });
}

hps_status hps_apply(hps_table* t, const uint64_t* ids, const float* grads,
                     const uint64_t* read_versions, size_t n, float lr, uint32_t step_tag,
                     uint32_t epoch, uint32_t* out_delays, int* accepted, uint32_t flags,
                     hps_stream stream) {
  return guarded([&] {
    REQUIRE(t, "hps_apply: null table");
    REQUIRE(n == 0 || (ids && grads), "hps_apply: null buffer");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    if (n == 0) {
      if (accepted) *accepted = epoch == t->impl->epoch;
      return;
    }
    hps::table_apply(t->impl, ids, grads, read_versions, n, lr, step_tag, epoch, out_delays,
                     accepted, flags, S(stream));
  });
}

hps_status hps_peek(hps_table* t, const uint64_t* ids, size_t n, float* out_w, float* out_acc,
                    uint64_t* out_versions, uint8_t* out_present, hps_stream stream) {
  return guarded([&] {
    REQUIRE(t, "hps_peek: null table");
    REQUIRE(n == 0 || ids, "hps_peek: null ids");
    if (n == 0) return;
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    hps::table_peek(t->impl, ids, n, out_w, out_acc, out_versions, out_present, S(stream));
  });
}

hps_status hps_batch_create(hps_table* t, int32_t aggregation, hps_batch** out) {
  return guarded([&] {
    REQUIRE(t && out, "hps_batch_create: null argument");
    REQUIRE(aggregation == HPS_MEAN || aggregation == HPS_SUM, "hps_batch_create: bad aggregation");
    *out = new hps_batch();
    (*out)->impl.table = t->impl;
    (*out)->impl.agg = aggregation;
  });
}

hps_status hps_batch_destroy(hps_batch* b) {
  return guarded([&] {
    if (!b) return;
    {
      hps::DeviceGuard dg(b->impl.table->device);
      cudaDeviceSynchronize();
      hps::batch_free(b->impl);
    }
    delete b;
  });
}

hps_status hps_batch_register(hps_batch* b, const uint64_t* ids, size_t n_ids,
                              const uint32_t* offsets, uint32_t B, uint32_t F,
                              const uint64_t* sample_keys, hps_stream stream) {
  return guarded([&] {
    REQUIRE(b, "hps_batch_register: null batch");
    REQUIRE(offsets, "hps_batch_register: null offsets");
    REQUIRE(n_ids == 0 || ids, "hps_batch_register: null ids");
    hps::Table* t = b->impl.table;
    std::lock_guard<std::mutex> g(t->mu);
    hps::DeviceGuard dg(t->device);
    hps::batch_register(b->impl, ids, n_ids, offsets, B, F, sample_keys, S(stream));
  });
}

hps_status hps_batch_defer_plan_join(hps_batch* b, int on) {
  return guarded([&] {
    REQUIRE(b, "hps_batch_defer_plan_join: null batch");
    b->impl.defer_join = on != 0;
  });
}

hps_status hps_batch_join_plan(hps_batch* b, hps_stream stream) {
  return guarded([&] {
    REQUIRE(b, "hps_batch_join_plan: null batch");
    hps::Table* t = b->impl.table;
    std::lock_guard<std::mutex> g(t->mu);
    hps::DeviceGuard dg(t->device);
    hps::batch_join_plan(b->impl, S(stream));
  });
}

hps_status hps_batch_pull(hps_batch* b, float* out_pooled, uint64_t* out_read_versions,
                          hps_stream stream) {
  return guarded([&] {
    REQUIRE(b, "hps_batch_pull: null batch");
    REQUIRE(out_pooled || b->impl.B == 0, "hps_batch_pull: null output");
    hps::Table* t = b->impl.table;
    std::lock_guard<std::mutex> g(t->mu);
    hps::DeviceGuard dg(t->device);
    hps::batch_pull(b->impl, b->impl.agg, out_pooled, out_read_versions, S(stream));
  });
}

hps_status hps_batch_push(hps_batch* b, const float* grads, float lr, uint32_t step_tag,
                          uint32_t epoch, int untracked, uint32_t* out_delays, int* accepted,
                          uint32_t flags, hps_stream stream) {
  return guarded([&] {
    REQUIRE(b, "hps_batch_push: null batch");
    // per-(sample, id) delays of a batch push land in the table's delay histogram
    // (hps_counters.delay_hist, StalenessStats::record_delay staleness.hpp:42-49); per-entry
    // delays are hps_apply's
    REQUIRE(!out_delays, "hps_batch_push: out_delays must be NULL (delays are recorded in "
                         "hps_counters.delay_hist; hps_apply returns per-entry delays)");
    REQUIRE(grads || b->impl.B == 0, "hps_batch_push: null gradients");
    hps::Table* t = b->impl.table;
    std::lock_guard<std::mutex> g(t->mu);
    hps::DeviceGuard dg(t->device);
    hps::batch_push(b->impl, b->impl.agg, grads, lr, step_tag, epoch, untracked,
                    nullptr, accepted, flags, S(stream));
  });
}

hps_status hps_batch_pairs(hps_batch* b, uint64_t* out_pairs) {
  return guarded([&] {
    REQUIRE(b && out_pairs, "hps_batch_pairs: null argument");
    hps::Table* t = b->impl.table;
    std::lock_guard<std::mutex> g(t->mu);
    hps::DeviceGuard dg(t->device);
    *out_pairs = hps::batch_pairs(b->impl);
  });
}

hps_status hps_pull_batch(hps_table* t, const uint64_t* ids, size_t n_ids, const uint32_t* offsets,
                          uint32_t B, uint32_t F, int32_t aggregation, float* out_pooled,
                          uint64_t* out_read_versions, hps_stream stream) {
  return guarded([&] {
    REQUIRE(t && offsets, "hps_pull_batch: null argument");
    REQUIRE(aggregation == HPS_MEAN || aggregation == HPS_SUM, "hps_pull_batch: bad aggregation");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    hps::Batch& b = t->impl->scratch;
    b.agg = aggregation;
    hps::batch_register(b, ids, n_ids, offsets, B, F, nullptr, S(stream));
    hps::batch_pull(b, aggregation, out_pooled, out_read_versions, S(stream));
  });
}

hps_status hps_push_batch(hps_table* t, const uint64_t* ids, size_t n_ids, const uint32_t* offsets,
                          uint32_t B, uint32_t F, int32_t aggregation, const float* grads,
                          const uint64_t* read_versions, const uint64_t* sample_keys, float lr,
                          uint32_t step_tag, uint32_t epoch, int* accepted, hps_stream stream) {
  return guarded([&] {
    REQUIRE(t && offsets, "hps_push_batch: null argument");
    REQUIRE(aggregation == HPS_MEAN || aggregation == HPS_SUM, "hps_push_batch: bad aggregation");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    hps::Batch& b = t->impl->scratch;
    b.agg = aggregation;
    hps::batch_register(b, ids, n_ids, offsets, B, F, sample_keys, S(stream));
    hps::batch_push(b, aggregation, grads, lr, step_tag, epoch, read_versions ? 0 : 1,
                    read_versions, accepted, 0, S(stream));
  });
}

hps_status hps_exchange_create(uint32_t world_size, uint32_t shard_count, int32_t aggregation,
                               int32_t device, hps_exchange** out) {
  return guarded([&] {
    REQUIRE(out, "hps_exchange_create: null out");
    REQUIRE(world_size >= 1 && world_size <= hps::kMaxWorld,
            "hps_exchange_create: world_size must be in [1, 32]");
    if (shard_count == 0) throw hps::Error(HPS_E_CONFIG, "hps_exchange_create: shard_count must be positive");
    REQUIRE(aggregation == HPS_MEAN || aggregation == HPS_SUM, "hps_exchange_create: bad aggregation");
    int dev = device;
    if (dev < 0) HPS_CUDA(cudaGetDevice(&dev));
    auto* x = new hps_exchange();
    x->impl.device = dev;
    x->impl.G = world_size;
    x->impl.S = shard_count;
    x->impl.agg = aggregation;
    try {
      hps::xbatch_init(x->impl);
    } catch (...) {
      delete x;
      throw;
    }
    *out = x;
  });
}

hps_status hps_exchange_destroy(hps_exchange* x) {
  return guarded([&] { delete x; });
}

hps_status hps_exchange_route(hps_exchange* x, const uint64_t* ids, size_t n_ids,
                              const uint32_t* offsets, uint32_t B, uint32_t F,
                              uint64_t* out_send_ids, uint64_t* out_counts, hps_stream stream) {
  return guarded([&] {
    REQUIRE(x && offsets && out_counts && (ids || n_ids == 0) && (out_send_ids || n_ids == 0),
            "hps_exchange_route: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_route(x->impl, ids, n_ids, offsets, B, F, out_send_ids, out_counts, S(stream));
  });
}

hps_status hps_exchange_pool(hps_exchange* x, const float* rows, uint32_t dim, float* out_pooled,
                             hps_stream stream) {
  return guarded([&] {
    REQUIRE(x && (out_pooled || !rows), "hps_exchange_pool: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_pool(x->impl, rows, dim, out_pooled, S(stream));
  });
}

hps_status hps_exchange_pairs(hps_exchange* x, const float* grads, uint32_t dim,
                              uint32_t* out_pair_pos, float* out_contrib,
                              uint64_t* out_pair_counts, hps_stream stream) {
  return guarded([&] {
    REQUIRE(x && out_pair_counts, "hps_exchange_pairs: null argument");
    REQUIRE(x->impl.N == 0 || (grads && out_pair_pos && out_contrib),
            "hps_exchange_pairs: null buffer");
    std::lock_guard<std::mutex> g(x->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_pairs(x->impl, grads, dim, out_pair_pos, out_contrib, out_pair_counts, S(stream));
  });
}

hps_status hps_table_apply_pairs(hps_table* t, const uint64_t* recv_ids,
                                 const uint64_t* recv_versions, const uint64_t* id_counts,
                                 const uint32_t* pair_pos, const float* contrib,
                                 const uint64_t* pair_counts, uint32_t world, float lr,
                                 uint32_t step_tag, uint32_t epoch, int* accepted,
                                 uint32_t flags, hps_stream stream) {
  return guarded([&] {
    REQUIRE(t && id_counts && pair_counts, "hps_table_apply_pairs: null argument");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    hps::table_apply_pairs(t->impl, recv_ids, recv_versions, id_counts, pair_pos, contrib,
                           pair_counts, world, lr, step_tag, epoch, accepted, flags, S(stream));
  });
}

hps_status hps_exchange_set_codec(hps_exchange* x, float kappa) {
  return guarded([&] {
    REQUIRE(x, "hps_exchange_set_codec: null exchange");
    std::lock_guard<std::mutex> g(x->mu);
    hps::xbatch_set_codec(x->impl, kappa);
  });
}

hps_status hps_exchange_arena(hps_exchange* x, uint64_t max_ids, uint64_t max_groups,
                              uint32_t dim, void* out_handle) {
  return guarded([&] {
    REQUIRE(x && out_handle, "hps_exchange_arena: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_arena(x->impl, max_ids, max_groups, dim, out_handle);
  });
}

hps_status hps_exchange_pooled(hps_exchange* x, float** out) {
  return guarded([&] {
    REQUIRE(x && out, "hps_exchange_pooled: null argument");
    REQUIRE(x->impl.arena, "hps_exchange_pooled: no arena");
    *out = reinterpret_cast<float*>(x->impl.arena + x->impl.off_pooled);
  });
}

hps_status hps_exchange_connect(hps_exchange* x, uint32_t rank, const void* handles) {
  return guarded([&] {
    REQUIRE(x && handles, "hps_exchange_connect: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_connect(x->impl, rank, handles);
  });
}

hps_status hps_exchange_forward(hps_exchange* x, hps_table* t, const uint64_t* ids, size_t n_ids,
                                const uint32_t* offsets, uint32_t B, uint32_t F,
                                hps_stream stream) {
  return guarded([&] {
    REQUIRE(x && t && offsets && (ids || n_ids == 0), "hps_exchange_forward: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    std::lock_guard<std::mutex> g2(t->impl->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_fwd(x->impl, t->impl, ids, n_ids, offsets, B, F, S(stream));
  });
}

hps_status hps_exchange_prefetch(hps_exchange* x, hps_table* t, const uint64_t* ids, size_t n_ids,
                                 const uint32_t* offsets, uint32_t B, uint32_t F,
                                 hps_stream stream) {
  return guarded([&] {
    REQUIRE(x && t && offsets && (ids || n_ids == 0), "hps_exchange_prefetch: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    std::lock_guard<std::mutex> g2(t->impl->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_prefetch(x->impl, t->impl, ids, n_ids, offsets, B, F, S(stream));
  });
}

hps_status hps_exchange_forward_prefetched(hps_exchange* x, hps_table* t, hps_stream stream) {
  return guarded([&] {
    REQUIRE(x && t, "hps_exchange_forward_prefetched: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    std::lock_guard<std::mutex> g2(t->impl->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_fwd_prefetched(x->impl, t->impl, S(stream));
  });
}

hps_status hps_exchange_backward(hps_exchange* x, hps_table* t, const float* grads, float lr,
                                 uint32_t step_tag, uint32_t epoch, int* accepted,
                                 uint32_t flags, hps_stream stream) {
  return guarded([&] {
    REQUIRE(x && t && (grads || x->impl.N == 0), "hps_exchange_backward: null argument");
    std::lock_guard<std::mutex> g(x->mu);
    std::lock_guard<std::mutex> g2(t->impl->mu);
    hps::DeviceGuard dg(x->impl.device);
    hps::xbatch_bwd(x->impl, t->impl, grads, lr, step_tag, epoch, accepted, flags, S(stream));
  });
}

uint64_t hps_launch_count(void) { return hps::g_launches.load(); }

hps_status hps_profile_enable(hps_table* t, int enable) {
  return guarded([&] {
    REQUIRE(t, "hps_profile_enable: null table");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::profile_enable(t->impl, enable != 0);
  });
}

hps_status hps_profile_get(hps_table* t, const char* region, double* total_ms, uint64_t* count) {
  return guarded([&] {
    REQUIRE(t && region && total_ms && count, "hps_profile_get: null argument");
    std::lock_guard<std::mutex> g(t->impl->mu);
    hps::DeviceGuard dg(t->impl->device);
    hps::profile_get(t->impl, region, total_ms, count);
  });
}

hps_status hps_dedup(const uint64_t* ids, size_t n, uint64_t* out_unique, uint32_t* out_inverse,
                     uint64_t* out_u, hps_stream stream) {
  return guarded([&] {
    REQUIRE(n == 0 || (ids && out_unique && out_inverse), "hps_dedup: null buffer");
    hps::dedup(ids, n, out_unique, out_inverse, out_u, S(stream));
  });
}

hps_status hps_compress_values(const float* values, uint64_t rows, uint32_t block_len,
                               float kappa, float* out_scales, uint16_t* out_payload,
                               hps_stream stream) {
  return guarded([&] {
    REQUIRE(rows == 0 || block_len == 0 || (values && out_scales && out_payload),
            "hps_compress_values: null buffer");
    hps::compress_values(values, rows, block_len, kappa, out_scales, out_payload, S(stream));
  });
}

hps_status hps_decompress_values(const float* scales, const uint16_t* payload, uint64_t rows,
                                 uint32_t block_len, float* out, hps_stream stream) {
  return guarded([&] {
    REQUIRE(rows == 0 || block_len == 0 || (scales && payload && out),
            "hps_decompress_values: null buffer");
    hps::decompress_values(scales, payload, rows, block_len, out, S(stream));
  });
}

hps_status hps_compress_indices(const uint64_t* ids, size_t n_ids, const uint32_t* offsets,
                                uint32_t B, uint32_t G, uint64_t* group_u_off, uint64_t* unique,
                                uint64_t* post_off, uint16_t* postings, hps_stream stream) {
  return guarded([&] {
    REQUIRE(offsets && group_u_off && unique && post_off && postings,
            "hps_compress_indices: null buffer");
    hps::compress_indices(ids, n_ids, offsets, B, G, group_u_off, unique, post_off, postings,
                          S(stream));
  });
}

}  // extern "C"
