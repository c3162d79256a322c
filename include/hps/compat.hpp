// compat.hpp -- the reference's operator classes over the C ABI (include/hps_c.h).
//
// Header-only C++17 adapters with the shapes of the reference's parameter-server and
// embedding-worker API (/root/reference/proj/include/hybridps), so a caller of that
// API switches by changing the namespace:
//
//   hybridps::PsShard          (embedding_ps.hpp:56-495)        -> hps_b200::PsShard
//   hybridps::ShardSet         (embedding_ps.hpp:504-551)       -> hps_b200::ShardSet
//   hybridps::ps_lookup / ps_apply_gradients (:556-564)         -> same names here
//   hybridps::EmbeddingWorker  (embedding_worker.hpp:470-801)   -> hps_b200::EmbeddingWorker
//                                                                  (sample + batch surfaces)
//
// Errors: every non-OK status is rethrown as the exception type the reference throws for
// it (errors.hpp:28-107); a stale caller epoch returns false as in the reference.
// Rows live in device memory on one GPU; all vectors below are host memory and are
// staged by the library.
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../hps_c.h"

namespace hps_b200 {

// ---- errors (errors.hpp:28-107) -------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define HPS_COMPAT_ERR(name) \
  struct name : Error {      \
    using Error::Error;      \
  };
HPS_COMPAT_ERR(PreconditionError)
HPS_COMPAT_ERR(ConfigError)
HPS_COMPAT_ERR(ProtocolError)
HPS_COMPAT_ERR(TransportError)
HPS_COMPAT_ERR(CheckpointCorruptError)
HPS_COMPAT_ERR(DivergenceError)
HPS_COMPAT_ERR(ConsistencyError)
HPS_COMPAT_ERR(UndefinedMetricError)
HPS_COMPAT_ERR(StaleSampleError)
HPS_COMPAT_ERR(BackpressureError)
HPS_COMPAT_ERR(ClockError)
HPS_COMPAT_ERR(SyncFailureError)
HPS_COMPAT_ERR(UnrecoverableRunError)
HPS_COMPAT_ERR(CudaError)
#undef HPS_COMPAT_ERR

inline void check(hps_status s) {
  if (s == HPS_OK) return;
  std::string m = hps_last_error();
  switch (s) {
    case HPS_E_PRECONDITION: throw PreconditionError(m);
    case HPS_E_CONFIG: throw ConfigError(m);
    case HPS_E_PROTOCOL: throw ProtocolError(m);
    case HPS_E_TRANSPORT: throw TransportError(m);
    case HPS_E_CHECKPOINT_CORRUPT: throw CheckpointCorruptError(m);
    case HPS_E_DIVERGENCE: throw DivergenceError(m);
    case HPS_E_CONSISTENCY: throw ConsistencyError(m);
    case HPS_E_UNDEFINED_METRIC: throw UndefinedMetricError(m);
    case HPS_E_STALE_SAMPLE: throw StaleSampleError(m);
    case HPS_E_BACKPRESSURE: throw BackpressureError(m);
    case HPS_E_CLOCK: throw ClockError(m);
    case HPS_E_SYNC_FAILURE: throw SyncFailureError(m);
    case HPS_E_UNRECOVERABLE: throw UnrecoverableRunError(m);
    default: throw CudaError(m);
  }
}

// ---- core.hpp ------------------------------------------------------------------------
inline uint64_t mix64(uint64_t x) { return hps_mix64(x); }                       // :36-44
inline uint32_t route_shard(uint64_t id, uint32_t s) { return hps_route_shard(id, s); }  // :145-150

struct SampleId {  // core.hpp:98-125: 8-bit rank | 56-bit counter; the apply-order key
  uint64_t raw = 0;
  static SampleId encode(uint32_t rank, uint64_t counter) {
    return SampleId{(static_cast<uint64_t>(rank & 0xffu) << 56) | (counter & ((1ull << 56) - 1))};
  }
  uint32_t rank() const { return static_cast<uint32_t>(raw >> 56); }
  bool operator<(const SampleId& o) const { return raw < o.raw; }
};
using IdFeatures = std::vector<std::vector<uint64_t>>;  // core.hpp:129-131

enum class EmbOptimizer : uint8_t { kAdagrad = 0, kSgd = 1 };  // embedding_ps.hpp:37
enum class Aggregation : uint8_t { kMean = 0, kSum = 1 };      // ModelConfig::Aggregation core.hpp:178
inline constexpr float kAdagradEps = 1e-10f;                   // embedding_ps.hpp:39

struct PsShardConfig {  // embedding_ps.hpp:41-46 (+ the CUDA device)
  uint64_t capacity = 1 << 16;
  uint32_t embedding_dim = 16;
  EmbOptimizer optimizer = EmbOptimizer::kAdagrad;
  uint64_t rng_salt = 0;
  int device = -1;
};

namespace detail {
struct TableDeleter {
  void operator()(hps_table* t) const { hps_table_destroy(t); }
};
struct BatchDeleter {
  void operator()(hps_batch* b) const { hps_batch_destroy(b); }
};
using TablePtr = std::unique_ptr<hps_table, TableDeleter>;
using BatchPtr = std::unique_ptr<hps_batch, BatchDeleter>;

inline TablePtr make_table(const std::vector<uint64_t>& salts, uint64_t capacity, uint32_t D,
                           EmbOptimizer opt, int device) {
  hps_table_cfg c{};
  c.shard_count = static_cast<uint32_t>(salts.size());
  c.shard_salts = salts.data();
  c.capacity = capacity;
  c.embedding_dim = D;
  c.optimizer = opt == EmbOptimizer::kSgd ? HPS_SGD : HPS_ADAGRAD;
  c.device = device;
  c.owner_rank = 0;
  c.world_size = 1;
  c.flags = HPS_TABLE_TAG_RING;  // PsShard's exact count_delay for any step-tag order
  hps_table* t = nullptr;
  check(hps_table_create(&c, &t));
  return TablePtr(t);
}

inline hps_counters counters(hps_table* t) {
  hps_counters c{};
  check(hps_table_counters(t, &c));
  return c;
}
}  // namespace detail

// ---- a table of S logical shards (one GPU) ---------------------------------------------
// Shared by PsShard (S = 1) and ShardSet (S >= 1): rows route to shard mix64(id) % S and
// initialise from that shard's salt, exactly as S separate PsShard objects would.
class Table {
 public:
  Table(std::vector<uint64_t> salts, uint64_t capacity, uint32_t dim, EmbOptimizer opt,
        int device)
      : salts_(std::move(salts)), dim_(dim),
        t_(detail::make_table(salts_, capacity, dim, opt, device)) {}

  uint32_t embedding_dim() const { return dim_; }
  hps_table* handle() const { return t_.get(); }

  // PsShard::lookup (embedding_ps.hpp:105-114): out_values[ids.size() * D].
  void lookup(const std::vector<uint64_t>& ids, float* out_values,
              uint64_t* out_versions = nullptr) {
    std::lock_guard<std::mutex> g(mu_);
    check(hps_lookup(t_.get(), ids.data(), ids.size(), out_values, out_versions, nullptr));
  }
  // PsShard::lookup_map (:117-126) / ShardSet::lookup (:531-541).
  std::map<uint64_t, std::vector<float>> lookup_map(const std::vector<uint64_t>& ids) {
    std::vector<float> v(ids.size() * dim_);
    lookup(ids, v.data());
    std::map<uint64_t, std::vector<float>> out;
    for (size_t i = 0; i < ids.size(); ++i)
      out[ids[i]] = std::vector<float>(v.begin() + i * dim_, v.begin() + (i + 1) * dim_);
    return out;
  }

  struct VersionedGrad {  // embedding_ps.hpp:128-132
    uint64_t id = 0;
    const float* grad = nullptr;
    uint64_t read_version = 0;
  };
  // PsShard::apply_gradients (:139-162): false = stale epoch, whole call dropped.
  bool apply_gradients(const std::vector<VersionedGrad>& grads, float lr, uint32_t step_tag,
                       uint32_t caller_epoch, std::vector<uint32_t>* delays_out) {
    const size_t n = grads.size();
    std::vector<uint64_t> ids(n), rv(n);
    std::vector<float> g(n * dim_);
    for (size_t i = 0; i < n; ++i) {
      ids[i] = grads[i].id;
      rv[i] = grads[i].read_version;
      for (uint32_t d = 0; d < dim_; ++d) g[i * dim_ + d] = grads[i].grad[d];
    }
    if (delays_out) delays_out->assign(n, 0);
    int accepted = 0;
    std::lock_guard<std::mutex> lk(mu_);
    check(hps_apply(t_.get(), ids.data(), g.data(), rv.data(), n, lr, step_tag, caller_epoch,
                    delays_out ? delays_out->data() : nullptr, &accepted, 0, nullptr));
    return accepted != 0;
  }
  // PsShard::apply_gradients_map (:165-189): ascending id order, untracked versions.
  void apply_gradients_map(const std::map<uint64_t, std::vector<float>>& grads, float lr) {
    std::vector<uint64_t> ids;
    std::vector<float> g;
    for (const auto& [id, v] : grads) {
      if (v.size() != dim_) throw PreconditionError("apply_gradients_map: gradient size != dim");
      ids.push_back(id);
      g.insert(g.end(), v.begin(), v.end());
    }
    int accepted = 0;
    std::lock_guard<std::mutex> lk(mu_);
    check(hps_apply(t_.get(), ids.data(), g.data(), nullptr, ids.size(), lr, 0,
                    hps_table_epoch(t_.get()), nullptr, &accepted, 0, nullptr));
  }

  void reset_for_recovery() { check(hps_table_reset(t_.get())); }         // :193-202
  uint32_t advance_epoch() { return hps_table_advance_epoch(t_.get()); }  // :204-207
  uint32_t epoch() const { return hps_table_epoch(t_.get()); }            // :91
  uint64_t miss_count() const { return detail::counters(t_.get()).misses; }            // :79
  uint64_t eviction_count() const { return detail::counters(t_.get()).evictions; }     // :75
  uint64_t clock_reset_count() const { return detail::counters(t_.get()).clock_resets; }  // :83
  uint64_t stale_epoch_drops() const {                                                   // :87
    return detail::counters(t_.get()).stale_epoch_drops;
  }
  uint64_t size() const { return detail::counters(t_.get()).size; }  // :95

 protected:
  std::vector<uint64_t> salts_;
  uint32_t dim_;
  detail::TablePtr t_;
  std::mutex mu_;  // the per-shard lock (embedding_ps.hpp:491)
};

// PsShard(const PsShardConfig&) (embedding_ps.hpp:63): one shard, salt = cfg.rng_salt.
class PsShard : public Table {
 public:
  explicit PsShard(const PsShardConfig& cfg)
      : Table({cfg.rng_salt}, cfg.capacity, cfg.embedding_dim, cfg.optimizer, cfg.device),
        capacity_(cfg.capacity) {}

  // PsShard::save_checkpoint (embedding_ps.hpp:222-260): the HPS1 image, its size.
  size_t save_checkpoint(std::vector<uint8_t>& out) const {
    uint64_t n = 0;
    check(hps_table_checkpoint_save(handle(), 0, capacity_, nullptr, 0, &n));
    out.assign(n, 0);
    check(hps_table_checkpoint_save(handle(), 0, capacity_, out.data(), n, &n));
    return n;
  }
  // recover_from_checkpoint (:280-292): state reverts to the image, the epoch advances
  // past the live one (CheckpointCorruptError on a bad image; nothing changes then).
  void recover_from_checkpoint(const std::vector<uint8_t>& buf) {
    const void* p = buf.data();
    const uint64_t n = buf.size();
    check(hps_table_checkpoint_load(handle(), &p, &n, 1, 1));
  }

 private:
  uint32_t capacity_;
};

// ShardSet(shard_count, base) (embedding_ps.hpp:506-516): shard i salt = mix64(base + i),
// per-shard capacity = base.capacity.
class ShardSet : public Table {
 public:
  ShardSet(uint32_t shard_count, const PsShardConfig& base)
      : Table(salts_for(shard_count, base.rng_salt), uint64_t(base.capacity) * shard_count,
              base.embedding_dim, base.optimizer, base.device),
        shard_count_(shard_count) {}
  uint32_t shard_count() const { return shard_count_; }
  uint32_t shard_of(uint64_t id) const { return route_shard(id, shard_count_); }  // :521-523
  std::map<uint64_t, std::vector<float>> lookup(const std::vector<uint64_t>& ids) {  // :531
    return lookup_map(ids);
  }
  void apply_gradients(const std::map<uint64_t, std::vector<float>>& g, float lr) {  // :543
    apply_gradients_map(g, lr);
  }

 private:
  static std::vector<uint64_t> salts_for(uint32_t n, uint64_t base) {
    if (n == 0) throw ConfigError("ShardSet: shard_count must be positive");
    std::vector<uint64_t> s(n);
    for (uint32_t i = 0; i < n; ++i) s[i] = mix64(base + i);
    return s;
  }
  uint32_t shard_count_;
};

inline std::map<uint64_t, std::vector<float>> ps_lookup(ShardSet& set,
                                                        const std::vector<uint64_t>& ids) {
  return set.lookup(ids);  // embedding_ps.hpp:556-559
}
inline void ps_apply_gradients(ShardSet& set, const std::map<uint64_t, std::vector<float>>& g,
                               float lr) {
  set.apply_gradients(g, lr);  // :561-564
}

// ---- embedding worker (embedding_worker.hpp:470-801) ------------------------------------
struct PullResult {  // embedding_worker.hpp:396-401
  uint32_t group_count = 0;
  uint32_t dim = 0;
  std::vector<float> values;
  std::vector<uint64_t> read_versions;
};

struct EmbeddingWorkerConfig {  // embedding_worker.hpp:449-458 (the fields this path uses)
  uint32_t rank = 0;
  uint32_t group_count = 0;
  uint32_t embedding_dim = 0;
  Aggregation aggregation = Aggregation::kMean;
  bool gated = true;  // stage pushes until flush_step_marker (sync mode)
};

// Sample surface: register_sample / serve_pull / apply_backward / flush_step_marker with
// the reference's meaning. Registered samples are buffered host-side; a flush applies
// every staged push of the step as ONE device batch in ascending SampleId order (the
// gated flush, :777-801), so the per-sample API still runs on the batched kernels.
// Batch surface: register_batch / pull_batch / push_batch over CSR buffers (host or
// device pointers) -- what a batched caller should use.
class EmbeddingWorker {
 public:
  EmbeddingWorker(EmbeddingWorkerConfig cfg, Table& table) : cfg_(cfg), table_(table) {
    hps_batch* b = nullptr;
    check(hps_batch_create(table.handle(), agg(), &b));
    batch_.reset(b);
    if (cfg_.embedding_dim == 0) cfg_.embedding_dim = table.embedding_dim();
  }

  // -- sample surface
  SampleId register_sample(const IdFeatures& ids) {  // :493-521
    if (cfg_.group_count && ids.size() != cfg_.group_count)
      throw PreconditionError("register_sample: group count mismatch");
    std::lock_guard<std::mutex> g(mu_);
    SampleId sid = SampleId::encode(cfg_.rank, next_++);
    samples_[sid.raw] = Staged{ids, {}, {}, false};
    return sid;
  }

  PullResult serve_pull(SampleId sid) {  // :523-571
    std::lock_guard<std::mutex> g(mu_);
    auto it = samples_.find(sid.raw);
    if (it == samples_.end()) throw StaleSampleError("serve_pull: unknown sample");
    std::vector<uint64_t> ids;
    std::vector<uint32_t> offs;
    csr(it->second.ids, ids, offs);
    const uint32_t G = static_cast<uint32_t>(it->second.ids.size());
    PullResult r{G, cfg_.embedding_dim, std::vector<float>(size_t(G) * cfg_.embedding_dim),
                 std::vector<uint64_t>(ids.size())};
    check(hps_pull_batch(table_.handle(), ids.data(), ids.size(), offs.data(), 1, G, agg(),
                         r.values.data(), r.read_versions.data(), nullptr));
    it->second.read_versions = r.read_versions;
    return r;
  }

  // :575-594. Unknown sample = counted drop (not an error), as in the reference.
  void apply_backward(SampleId sid, const std::vector<float>& grads, float lr,
                      uint64_t step = 0, bool has_step = false) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = samples_.find(sid.raw);
    if (it == samples_.end()) {
      ++unknown_drops_;
      return;
    }
    it->second.grads = grads;
    it->second.pushed = true;
    lr_ = lr;
    step_ = has_step ? step : step_;
    if (!cfg_.gated) flush_locked(static_cast<uint32_t>(step_));
  }

  void flush_step_marker(uint64_t step, uint32_t /*nn_rank*/) {  // :599-620 (one NN rank)
    std::lock_guard<std::mutex> g(mu_);
    flush_locked(static_cast<uint32_t>(step));
  }
  void drop_buffer() {
    std::lock_guard<std::mutex> g(mu_);
    samples_.clear();
  }
  uint64_t unknown_sample_drops() const { return unknown_drops_; }

  // -- batch surface (hps_batch_register / pull / push)
  void register_batch(const uint64_t* ids, size_t n, const uint32_t* offsets, uint32_t B,
                      uint32_t F, const uint64_t* sample_keys = nullptr, hps_stream s = nullptr) {
    check(hps_batch_register(batch_.get(), ids, n, offsets, B, F, sample_keys, s));
  }
  void pull_batch(float* out_pooled, uint64_t* out_read_versions = nullptr,
                  hps_stream s = nullptr) {
    check(hps_batch_pull(batch_.get(), out_pooled, out_read_versions, s));
  }
  bool push_batch(const float* grads, float lr, uint32_t step, uint32_t flags = 0,
                  hps_stream s = nullptr) {
    int accepted = 0;
    check(hps_batch_push(batch_.get(), grads, lr, step, table_.epoch(), 0, nullptr, &accepted,
                         flags, s));
    return accepted != 0;
  }

 private:
  struct Staged {
    IdFeatures ids;
    std::vector<float> grads;
    std::vector<uint64_t> read_versions;
    bool pushed;
  };
  int32_t agg() const { return cfg_.aggregation == Aggregation::kSum ? HPS_SUM : HPS_MEAN; }
  static void csr(const IdFeatures& f, std::vector<uint64_t>& ids, std::vector<uint32_t>& offs) {
    offs.push_back(static_cast<uint32_t>(ids.size()));
    for (const auto& g : f) {
      ids.insert(ids.end(), g.begin(), g.end());
      offs.push_back(static_cast<uint32_t>(ids.size()));
    }
  }
  // The gated flush: every pushed sample, ascending SampleId, one batch.
  void flush_locked(uint32_t step) {
    std::vector<uint64_t> keys, ids, rv;
    std::vector<uint32_t> offs{0};
    std::vector<float> grads;
    uint32_t F = 0;
    for (auto it = samples_.begin(); it != samples_.end();) {  // std::map: ascending sid
      if (!it->second.pushed) {
        ++it;
        continue;
      }
      const Staged& s = it->second;
      F = static_cast<uint32_t>(s.ids.size());
      keys.push_back(it->first);
      for (const auto& g : s.ids) {
        ids.insert(ids.end(), g.begin(), g.end());
        offs.push_back(static_cast<uint32_t>(ids.size()));
      }
      rv.insert(rv.end(), s.read_versions.begin(), s.read_versions.end());
      grads.insert(grads.end(), s.grads.begin(), s.grads.end());
      it = samples_.erase(it);
    }
    if (keys.empty()) return;
    int accepted = 0;
    check(hps_push_batch(table_.handle(), ids.data(), ids.size(), offs.data(),
                         static_cast<uint32_t>(keys.size()), F, agg(), grads.data(),
                         rv.size() == ids.size() ? rv.data() : nullptr, keys.data(), lr_, step,
                         table_.epoch(), &accepted, nullptr));
  }

  EmbeddingWorkerConfig cfg_;
  Table& table_;
  detail::BatchPtr batch_;
  std::mutex mu_;
  std::map<uint64_t, Staged> samples_;
  uint64_t next_ = 0;
  uint64_t unknown_drops_ = 0;
  uint64_t step_ = 0;
  float lr_ = 0.0f;
};

}  // namespace hps_b200
