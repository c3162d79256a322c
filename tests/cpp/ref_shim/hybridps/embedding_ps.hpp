// TEST INFRASTRUCTURE: the reference's parameter-server header (embedding_ps.hpp) restated
// over the C ABI (include/hps_c.h), so the reference's own test source
// /root/reference/proj/tests/test_embedding_ps.cpp compiles UNMODIFIED against the device
// table: this directory comes first on the include path and shadows
// hybridps/embedding_ps.hpp, while hybridps/core.hpp and hybridps/errors.hpp (mixer, Rng,
// exception types) are the reference's own.
//
// Every PsShard is one device table with one logical shard of the configured capacity
// (HPS_TABLE_LRU: LruStore eviction) and the tag ring (HPS_TABLE_TAG_RING: exact
// count_delay); calls are synchronous. Class, member and error semantics follow
// embedding_ps.hpp:37-566; every member forwards to the ABI entry point noted.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "hps_c.h"
#include "hybridps/core.hpp"
#include "hybridps/errors.hpp"

namespace hybridps {

enum class EmbOptimizer : uint8_t { kAdagrad = 0, kSgd = 1 };  // embedding_ps.hpp:37
inline constexpr float kAdagradEps = 1e-10f;                   // :39

struct PsShardConfig {  // :41-46
  uint32_t capacity = 1 << 16;
  uint32_t embedding_dim = 16;
  EmbOptimizer optimizer = EmbOptimizer::kAdagrad;
  uint64_t rng_salt = 0;
};

namespace shim {
[[noreturn]] inline void raise(hps_status s) {
  const std::string m = hps_last_error();
  switch (s) {
    case HPS_E_PRECONDITION: throw PreconditionError(m);
    case HPS_E_CONFIG: throw ConfigError(m);
    case HPS_E_PROTOCOL: throw ProtocolError(m);
    case HPS_E_CHECKPOINT_CORRUPT: throw CheckpointCorruptError(m);
    case HPS_E_DIVERGENCE: throw DivergenceError(m);
    case HPS_E_STALE_SAMPLE: throw StaleSampleError(m);
    case HPS_E_CLOCK: throw ClockError(m);
    case HPS_E_SYNC_FAILURE: throw SyncFailureError(m);
    default: throw Error(m);
  }
}
inline void check(hps_status s) {
  if (s != HPS_OK) raise(s);
}
template <typename T>
T rd(const uint8_t* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}
}  // namespace shim

class PsShard {
 public:
  static constexpr uint32_t kTagRing = 16;
  static constexpr uint32_t kNoStep = 0xffffffffu;
  static constexpr size_t kHeaderBytes = 64;

  struct VersionedGrad {  // :128-132
    uint64_t id = 0;
    const float* grad = nullptr;
    uint64_t read_version = 0;
  };

  explicit PsShard(const PsShardConfig& cfg) : cfg_(cfg) {
    if (cfg.embedding_dim == 0) throw ConfigError("PsShard: embedding_dim must be positive");
    if (cfg.capacity == 0 || cfg.capacity >= 0xffffffffu)
      throw ConfigError("LruStore: capacity must be in [1, 2^32-2]");
    hps_table_cfg c{};
    c.shard_count = 1;
    c.shard_salts = &cfg_.rng_salt;
    c.embedding_dim = cfg.embedding_dim;
    c.optimizer = cfg.optimizer == EmbOptimizer::kSgd ? HPS_SGD : HPS_ADAGRAD;
    c.device = -1;
    c.world_size = 1;
    c.flags = HPS_TABLE_LRU | HPS_TABLE_TAG_RING;
    c.shard_capacity = cfg.capacity;
    shim::check(hps_table_create(&c, &t_));
  }
  ~PsShard() { hps_table_destroy(t_); }
  PsShard(const PsShard&) = delete;
  PsShard& operator=(const PsShard&) = delete;

  uint32_t embedding_dim() const { return cfg_.embedding_dim; }
  uint32_t capacity() const { return cfg_.capacity; }
  EmbOptimizer optimizer() const { return cfg_.optimizer; }
  uint64_t rng_salt() const { return cfg_.rng_salt; }
  uint64_t eviction_count() const { return counters().evictions; }
  uint64_t miss_count() const { return counters().misses; }
  uint64_t clock_reset_count() const { return counters().clock_resets; }
  uint64_t stale_epoch_drops() const { return counters().stale_epoch_drops; }
  uint32_t epoch() const { return hps_table_epoch(t_); }
  uint32_t size() const { return static_cast<uint32_t>(counters().size); }

  // hps_lookup (:105-114)
  void lookup(const std::vector<uint64_t>& ids, float* out_values,
              uint64_t* out_versions = nullptr) {
    std::vector<uint64_t> v(ids.size());
    shim::check(hps_lookup(t_, ids.data(), ids.size(), out_values, v.data(), nullptr));
    if (out_versions) std::memcpy(out_versions, v.data(), v.size() * sizeof(uint64_t));
  }
  std::map<uint64_t, std::vector<float>> lookup_map(const std::vector<uint64_t>& ids) {
    std::vector<float> buf(ids.size() * cfg_.embedding_dim);
    lookup(ids, buf.data());
    std::map<uint64_t, std::vector<float>> out;
    for (size_t i = 0; i < ids.size(); ++i)
      out[ids[i]] = std::vector<float>(buf.begin() + i * cfg_.embedding_dim,
                                       buf.begin() + (i + 1) * cfg_.embedding_dim);
    return out;
  }

  // hps_apply, tracked (:139-162)
  bool apply_gradients(const std::vector<VersionedGrad>& grads, float lr, uint32_t step_tag,
                       uint32_t caller_epoch, std::vector<uint32_t>* delays_out) {
    const size_t n = grads.size(), D = cfg_.embedding_dim;
    std::vector<uint64_t> ids(n), rv(n);
    std::vector<float> g(n * D);
    for (size_t i = 0; i < n; ++i) {
      ids[i] = grads[i].id;
      rv[i] = grads[i].read_version;
      std::memcpy(&g[i * D], grads[i].grad, D * sizeof(float));
    }
    std::vector<uint32_t> dl(n);
    int accepted = 0;
    shim::check(hps_apply(t_, ids.data(), g.data(), rv.data(), n, lr, step_tag, caller_epoch,
                          dl.data(), &accepted, 0, nullptr));
    if (!accepted) return false;
    if (delays_out) *delays_out = dl;
    return true;
  }

  // hps_apply, untracked (:165-189)
  void apply_gradients_map(const std::map<uint64_t, std::vector<float>>& grads, float lr) {
    const size_t D = cfg_.embedding_dim;
    std::vector<uint64_t> ids;
    std::vector<float> g;
    for (const auto& [id, vec] : grads) {
      if (vec.size() != D)
        throw PreconditionError("apply_gradients: gradient width mismatch for id " +
                                std::to_string(id));
      ids.push_back(id);
      g.insert(g.end(), vec.begin(), vec.end());
    }
    int accepted = 0;
    shim::check(hps_apply(t_, ids.data(), g.data(), nullptr, ids.size(), lr, 0, epoch(),
                          nullptr, &accepted, 0, nullptr));
  }

  void reset_for_recovery() { shim::check(hps_table_reset(t_)); }  // :193
  uint32_t advance_epoch() { return hps_table_advance_epoch(t_); }  // :204

  // hps_table_checkpoint_save / _load (HPS1 images, :211-402)
  size_t save_checkpoint(std::vector<uint8_t>& out) const {
    uint64_t n = 0;
    shim::check(hps_table_checkpoint_save(t_, 0, 0, nullptr, 0, &n));
    out.assign(n, 0);
    shim::check(hps_table_checkpoint_save(t_, 0, 0, out.data(), n, &n));
    return n;
  }
  size_t save_checkpoint_file(const std::string& path) const {
    std::vector<uint8_t> buf;
    save_checkpoint(buf);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw Error("save_checkpoint: cannot open " + path);
    f.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
    if (!f) throw Error("save_checkpoint: write failed for " + path);
    return buf.size();
  }
  static std::unique_ptr<PsShard> load_checkpoint(const std::vector<uint8_t>& buf) {
    auto s = std::make_unique<PsShard>(config_of(buf));
    s->adopt(buf, 0);
    return s;
  }
  static std::unique_ptr<PsShard> load_checkpoint_file(const std::string& path) {
    return load_checkpoint(read_file(path));
  }
  void recover_from_checkpoint(const std::vector<uint8_t>& buf) {
    const PsShardConfig c = config_of(buf);
    if (c.embedding_dim != cfg_.embedding_dim || c.capacity != cfg_.capacity ||
        c.optimizer != cfg_.optimizer || c.rng_salt != cfg_.rng_salt)
      throw CheckpointCorruptError("recover_from_checkpoint: configuration mismatch");
    adopt(buf, 1);
  }
  void recover_from_checkpoint_file(const std::string& path) {
    recover_from_checkpoint(read_file(path));
  }

  // LruStore::for_each_mru_to_lru (lru_store.hpp:132-136): the image's recency chain
  std::vector<uint64_t> recency_ids() const {
    std::vector<uint8_t> im;
    save_checkpoint(im);
    const uint32_t hwm = shim::rd<uint32_t>(&im[24]);
    uint32_t s = shim::rd<uint32_t>(&im[28]);
    std::vector<uint64_t> out;
    const uint8_t* ids = im.data() + kHeaderBytes;
    const uint8_t* next = ids + 12ull * hwm;
    while (s != 0xffffffffu && out.size() < hwm) {
      out.push_back(shim::rd<uint64_t>(ids + 8ull * s));
      s = shim::rd<uint32_t>(next + 4ull * s);
    }
    return out;
  }

 private:
  hps_counters counters() const {
    hps_counters c{};
    shim::check(hps_table_counters(t_, &c));
    return c;
  }
  // The configuration an image carries (a corrupt image is refused by the load itself;
  // the header fields are only trusted once its checksum holds).
  static PsShardConfig config_of(const std::vector<uint8_t>& b) {
    if (b.size() < kHeaderBytes) throw CheckpointCorruptError("load_checkpoint: truncated header");
    uint64_t h = 0xcbf29ce484222325ULL;  // fnv1a64 core.hpp:187, checksum field zeroed
    for (size_t i = 0; i < b.size(); ++i) {
      h ^= (i >= 56 && i < 64) ? 0 : b[i];
      h *= 0x100000001b3ULL;
    }
    if (std::memcmp(b.data(), "HPS1", 4) != 0) throw CheckpointCorruptError("load_checkpoint: bad magic");
    if (h != shim::rd<uint64_t>(&b[56])) throw CheckpointCorruptError("load_checkpoint: checksum mismatch");
    if (b[5] > 1) throw CheckpointCorruptError("load_checkpoint: unknown optimizer kind");
    PsShardConfig c;
    c.optimizer = b[5] ? EmbOptimizer::kSgd : EmbOptimizer::kAdagrad;
    c.embedding_dim = shim::rd<uint32_t>(&b[8]);
    c.capacity = shim::rd<uint32_t>(&b[12]);
    c.rng_salt = shim::rd<uint64_t>(&b[16]);
    if (c.embedding_dim == 0 || c.capacity == 0)
      throw CheckpointCorruptError("load_checkpoint: degenerate dimensions");
    return c;
  }
  void adopt(const std::vector<uint8_t>& buf, int recover) {
    const void* im = buf.data();
    const uint64_t n = buf.size();
    shim::check(hps_table_checkpoint_load(t_, &im, &n, 1, recover));
  }
  static std::vector<uint8_t> read_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw Error("load_checkpoint: cannot open " + path);
    return std::vector<uint8_t>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  }

  PsShardConfig cfg_;
  hps_table* t_ = nullptr;
};

// :504-551
class ShardSet {
 public:
  ShardSet(uint32_t shard_count, const PsShardConfig& base) {
    if (shard_count == 0) throw ConfigError("ShardSet: shard_count must be positive");
    for (uint32_t i = 0; i < shard_count; ++i) {
      PsShardConfig cfg = base;
      cfg.rng_salt = mix64(base.rng_salt + i);
      shards_.push_back(std::make_unique<PsShard>(cfg));
    }
  }
  uint32_t shard_count() const { return static_cast<uint32_t>(shards_.size()); }
  PsShard& shard(uint32_t i) { return *shards_[i]; }
  const PsShard& shard(uint32_t i) const { return *shards_[i]; }
  uint32_t shard_of(uint64_t id) const {
    return hps_route_shard(id, static_cast<uint32_t>(shards_.size()));
  }
  uint64_t eviction_count() const {
    uint64_t n = 0;
    for (const auto& s : shards_) n += s->eviction_count();
    return n;
  }
  std::map<uint64_t, std::vector<float>> lookup(const std::vector<uint64_t>& ids) {
    std::vector<std::vector<uint64_t>> by(shards_.size());
    for (uint64_t id : ids) by[shard_of(id)].push_back(id);
    std::map<uint64_t, std::vector<float>> out;
    for (size_t s = 0; s < shards_.size(); ++s)
      if (!by[s].empty()) out.merge(shards_[s]->lookup_map(by[s]));
    return out;
  }
  void apply_gradients(const std::map<uint64_t, std::vector<float>>& grads, float lr) {
    std::vector<std::map<uint64_t, std::vector<float>>> by(shards_.size());
    for (const auto& [id, g] : grads) by[shard_of(id)][id] = g;
    for (size_t s = 0; s < shards_.size(); ++s)
      if (!by[s].empty()) shards_[s]->apply_gradients_map(by[s], lr);
  }

 private:
  std::vector<std::unique_ptr<PsShard>> shards_;
};

inline std::map<uint64_t, std::vector<float>> ps_lookup(ShardSet& set,
                                                        const std::vector<uint64_t>& ids) {
  return set.lookup(ids);
}
inline void ps_apply_gradients(ShardSet& set, const std::map<uint64_t, std::vector<float>>& grads,
                               float lr) {
  set.apply_gradients(grads, lr);
}

}  // namespace hybridps
