// Reference driver: the UNMODIFIED reference headers (/root/reference/proj/include)
// behind a small C ABI so Python tests and bench.py's reference arm can run the
// reference's own CPU path on the same arrays as the GPU path.
//
// TEST INFRASTRUCTURE / ORACLE ONLY. Built by oracle/Makefile into
// oracle/_ref/libhps_ref.so. Only tests/, __graft_entry__.smoke() and bench.py's
// reference / cpu_baseline legs may load it.
//
// What it drives (sync / staleness-0 order):
//   * S PsShard (embedding_ps.hpp:56) behind PsShardService (embedding_worker.hpp:185)
//     on a LocalHub (transport.hpp:70), per-shard salts supplied by the caller;
//   * E EmbeddingWorker (embedding_worker.hpp:470); sample i -> EW i % E
//     (data.hpp:384-413 round-robin), SampleId = rank<<56 | counter (core.hpp:98-125);
//   * pull: serve_pull for every sample (optionally from T threads, as the
//     orchestrator's pull pool does, orchestrator.hpp:623-625);
//   * push: apply_backward in ascending SampleId order (the gated flush order,
//     embedding_worker.hpp:788-800 + ladder :298-341).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "hybridps/codec.hpp"
#include "hybridps/core.hpp"
#include "hybridps/dense_nn.hpp"
#include "hybridps/embedding_ps.hpp"
#include "hybridps/embedding_worker.hpp"
#include "hybridps/errors.hpp"
#include "hybridps/nn_worker.hpp"
#include "hybridps/transport.hpp"

using namespace hybridps;

namespace {

thread_local std::string g_err;

// Same numbering as include/hps_c.h (hps_status), 1:1 with errors.hpp.
int map_exception(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const PreconditionError*>(&e)) return 1;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const ProtocolError*>(&e)) return 3;
  if (dynamic_cast<const TransportError*>(&e)) return 4;
  if (dynamic_cast<const CheckpointCorruptError*>(&e)) return 5;
  if (dynamic_cast<const DivergenceError*>(&e)) return 6;
  if (dynamic_cast<const ConsistencyError*>(&e)) return 7;
  if (dynamic_cast<const UndefinedMetricError*>(&e)) return 8;
  if (dynamic_cast<const StaleSampleError*>(&e)) return 9;
  if (dynamic_cast<const BackpressureError*>(&e)) return 10;
  if (dynamic_cast<const ClockError*>(&e)) return 11;
  if (dynamic_cast<const SyncFailureError*>(&e)) return 12;
  if (dynamic_cast<const UnrecoverableRunError*>(&e)) return 13;
  return 99;
}

struct RefTable {
  uint32_t S = 0, D = 0, F = 0, E = 1;
  ModelConfig::Aggregation agg = ModelConfig::Aggregation::kMean;
  std::vector<std::unique_ptr<PsShard>> shards;
  LocalHub hub;
  std::vector<std::shared_ptr<Endpoint>> eps;
  std::vector<std::unique_ptr<EmbeddingWorker>> ews;
  std::vector<SampleId> sids;  // last pulled batch, batch order
};

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
uint64_t ref_mix64(uint64_t x) { return mix64(x); }
uint32_t ref_route_shard(uint64_t id, uint32_t s) { return s ? route_shard(id, s) : 0u; }

// opt: 0 Adagrad, 1 SGD (EmbOptimizer). agg: 0 mean, 1 sum (Aggregation).
// compress: PS pull replies and EW push frames carry compress_values blocks
// (PsShardService(shard, true), EmbeddingWorkerConfig::compress_values).
void* ref_table_create(uint32_t S, const uint64_t* salts, uint32_t capacity, uint32_t D, int opt,
                       int agg, uint32_t F, uint32_t E, uint64_t ew_buffer, int compress) {
  RefTable* t = nullptr;
  int rc = guarded([&] {
    auto tab = std::make_unique<RefTable>();
    tab->S = S;
    tab->D = D;
    tab->F = F;
    tab->E = E ? E : 1;
    tab->agg = agg ? ModelConfig::Aggregation::kSum : ModelConfig::Aggregation::kMean;
    for (uint32_t s = 0; s < S; ++s) {
      PsShardConfig c;
      c.capacity = capacity;
      c.embedding_dim = D;
      c.optimizer = opt ? EmbOptimizer::kSgd : EmbOptimizer::kAdagrad;
      c.rng_salt = salts[s];
      tab->shards.push_back(std::make_unique<PsShard>(c));
      std::string name = "ps" + std::to_string(s);
      tab->hub.serve(name, PsShardService(*tab->shards[s], compress != 0));
      tab->eps.push_back(tab->hub.endpoint(name));
    }
    for (uint32_t r = 0; r < tab->E; ++r) {
      EmbeddingWorkerConfig ec;
      ec.rank = r;
      ec.group_count = F;
      ec.embedding_dim = D;
      ec.aggregation = tab->agg;
      ec.buffer_capacity = ew_buffer ? ew_buffer : (1u << 20);
      ec.compress_values = compress != 0;
      tab->ews.push_back(std::make_unique<EmbeddingWorker>(ec, tab->eps));
    }
    t = tab.release();
  });
  return rc == 0 ? t : nullptr;
}

void ref_table_destroy(void* h) { delete static_cast<RefTable*>(h); }

// One sync step over a batch in CSR form: ids[N], offsets[B*F+1] (u64, sample-major,
// group-minor). flags bit0 = pull, bit1 = push (ordered, one thread), bit2 = push on
// `threads` threads (hybrid). Pull writes out_pooled[B*F*D] and
// out_read_versions[N] (per listing, the PullResult order). Push applies grads[B*F*D]
// in ascending SampleId order for the batch registered by the last pull.
int ref_step(void* h, uint32_t B, const uint64_t* ids, const uint64_t* offsets, const float* grads,
             float lr, uint64_t step, int has_step, int threads, int flags, float* out_pooled,
             uint64_t* out_read_versions, uint64_t* out_sids) {
  RefTable* t = static_cast<RefTable*>(h);
  return guarded([&] {
    const uint32_t F = t->F, D = t->D;
    if (flags & 1) {
      t->sids.assign(B, SampleId{});
      for (uint32_t i = 0; i < B; ++i) {
        IdFeatures f;
        f.groups.resize(F);
        for (uint32_t g = 0; g < F; ++g) {
          uint64_t a = offsets[(uint64_t)i * F + g], b = offsets[(uint64_t)i * F + g + 1];
          f.groups[g].assign(ids + a, ids + b);
        }
        t->sids[i] = t->ews[i % t->E]->register_sample(f);
      }
      int T = std::max(1, threads);
      std::vector<std::exception_ptr> errs(T);
      auto work = [&](int w) {
        try {
          for (uint32_t i = w; i < B; i += T) {
            PullResult r = t->ews[i % t->E]->serve_pull(t->sids[i]);
            if (out_pooled)
              std::memcpy(out_pooled + (uint64_t)i * F * D, r.values.data(),
                          sizeof(float) * F * D);
            if (out_read_versions)
              std::memcpy(out_read_versions + offsets[(uint64_t)i * F], r.read_versions.data(),
                          sizeof(uint64_t) * r.read_versions.size());
          }
        } catch (...) {
          errs[w] = std::current_exception();
        }
      };
      if (T == 1) {
        work(0);
      } else {
        std::vector<std::thread> th;
        for (int w = 0; w < T; ++w) th.emplace_back(work, w);
        for (auto& x : th) x.join();
      }
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
      if (out_sids)
        for (uint32_t i = 0; i < B; ++i) out_sids[i] = t->sids[i].raw;
    }
    if (flags & 4) {
      // hybrid (asynchronous) push: T threads call apply_backward concurrently, each on
      // its own samples in ascending SampleId; no order across threads (the reference's
      // hybrid training, orchestrator.hpp:799-830)
      std::vector<uint32_t> order(t->sids.size());
      for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
      std::sort(order.begin(), order.end(),
                [&](uint32_t a, uint32_t b) { return t->sids[a] < t->sids[b]; });
      const int T = std::max(1, threads);
      std::vector<std::exception_ptr> errs(T);
      auto work = [&](int w) {
        try {
          std::vector<float> g((size_t)F * D);
          for (size_t k = w; k < order.size(); k += T) {
            const uint32_t i = order[k];
            std::memcpy(g.data(), grads + (uint64_t)i * F * D, sizeof(float) * F * D);
            t->ews[i % t->E]->apply_backward(t->sids[i], g, lr, step, has_step != 0);
          }
        } catch (...) {
          errs[w] = std::current_exception();
        }
      };
      std::vector<std::thread> th;
      for (int w = 0; w < T; ++w) th.emplace_back(work, w);
      for (auto& x : th) x.join();
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    } else if (flags & 2) {
      std::vector<uint32_t> order(t->sids.size());
      for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
      std::sort(order.begin(), order.end(),
                [&](uint32_t a, uint32_t b) { return t->sids[a] < t->sids[b]; });
      std::vector<float> g((size_t)F * D);
      for (uint32_t i : order) {
        std::memcpy(g.data(), grads + (uint64_t)i * F * D, sizeof(float) * F * D);
        t->ews[i % t->E]->apply_backward(t->sids[i], g, lr, step, has_step != 0);
      }
    }
  });
}

void ref_set_epoch(void* h, uint32_t e) {
  for (auto& ew : static_cast<RefTable*>(h)->ews) ew->set_ps_epoch(e);
}

// --- direct PsShard surface (embedding_ps.hpp:105-207) ------------------------------

int ref_shard_lookup(void* h, uint32_t s, uint64_t n, const uint64_t* ids, float* out_values,
                     uint64_t* out_versions) {
  RefTable* t = static_cast<RefTable*>(h);
  return guarded([&] {
    std::vector<uint64_t> v(ids, ids + n);
    t->shards.at(s)->lookup(v, out_values, out_versions);
  });
}

// Tracked apply (PsShard::apply_gradients). *accepted = 0 on stale epoch.
int ref_shard_apply(void* h, uint32_t s, uint64_t n, const uint64_t* ids, const float* grads,
                    const uint64_t* read_versions, float lr, uint32_t step_tag, uint32_t epoch,
                    uint32_t* out_delays, int* accepted) {
  RefTable* t = static_cast<RefTable*>(h);
  return guarded([&] {
    PsShard& sh = *t->shards.at(s);
    std::vector<PsShard::VersionedGrad> g(n);
    for (uint64_t i = 0; i < n; ++i)
      g[i] = {ids[i], grads + i * sh.embedding_dim(), read_versions ? read_versions[i] : 0};
    std::vector<uint32_t> delays;
    bool ok = sh.apply_gradients(g, lr, step_tag, epoch, &delays);
    if (accepted) *accepted = ok ? 1 : 0;
    if (ok && out_delays) std::copy(delays.begin(), delays.end(), out_delays);
  });
}

// Untracked map-shaped apply (PsShard::apply_gradients_map). ids must be distinct.
int ref_shard_apply_map(void* h, uint32_t s, uint64_t n, const uint64_t* ids, const float* grads,
                        float lr) {
  RefTable* t = static_cast<RefTable*>(h);
  return guarded([&] {
    PsShard& sh = *t->shards.at(s);
    std::map<uint64_t, std::vector<float>> m;
    for (uint64_t i = 0; i < n; ++i)
      m[ids[i]] = std::vector<float>(grads + i * sh.embedding_dim(),
                                     grads + (i + 1) * sh.embedding_dim());
    sh.apply_gradients_map(m, lr);
  });
}

// counters: miss, eviction, clock_reset, stale_epoch_drops, epoch, size
int ref_shard_counters(void* h, uint32_t s, uint64_t* out6) {
  RefTable* t = static_cast<RefTable*>(h);
  return guarded([&] {
    PsShard& sh = *t->shards.at(s);
    out6[0] = sh.miss_count();
    out6[1] = sh.eviction_count();
    out6[2] = sh.clock_reset_count();
    out6[3] = sh.stale_epoch_drops();
    out6[4] = sh.epoch();
    out6[5] = sh.size();
  });
}

uint32_t ref_shard_advance_epoch(void* h, uint32_t s) {
  return static_cast<RefTable*>(h)->shards.at(s)->advance_epoch();
}

// HPS1 checkpoint image of shard s (embedding_ps.hpp:222-260). Returns the byte
// count; copies when cap is large enough.
int64_t ref_shard_export(void* h, uint32_t s, uint8_t* buf, uint64_t cap) {
  RefTable* t = static_cast<RefTable*>(h);
  std::vector<uint8_t> out;
  int rc = guarded([&] { t->shards.at(s)->save_checkpoint(out); });
  if (rc) return -rc;
  if (buf && cap >= out.size()) std::memcpy(buf, out.data(), out.size());
  return static_cast<int64_t>(out.size());
}

// PsShard::recover_from_checkpoint (embedding_ps.hpp:280-292) of shard s from an HPS1
// image; validate_only != 0: PsShard::load_checkpoint (:262-268) into a fresh shard that
// is discarded (the parse/restore validation alone).
int ref_shard_import(void* h, uint32_t s, const uint8_t* buf, uint64_t n, int validate_only) {
  RefTable* t = static_cast<RefTable*>(h);
  return guarded([&] {
    std::vector<uint8_t> img(buf, buf + n);
    if (validate_only) (void)PsShard::load_checkpoint(img);
    else t->shards.at(s)->recover_from_checkpoint(img);
  });
}

// compress_values / decompress_values (codec.hpp:222-261), one block per row of len.
int ref_compress_values(const float* v, uint64_t rows, uint32_t len, float kappa, float* scales,
                        uint16_t* payload) {
  return guarded([&] {
    for (uint64_t r = 0; r < rows; ++r) {
      CompressedBlock b = compress_values(std::vector<float>(v + r * len, v + (r + 1) * len), kappa);
      scales[r] = b.scale;
      std::memcpy(payload + r * len, b.payload.data(), len * sizeof(uint16_t));
    }
  });
}

int ref_decompress_values(const float* scales, const uint16_t* payload, uint64_t rows,
                          uint32_t len, float* out) {
  return guarded([&] {
    for (uint64_t r = 0; r < rows; ++r) {
      CompressedBlock b;
      b.scale = scales[r];
      b.block_len = len;
      b.payload.assign(payload + r * len, payload + (r + 1) * len);
      std::vector<float> o = decompress_values(b);
      std::memcpy(out + r * len, o.data(), len * sizeof(float));
    }
  });
}

// compress_indices (codec.hpp:123-156) over a CSR batch. Outputs, all caller-sized
// for the worst case (N listings): group_u_off[G+1], unique[<=N], post_off[<=N+1]
// (relative to the flat postings array), postings[<=N] (u16 sample indices).
int ref_compress_indices(uint32_t B, uint32_t G, const uint64_t* ids, const uint64_t* offsets,
                         uint64_t* group_u_off, uint64_t* unique, uint64_t* post_off,
                         uint16_t* postings) {
  return guarded([&] {
    std::vector<IdFeatures> batch(B);
    for (uint32_t i = 0; i < B; ++i) {
      batch[i].groups.resize(G);
      for (uint32_t g = 0; g < G; ++g)
        batch[i].groups[g].assign(ids + offsets[(uint64_t)i * G + g],
                                  ids + offsets[(uint64_t)i * G + g + 1]);
    }
    CompressedIndices c = compress_indices(batch);
    uint64_t u = 0, p = 0;
    group_u_off[0] = 0;
    post_off[0] = 0;
    for (uint32_t g = 0; g < G && g < c.groups.size(); ++g) {
      const GroupPostings& gp = c.groups[g];
      for (size_t k = 0; k < gp.unique_ids.size(); ++k) {
        unique[u] = gp.unique_ids[k];
        for (uint16_t sidx : gp.postings[k]) postings[p++] = sidx;
        post_off[++u] = p;
      }
      group_u_off[g + 1] = u;
    }
    for (uint32_t g = c.groups.size(); g < G; ++g) group_u_off[g + 1] = u;
  });
}

// ---- dense tower (the C5 hybrid step) ----------------------------

// DenseNet(dims, Rng(mix64(init_seed))) as NnWorker builds it (nn_worker.hpp:331-336,
// dense_nn.hpp:42-66); dims = input + hidden widths (the output unit is appended).
// Returns the parameter count; copies the params when cap is large enough.
int64_t ref_dense_init(const uint64_t* dims, uint32_t ndims, uint64_t init_seed, float* out,
                       uint64_t cap) {
  int64_t n = -1;
  int rc = guarded([&] {
    std::vector<size_t> d(dims, dims + ndims);
    Rng rng(mix64(init_seed));
    DenseNet<float> net(d, rng);
    n = static_cast<int64_t>(net.param_count());
    if (out && cap >= net.param_count())
      std::memcpy(out, net.params().data(), net.param_count() * sizeof(float));
  });
  return rc ? -rc : n;
}

// batch_forward_backward (dense_nn.hpp:218-246) of a net holding `params`: mean BCE
// loss, probabilities, mean-loss dense gradient, per-sample input gradients.
int ref_dense_fwd_bwd(const uint64_t* dims, uint32_t ndims, const float* params, uint32_t B,
                      const float* inputs, const float* labels, float* out_loss,
                      float* out_probs, float* out_dense_grad, float* out_input_grads) {
  return guarded([&] {
    std::vector<size_t> d(dims, dims + ndims);
    Rng rng(0);
    DenseNet<float> net(d, rng);
    std::memcpy(net.params().data(), params, net.param_count() * sizeof(float));
    const size_t in = d.front();
    std::vector<std::vector<float>> x(B);
    std::vector<float> y(labels, labels + B);
    for (uint32_t i = 0; i < B; ++i) x[i].assign(inputs + i * in, inputs + (i + 1) * in);
    BatchResult<float> r = batch_forward_backward(net, x, y);
    *out_loss = r.mean_loss;
    std::memcpy(out_probs, r.probs.data(), B * sizeof(float));
    std::memcpy(out_dense_grad, r.dense_grad.data(), r.dense_grad.size() * sizeof(float));
    for (uint32_t i = 0; i < B; ++i)
      std::memcpy(out_input_grads + i * in, r.input_grads[i].data(), in * sizeof(float));
  });
}

// AllReduceHub::reduce (nn_worker.hpp:85-87, canonical_mean :214-226): K ranks on K
// threads contribute parts[k*n .. (k+1)*n); out = the canonical mean every rank receives.
int ref_allreduce(uint32_t K, uint64_t n, const float* parts, float* out) {
  return guarded([&] {
    AllReduceHub hub(K);
    std::vector<std::vector<float>> res(K);
    std::vector<std::thread> th;
    for (uint32_t k = 0; k < K; ++k)
      th.emplace_back([&, k] {
        std::vector<float> g(parts + k * n, parts + (k + 1) * n);
        res[k] = hub.reduce(k, 0, g);
      });
    for (auto& t : th) t.join();
    std::memcpy(out, res[0].data(), n * sizeof(float));
  });
}

// sgd_step (dense_nn.hpp:263-273): params -= lr * grad, refusing non-finite gradients.
int ref_sgd_step(float* params, const float* grad, uint64_t n, float lr) {
  return guarded([&] {
    std::vector<float> p(params, params + n), g(grad, grad + n);
    sgd_step(p, g, lr);
    std::memcpy(params, p.data(), n * sizeof(float));
  });
}

}  // extern "C"

