// Drives include/hps/compat.hpp the way the reference's own tests drive hybridps::PsShard /
// ShardSet / EmbeddingWorker (test_embedding_ps.cpp:87-136, test_embedding_worker.cpp:216-362).
// Exit 0 = every check held. Needs a GPU to run; compiled by tests/test_abi.py on CPU.
#include <cstdio>
#include <cstring>

#include "hps/compat.hpp"

using namespace hps_b200;

static int fails = 0;
#define EXPECT(c)                                           \
  do {                                                      \
    if (!(c)) {                                             \
      std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                              \
    }                                                       \
  } while (0)

int main() {
  // SGD bit-exact w - 0.5*g (test_embedding_ps.cpp:87-100)
  PsShardConfig cfg;
  cfg.capacity = 1024;
  cfg.embedding_dim = 4;
  cfg.optimizer = EmbOptimizer::kSgd;
  cfg.rng_salt = 99;
  PsShard ps(cfg);
  std::vector<float> before(4), after(4);
  std::vector<uint64_t> ver(1);
  ps.lookup({42}, before.data(), ver.data());
  EXPECT(ver[0] == 0);
  EXPECT(ps.miss_count() == 1);
  const float g[4] = {1.0f, -2.0f, 0.5f, 0.0f};
  std::vector<PsShard::VersionedGrad> vg{{42, g, 0}};
  std::vector<uint32_t> delays;
  EXPECT(ps.apply_gradients(vg, 0.5f, 1, ps.epoch(), &delays));
  ps.lookup({42}, after.data(), ver.data());
  for (int d = 0; d < 4; ++d) EXPECT(after[d] == before[d] - 0.5f * g[d]);
  EXPECT(ver[0] == 1 && delays.size() == 1 && delays[0] == 0);
  // stale epoch drops the call (embedding_ps.hpp:141-145)
  ps.advance_epoch();
  EXPECT(!ps.apply_gradients(vg, 0.5f, 2, 0, nullptr));
  EXPECT(ps.stale_epoch_drops() == 1);
  // non-finite rejected atomically (test_embedding_ps.cpp:120-136)
  const float bad[4] = {1.0f, NAN, 0.0f, 0.0f};
  std::vector<PsShard::VersionedGrad> vb{{42, g, 1}, {43, bad, 0}};
  bool threw = false;
  try {
    ps.apply_gradients(vb, 0.5f, 3, ps.epoch(), nullptr);
  } catch (const DivergenceError&) {
    threw = true;
  }
  EXPECT(threw);
  std::vector<float> again(4);
  ps.lookup({42}, again.data());
  EXPECT(std::memcmp(again.data(), after.data(), sizeof(float) * 4) == 0);

  // ShardSet + EmbeddingWorker: one id pooled = its row (test_embedding_worker.cpp:216-232),
  // then a gated flush applies SGD exactly (:338-362)
  PsShardConfig base;
  base.capacity = 4096;
  base.embedding_dim = 8;
  base.optimizer = EmbOptimizer::kSgd;
  base.rng_salt = 7;
  ShardSet set(4, base);
  EXPECT(set.shard_of(12345) == route_shard(12345, 4));
  EmbeddingWorkerConfig ecfg;
  ecfg.group_count = 2;
  ecfg.embedding_dim = 8;
  ecfg.aggregation = Aggregation::kSum;
  EmbeddingWorker ew(ecfg, set);
  SampleId sid = ew.register_sample({{10}, {}});
  PullResult pr = ew.serve_pull(sid);
  auto row = set.lookup({10});
  for (int d = 0; d < 8; ++d) EXPECT(pr.values[d] == row[10][d]);
  for (int d = 8; d < 16; ++d) EXPECT(pr.values[d] == 0.0f);
  std::vector<float> grads(16, 0.25f);
  ew.apply_backward(sid, grads, 0.5f, 1, true);
  ew.flush_step_marker(1, 0);
  auto row2 = set.lookup({10});
  for (int d = 0; d < 8; ++d) EXPECT(row2[10][d] == row[10][d] - 0.5f * 0.25f);

  // checkpoint round trip (test_embedding_ps.cpp:243-391): save, corrupt -> rejected and
  // unchanged, recover -> same row, epoch past the live one
  std::vector<uint8_t> img;
  EXPECT(ps.save_checkpoint(img) == img.size() && img.size() > 64);
  EXPECT(std::memcmp(img.data(), "HPS1", 4) == 0);
  std::vector<uint8_t> broken = img;
  broken[70] ^= 1;
  threw = false;
  try {
    ps.recover_from_checkpoint(broken);
  } catch (const CheckpointCorruptError&) {
    threw = true;
  }
  EXPECT(threw);
  const uint32_t e_live = ps.epoch();
  ps.recover_from_checkpoint(img);
  EXPECT(ps.epoch() == e_live + 1);
  std::vector<float> restored(4);
  ps.lookup({42}, restored.data(), ver.data());
  EXPECT(std::memcmp(restored.data(), after.data(), sizeof(float) * 4) == 0 && ver[0] == 1);
  if (fails == 0) std::printf("compat_smoke OK\n");
  return fails ? 1 : 0;
}
