// HPS1 checkpoint images of the device table.
//
// The reference persists one PsShard as a fixed 64-byte header plus flat little-endian
// arrays (PsShard::save_checkpoint embedding_ps.hpp:222-260):
//   magic "HPS1" | version u8 = 1 | optimizer u8 | pad u16 | dim u32 | capacity u32 |
//   salt u64 | hwm u32 | head u32 | tail u32 | free_head u32 | live u32 | epoch u32 |
//   evictions u64 | checksum u64 (FNV-1a over the image with this field zeroed)
//   ids[hwm] u64 | prev[hwm] u32 | next[hwm] u32 | versions[hwm] u64 | rows[hwm][2D] f32
// A device table holds S logical shards; save writes the image of one of them, load
// adopts a set of images (load_checkpoint / recover_from_checkpoint :262-300), validated
// exactly as the reference's parse + LruStore::restore do (:318-362,
// lru_store.hpp:172-224) before anything changes.
//
// The device table keeps no recency list (no LRU eviction), so
// a saved image lists the shard's rows in slot (first-insertion) order with the recency
// chain running from the newest slot (head, most recent) to the oldest (tail). That is
// byte-identical to the reference's image whenever its recency order is its insertion
// order, and a valid image the reference loads in every case; a loaded image's chain
// order is not kept.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "table.cuh"
#include "table_impl.h"

namespace hps {

namespace {

constexpr size_t kHdr = 64;
constexpr size_t kSumOff = 56;
constexpr uint32_t kNil = 0xffffffffu;  // LruStore::kNil lru_store.hpp:36

uint64_t fnv1a64(const uint8_t* p, size_t n, uint64_t h = 0xcbf29ce484222325ULL) {  // core.hpp:187
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

template <typename T>
T rd(const uint8_t* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}
template <typename T>
void wr(uint8_t* p, T v) {
  std::memcpy(p, &v, sizeof(T));
}

[[noreturn]] void corrupt(const std::string& m) { throw Error(HPS_E_CHECKPOINT_CORRUPT, m); }

struct Image {
  uint32_t opt, dim, capacity, hwm, head, tail, free_head, live, epoch;
  uint64_t salt;
  const uint64_t* ids;  // unaligned-safe copies below
  std::vector<uint32_t> live_slots;  // recency chain, head first
  const uint8_t* base;
};

// PsShard::parse (embedding_ps.hpp:318-362) + LruStore::restore checks (:172-224).
Image parse(const uint8_t* p, uint64_t n) {
  if (n < kHdr) corrupt("load_checkpoint: truncated header");
  if (std::memcmp(p, "HPS1", 4) != 0) corrupt("load_checkpoint: bad magic");
  if (p[4] != 1) corrupt("load_checkpoint: unsupported format version " + std::to_string(p[4]));
  {
    // checksum over the image with its own field zeroed, without copying the image
    uint64_t h = fnv1a64(p, kSumOff);
    const uint8_t zero[8] = {0};
    h = fnv1a64(zero, 8, h);
    h = fnv1a64(p + kSumOff + 8, n - kSumOff - 8, h);
    if (h != rd<uint64_t>(p + kSumOff)) corrupt("load_checkpoint: checksum mismatch");
  }
  Image im{};
  im.base = p;
  im.opt = p[5];
  if (im.opt > 1) corrupt("load_checkpoint: unknown optimizer kind");
  im.dim = rd<uint32_t>(p + 8);
  im.capacity = rd<uint32_t>(p + 12);
  im.salt = rd<uint64_t>(p + 16);
  im.hwm = rd<uint32_t>(p + 24);
  im.head = rd<uint32_t>(p + 28);
  im.tail = rd<uint32_t>(p + 32);
  im.free_head = rd<uint32_t>(p + 36);
  im.live = rd<uint32_t>(p + 40);
  im.epoch = rd<uint32_t>(p + 44);
  if (im.dim == 0 || im.capacity == 0) corrupt("load_checkpoint: degenerate dimensions");
  const uint64_t H = im.hwm;
  const uint64_t body = H * (2 * 8 + 2 * 4) + H * im.dim * 2ull * 4;
  if (n != kHdr + body) corrupt("load_checkpoint: length mismatch");
  if (im.hwm > im.capacity) corrupt("LruStore::restore: high-water mark exceeds capacity");
  const uint8_t* q = p + kHdr;
  const uint8_t* ids = q;
  const uint8_t* prev = ids + 8 * H;
  const uint8_t* next = prev + 4 * H;
  auto id_at = [&](uint32_t s) { return rd<uint64_t>(ids + 8ull * s); };
  auto prev_at = [&](uint32_t s) { return rd<uint32_t>(prev + 4ull * s); };
  auto next_at = [&](uint32_t s) { return rd<uint32_t>(next + 4ull * s); };
  std::vector<uint8_t> seen(H, 0);
  std::vector<uint64_t> chain_ids;
  uint32_t cnt = 0, expect_prev = kNil;
  for (uint32_t s = im.head; s != kNil; s = next_at(s)) {
    if (s >= H) corrupt("LruStore::restore: slot index out of range");
    if (seen[s]) corrupt("LruStore::restore: recency chain has a cycle");
    seen[s] = 1;
    if (prev_at(s) != expect_prev) corrupt("LruStore::restore: prev/next links inconsistent");
    im.live_slots.push_back(s);
    chain_ids.push_back(id_at(s));
    expect_prev = s;
    if (++cnt > H) corrupt("LruStore::restore: chain longer than slots");
  }
  if (expect_prev != im.tail) corrupt("LruStore::restore: tail does not terminate the chain");
  if (cnt != im.live) corrupt("LruStore::restore: live count mismatch");
  std::sort(chain_ids.begin(), chain_ids.end());
  if (std::adjacent_find(chain_ids.begin(), chain_ids.end()) != chain_ids.end())
    corrupt("LruStore::restore: duplicate id in chain");
  uint32_t f = 0;
  for (uint32_t s = im.free_head; s != kNil; s = next_at(s)) {
    if (s >= H) corrupt("LruStore::restore: slot index out of range");
    if (seen[s]) corrupt("LruStore::restore: slot both live and free");
    seen[s] = 1;
    if (++f > H) corrupt("LruStore::restore: free list cycle");
  }
  if (cnt + f != H) corrupt("LruStore::restore: live and free slots do not partition the slot range");
  return im;
}

}  // namespace

uint64_t table_ckpt_save(Table* t, uint32_t shard, uint32_t shard_capacity, uint8_t* buf,
                         uint64_t cap) {
  DeviceGuard g(t->device);
  const uint32_t S = t->cfg.shard_count;
  if (shard >= S) throw Error(HPS_E_PRECONDITION, "checkpoint_save: shard out of range");
  const uint32_t D = t->cfg.embedding_dim;
  HPS_CUDA(cudaDeviceSynchronize());
  std::vector<uint32_t> sel;
  std::vector<uint64_t> sid;
  std::vector<uint32_t> lru_order;  // LRU mode: image slots, most recent first
  unsigned long long evictions = 0;
  if (t->d.lru) {
    // LRU mode: the shard's own slot range, in recency order (newest first, by stamp)
    uint32_t hwm = 0;
    const uint32_t base = shard * t->d.shard_cap;
    HPS_CUDA(cudaMemcpy(&hwm, t->d.shard_hwm + shard, sizeof(hwm), cudaMemcpyDeviceToHost));
    HPS_CUDA(cudaMemcpy(&evictions, t->d.shard_evict + shard, sizeof(evictions),
                        cudaMemcpyDeviceToHost));
    hwm = std::min(hwm, t->d.shard_cap);
    sid.resize(static_cast<uint64_t>(base) + hwm);
    std::vector<unsigned long long> stamp(hwm);
    if (hwm) {
      HPS_CUDA(cudaMemcpy(sid.data() + base, t->d.slot_id + base, hwm * sizeof(uint64_t),
                          cudaMemcpyDeviceToHost));
      HPS_CUDA(cudaMemcpy(stamp.data(), t->d.stamp + base, hwm * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost));
    }
    // image slot k = device slot base + k; the recency chain follows the stamps
    for (uint32_t k = 0; k < hwm; ++k) sel.push_back(base + k);
    lru_order.resize(hwm);
    for (uint32_t k = 0; k < hwm; ++k) lru_order[k] = k;
    std::stable_sort(lru_order.begin(), lru_order.end(),
                     [&](uint32_t x, uint32_t y) { return stamp[x] > stamp[y]; });  // newest first
  } else {
    uint32_t hwm = 0;
    HPS_CUDA(cudaMemcpy(&hwm, t->d.hwm, sizeof(hwm), cudaMemcpyDeviceToHost));
    hwm = std::min(hwm, t->d.capacity);
    sid.resize(hwm);
    if (hwm)
      HPS_CUDA(cudaMemcpy(sid.data(), t->d.slot_id, hwm * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    for (uint32_t s = 0; s < hwm; ++s)
      if (route_shard(sid[s], S) == shard) sel.push_back(s);
  }
  const uint64_t n = sel.size();
  const uint64_t bytes = kHdr + n * (2 * 8 + 2 * 4) + n * D * 2ull * 4;
  if (!buf || cap < bytes) return bytes;
  const uint64_t capacity =
      shard_capacity ? shard_capacity : (t->d.lru ? t->d.shard_cap : t->cfg.capacity);
  if (capacity > 0xffffffffull || n > 0xffffffffull)
    throw Error(HPS_E_CONFIG, "checkpoint_save: capacity does not fit the HPS1 header");
  // rows + versions of the shard's slots, gathered on the device
  uint32_t* d_sel = nullptr;
  float* d_rows = nullptr;
  uint64_t* d_ver = nullptr;
  std::vector<uint64_t> ver(n);
  try {
    if (n) {
      HPS_CUDA(cudaMalloc(&d_sel, n * sizeof(uint32_t)));
      HPS_CUDA(cudaMalloc(&d_rows, n * D * 2ull * sizeof(float)));
      HPS_CUDA(cudaMalloc(&d_ver, n * sizeof(uint64_t)));
      HPS_CUDA(cudaMemcpy(d_sel, sel.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
      launch_ckpt_gather(t->d, d_sel, n, d_rows, d_ver, nullptr);
      HPS_CUDA(cudaMemcpy(buf + kHdr + n * 24, d_rows, n * D * 2ull * sizeof(float),
                          cudaMemcpyDeviceToHost));
      HPS_CUDA(cudaMemcpy(ver.data(), d_ver, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    }
  } catch (...) {
    cudaFree(d_sel);
    cudaFree(d_rows);
    cudaFree(d_ver);
    throw;
  }
  cudaFree(d_sel);
  cudaFree(d_rows);
  cudaFree(d_ver);
  const uint32_t n32 = static_cast<uint32_t>(n);
  std::memset(buf, 0, kHdr);
  std::memcpy(buf, "HPS1", 4);
  buf[4] = 1;
  buf[5] = static_cast<uint8_t>(t->cfg.optimizer);
  wr<uint32_t>(buf + 8, D);
  wr<uint32_t>(buf + 12, static_cast<uint32_t>(capacity));
  wr<uint64_t>(buf + 16, t->salts[shard]);
  wr<uint32_t>(buf + 24, n32);                       // hwm: the slots are dense
  if (t->d.lru) {
    wr<uint32_t>(buf + 28, n32 ? lru_order[0] : kNil);       // head = most recent
    wr<uint32_t>(buf + 32, n32 ? lru_order[n32 - 1] : kNil);  // tail = least recent
  } else {
    wr<uint32_t>(buf + 28, n32 ? n32 - 1 : kNil);  // head = newest slot (most recent)
    wr<uint32_t>(buf + 32, n32 ? 0u : kNil);       // tail = oldest slot
  }
  wr<uint32_t>(buf + 36, kNil);                      // no free slots (nothing evicted)
  wr<uint32_t>(buf + 40, n32);
  wr<uint32_t>(buf + 44, t->epoch);
  wr<uint64_t>(buf + 48, evictions);                 // (LRU mode; 0 otherwise)
  uint8_t* q = buf + kHdr;
  for (uint64_t i = 0; i < n; ++i) wr<uint64_t>(q + 8 * i, sid[sel[i]]);
  q += 8 * n;
  if (t->d.lru) {  // prev = the next more recent slot, next = the next less recent one
    for (uint64_t r = 0; r < n; ++r) {
      wr<uint32_t>(q + 4ull * lru_order[r], r ? lru_order[r - 1] : kNil);
      wr<uint32_t>(q + 4ull * n + 4ull * lru_order[r], r + 1 < n ? lru_order[r + 1] : kNil);
    }
  } else {
    for (uint64_t i = 0; i < n; ++i) wr<uint32_t>(q + 4 * i, i + 1 < n ? uint32_t(i + 1) : kNil);
    for (uint64_t i = 0; i < n; ++i) wr<uint32_t>(q + 4 * n + 4 * i, i ? uint32_t(i - 1) : kNil);
  }
  q += 8 * n;
  std::memcpy(q, ver.data(), n * 8);
  wr<uint64_t>(buf + kSumOff, fnv1a64(buf, bytes));
  return bytes;
}

void table_ckpt_load(Table* t, const uint8_t* const* images, const uint64_t* sizes, uint32_t count,
                     int recover) {
  DeviceGuard g(t->device);
  const uint32_t S = t->cfg.shard_count, D = t->cfg.embedding_dim;
  // 1. validate everything before anything changes
  std::vector<Image> ims;
  std::vector<uint32_t> shard_of;
  uint64_t total = 0;
  uint32_t max_epoch = 0;
  for (uint32_t k = 0; k < count; ++k) {
    if (!images[k]) throw Error(HPS_E_PRECONDITION, "checkpoint_load: null image");
    Image im = parse(images[k], sizes[k]);
    if (im.dim != D || static_cast<int>(im.opt) != t->cfg.optimizer)
      throw Error(HPS_E_CHECKPOINT_CORRUPT, "recover_from_checkpoint: configuration mismatch");
    uint32_t s = S;
    for (uint32_t j = 0; j < S; ++j)
      if (t->salts[j] == im.salt) {
        s = j;
        break;
      }
    if (s == S) throw Error(HPS_E_CONFIG, "checkpoint_load: image salt matches no shard of this table");
    if (std::find(shard_of.begin(), shard_of.end(), s) != shard_of.end())
      throw Error(HPS_E_PRECONDITION, "checkpoint_load: two images for one shard");
    const uint8_t* ids = images[k] + kHdr;
    const uint8_t* vers = ids + uint64_t(im.hwm) * 16;
    const uint8_t* rows = ids + uint64_t(im.hwm) * 24;
    for (uint32_t sl : im.live_slots) {
      const uint64_t id = rd<uint64_t>(ids + 8ull * sl);
      if (route_shard(id, S) != s)
        throw Error(HPS_E_CONFIG, "checkpoint_load: image holds an id of another shard");
      if (rd<uint64_t>(vers + 8ull * sl) > 0xffffffffull)
        throw Error(HPS_E_CONFIG, "checkpoint_load: version exceeds the device's 32-bit clock");
      if (t->d.svt)
        for (uint32_t d = 0; d < 64; ++d)
          if (rd<uint32_t>(rows + (uint64_t(sl) * 2 * D + D + d) * 4) >> 31)
            throw Error(HPS_E_CONFIG, "checkpoint_load: negative accumulator");
    }
    total += im.live;
    max_epoch = std::max(max_epoch, im.epoch);
    shard_of.push_back(s);
    ims.push_back(std::move(im));
  }
  if (total > t->d.capacity) throw Error(HPS_E_CONFIG, "checkpoint_load: images exceed the table capacity");
  if (t->d.lru)
    for (const Image& im : ims) {
      if (im.hwm > t->d.shard_cap)
        throw Error(HPS_E_CONFIG, "checkpoint_load: an image holds more rows than a shard's capacity");
      if (im.free_head != kNil)
        throw Error(HPS_E_CONFIG, "checkpoint_load: images with free slots need a table without "
                                  "HPS_TABLE_LRU");
    }
  // 2. pack the live rows (recency order) and adopt them on the device
  std::vector<uint64_t> ids(total), vers(total);
  std::vector<float> rows(total * 2ull * D);
  // LRU mode: every row back in its image slot (so a save reproduces the image byte for
  // byte), stamped by its position in the recency chain
  std::vector<uint32_t> at(t->d.lru ? total : 0);
  std::vector<unsigned long long> stamps(t->d.lru ? total : 0);
  std::vector<uint32_t> hwm_of(S, 0);
  uint64_t o = 0;
  for (uint32_t k = 0; k < count; ++k) {
    const Image& im = ims[k];
    const uint8_t* pid = images[k] + kHdr;
    const uint8_t* pv = pid + uint64_t(im.hwm) * 16;
    const uint8_t* pr = pid + uint64_t(im.hwm) * 24;
    hwm_of[shard_of[k]] = im.hwm;
    uint64_t rank = 0;
    for (uint32_t sl : im.live_slots) {
      ids[o] = rd<uint64_t>(pid + 8ull * sl);
      vers[o] = rd<uint64_t>(pv + 8ull * sl);
      std::memcpy(&rows[o * 2 * D], pr + uint64_t(sl) * 2 * D * 4, 2ull * D * 4);
      if (t->d.lru) {
        at[o] = shard_of[k] * t->d.shard_cap + sl;
        stamps[o] = 1 + im.live - rank;  // head (most recent) first
      }
      ++rank;
      ++o;
    }
  }
  HPS_CUDA(cudaDeviceSynchronize());
  table_clear(t, nullptr);
  Batch& b = t->scratch;
  batch_reserve(b, total, 0, 0);
  b.registered = false;
  uint64_t* d_ids = nullptr;
  uint64_t* d_ver = nullptr;
  float* d_rows = nullptr;
  uint32_t* d_at = nullptr;
  unsigned long long* d_st = nullptr;
  auto release = [&] {
    cudaFree(d_ids);
    cudaFree(d_ver);
    cudaFree(d_rows);
    cudaFree(d_at);
    cudaFree(d_st);
  };
  try {
    if (total) {
      HPS_CUDA(cudaMalloc(&d_ids, total * 8));
      HPS_CUDA(cudaMalloc(&d_ver, total * 8));
      HPS_CUDA(cudaMalloc(&d_rows, total * 2ull * D * 4));
      HPS_CUDA(cudaMemcpy(d_ids, ids.data(), total * 8, cudaMemcpyHostToDevice));
      HPS_CUDA(cudaMemcpy(d_ver, vers.data(), total * 8, cudaMemcpyHostToDevice));
      HPS_CUDA(cudaMemcpy(d_rows, rows.data(), total * 2ull * D * 4, cudaMemcpyHostToDevice));
      HPS_CUDA(cudaMemset(b.small, 0, 8 * sizeof(uint32_t)));
      if (t->d.lru) {
        HPS_CUDA(cudaMalloc(&d_at, total * sizeof(uint32_t)));
        HPS_CUDA(cudaMalloc(&d_st, total * sizeof(unsigned long long)));
        HPS_CUDA(cudaMemcpy(d_at, at.data(), total * 4, cudaMemcpyHostToDevice));
        HPS_CUDA(cudaMemcpy(d_st, stamps.data(), total * 8, cudaMemcpyHostToDevice));
        HPS_CUDA(cudaMemcpy(t->d.shard_hwm, hwm_of.data(), S * 4, cudaMemcpyHostToDevice));
      }
      launch_ckpt_restore(t->d, d_ids, d_rows, d_ver, total, b.new_slots, &b.small[2], nullptr,
                          d_at, d_st);
    }
    HPS_CUDA(cudaDeviceSynchronize());
  } catch (...) {
    release();
    throw;
  }
  release();
  if (t->d.lru) {  // LruStore::restore keeps the eviction count (embedding_ps.hpp:400)
    std::vector<unsigned long long> ev(S, 0);
    for (uint32_t k = 0; k < count; ++k) ev[shard_of[k]] = rd<uint64_t>(images[k] + 48);
    HPS_CUDA(cudaMemcpy(t->d.shard_evict, ev.data(), S * sizeof(unsigned long long),
                        cudaMemcpyHostToDevice));
    unsigned long long tot = 0;
    for (auto v : ev) tot += v;
    HPS_CUDA(cudaMemcpy(t->d.ctr + kCtrEvictions, &tot, sizeof(tot), cudaMemcpyHostToDevice));
    t->clock = total + 2;
  }
  t->outstanding.clear();  // batches registered before the load refer to old slots
  t->epoch = recover ? std::max(t->epoch, max_epoch) + 1 : max_epoch;
  check_flags(t, nullptr, false);
}

}  // namespace hps
