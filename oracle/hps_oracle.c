/* CPU restatement of the reference's embedding lookup+update path.
 *
 * TEST INFRASTRUCTURE ONLY (see hps_oracle.h). Parity pinned against the
 * reference build oracle/_ref/libhps_ref.so and the reference's known-answer
 * tests; see tests/test_oracle_pinning.py.
 *
 * Compiled with -O2 -ffp-contract=off (oracle/Makefile): every float/double
 * operation below rounds individually, as the reference does on default x86-64.
 *
 * Scope notes: rows are never evicted (unbounded capacity). The reference's
 * LRU eviction only changes values when a shard's working set exceeds its
 * capacity (SURVEY.md §7 hard part 3), which no parity config does.
 */
#include "hps_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_GAMMA 0x9e3779b97f4a7c15ULL
#define ORC_TAG_RING 16u
#define ORC_NO_STEP 0xffffffffu

/* core.hpp:36-44 (splitmix64 finalizer with the pinned constants core.hpp:32-34). */
uint64_t orc_mix64(uint64_t x) {
  x += ORC_GAMMA;
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

/* core.hpp:145-150: mix64(id) % shard_count. */
uint32_t orc_route_shard(uint64_t id, uint32_t shard_count) {
  return shard_count ? (uint32_t)(orc_mix64(id) % shard_count) : 0u;
}

/* embedding_ps.hpp:424-429 with Rng (core.hpp:49-63): the d-th draw of
 * Rng(mix64(id ^ mix64(salt))) is mix64(seed + d*gamma); uniform01 keeps the top
 * 53 bits; uniform(lo, hi) = lo + (hi - lo) * u in double, then cast to float. */
void orc_init_row(uint64_t id, uint64_t shard_salt, uint32_t dim, float* out_w) {
  uint64_t seed = orc_mix64(id ^ orc_mix64(shard_salt));
  double limit = 1.0 / sqrt((double)dim);
  double lo = -limit, hi = limit;
  double span = hi - lo;
  for (uint32_t d = 0; d < dim; ++d) {
    uint64_t r = orc_mix64(seed + (uint64_t)d * ORC_GAMMA);
    double u = (double)(r >> 11) * 0x1.0p-53;
    double prod = span * u;
    out_w[d] = (float)(lo + prod);
  }
}

/* ----------------------------------------------------------------------------
 * Row store: open-addressing id -> row index, rows [w D | acc D] (the reference
 * row layout, embedding_ps.hpp:64), u64 version + 16-deep step-tag ring per row
 * (embedding_ps.hpp:493-494).
 * -------------------------------------------------------------------------- */

struct orc_table {
  uint32_t S, D;
  int opt;
  uint64_t* salts;
  /* index */
  uint64_t* keys;
  uint32_t* vals; /* row index + 1; 0 = empty */
  uint64_t cap;   /* power of two */
  /* rows */
  uint64_t n, row_cap;
  float* rows;
  uint64_t* versions;
  uint32_t* rings;
  uint64_t misses, clock_resets, stale_drops;
  uint32_t epoch;
};

static uint64_t slot_hash(uint64_t id) { return orc_mix64(id ^ 0x6a09e667f3bcc909ULL); }

static void index_insert(orc_table* t, uint64_t id, uint32_t v) {
  uint64_t m = t->cap - 1, h = slot_hash(id) & m;
  while (t->vals[h]) h = (h + 1) & m;
  t->keys[h] = id;
  t->vals[h] = v;
}

static int64_t index_find(const orc_table* t, uint64_t id) {
  if (!t->cap) return -1;
  uint64_t m = t->cap - 1, h = slot_hash(id) & m;
  while (t->vals[h]) {
    if (t->keys[h] == id) return (int64_t)t->vals[h] - 1;
    h = (h + 1) & m;
  }
  return -1;
}

static void grow(orc_table* t) {
  if ((t->n + 1) * 2 > t->cap) {
    uint64_t oc = t->cap;
    uint64_t* ok = t->keys;
    uint32_t* ov = t->vals;
    t->cap = oc ? oc * 2 : 1024;
    t->keys = (uint64_t*)calloc(t->cap, sizeof(uint64_t));
    t->vals = (uint32_t*)calloc(t->cap, sizeof(uint32_t));
    for (uint64_t i = 0; i < oc; ++i)
      if (ov[i]) index_insert(t, ok[i], ov[i]);
    free(ok);
    free(ov);
  }
  if (t->n + 1 > t->row_cap) {
    t->row_cap = t->row_cap ? t->row_cap * 2 : 1024;
    t->rows = (float*)realloc(t->rows, t->row_cap * 2 * t->D * sizeof(float));
    t->versions = (uint64_t*)realloc(t->versions, t->row_cap * sizeof(uint64_t));
    t->rings = (uint32_t*)realloc(t->rings, t->row_cap * ORC_TAG_RING * sizeof(uint32_t));
  }
}

orc_table* orc_table_create(uint32_t S, const uint64_t* salts, uint32_t D, int opt) {
  if (S == 0 || D == 0) return NULL;
  orc_table* t = (orc_table*)calloc(1, sizeof(orc_table));
  t->S = S;
  t->D = D;
  t->opt = opt;
  t->salts = (uint64_t*)malloc(S * sizeof(uint64_t));
  memcpy(t->salts, salts, S * sizeof(uint64_t));
  return t;
}

void orc_table_destroy(orc_table* t) {
  if (!t) return;
  free(t->salts);
  free(t->keys);
  free(t->vals);
  free(t->rows);
  free(t->versions);
  free(t->rings);
  free(t);
}

uint32_t orc_table_epoch(const orc_table* t) { return t->epoch; }
uint32_t orc_table_advance_epoch(orc_table* t) { return ++t->epoch; }
uint64_t orc_table_size(const orc_table* t) { return t->n; }
void orc_table_counters(const orc_table* t, uint64_t* o) {
  o[0] = t->misses;
  o[1] = t->clock_resets;
  o[2] = t->stale_drops;
  o[3] = t->n;
}

/* PsShard::find_or_init, embedding_ps.hpp:417-434 (shard = route_shard(id, S)
 * picks the salt, ShardSet::shard_of embedding_ps.hpp:521-523). */
static uint32_t find_or_init(orc_table* t, uint64_t id) {
  int64_t r = index_find(t, id);
  if (r >= 0) return (uint32_t)r;
  grow(t);
  uint32_t row = (uint32_t)t->n++;
  index_insert(t, id, row + 1);
  t->misses++;
  float* w = t->rows + (uint64_t)row * 2 * t->D;
  orc_init_row(id, t->salts[orc_route_shard(id, t->S)], t->D, w);
  memset(w + t->D, 0, t->D * sizeof(float));
  t->versions[row] = 0;
  for (uint32_t k = 0; k < ORC_TAG_RING; ++k) t->rings[(uint64_t)row * ORC_TAG_RING + k] = ORC_NO_STEP;
  return row;
}

/* PsShard::apply_one, embedding_ps.hpp:436-449. Every operation rounds to float. */
static void apply_one(orc_table* t, uint32_t row, const float* g, float lr) {
  float* w = t->rows + (uint64_t)row * 2 * t->D;
  float* a = w + t->D;
  for (uint32_t d = 0; d < t->D; ++d) {
    if (t->opt == 0) {
      float gg = g[d] * g[d];
      a[d] = a[d] + gg;
      float num = lr * g[d];
      float den = sqrtf(a[d]) + 1e-10f;
      float step = num / den;
      w[d] = w[d] - step;
    } else {
      float step = lr * g[d];
      w[d] = w[d] - step;
    }
  }
}

/* PsShard::count_delay, embedding_ps.hpp:454-480. */
static uint32_t count_delay(orc_table* t, uint32_t row, uint64_t read_version, uint32_t step_tag) {
  uint64_t v = t->versions[row];
  if (read_version > v) {
    t->clock_resets++;
    return 0;
  }
  const uint32_t* ring = t->rings + (uint64_t)row * ORC_TAG_RING;
  uint32_t distinct[ORC_TAG_RING];
  uint32_t n = 0;
  uint64_t lo = read_version + 1;
  if (v >= ORC_TAG_RING && lo < v - ORC_TAG_RING + 1) lo = v - ORC_TAG_RING + 1;
  for (uint64_t k = lo; k <= v; ++k) {
    uint32_t tag = ring[(k - 1) % ORC_TAG_RING];
    if (tag == ORC_NO_STEP || tag >= step_tag) continue;
    int dup = 0;
    for (uint32_t j = 0; j < n; ++j)
      if (distinct[j] == tag) dup = 1;
    if (!dup) distinct[n++] = tag;
  }
  return n;
}

/* PsShard::bump_version, embedding_ps.hpp:482-488. */
static void bump_version(orc_table* t, uint32_t row, uint32_t step_tag) {
  uint64_t v = t->versions[row];
  uint32_t* ring = t->rings + (uint64_t)row * ORC_TAG_RING;
  if (v > 0 && ring[(v - 1) % ORC_TAG_RING] == step_tag) return;
  t->versions[row] = v + 1;
  ring[v % ORC_TAG_RING] = step_tag;
}

/* PsShard::lookup, embedding_ps.hpp:105-114. */
void orc_lookup(orc_table* t, const uint64_t* ids, size_t n, float* out_values,
                uint64_t* out_versions) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t row = find_or_init(t, ids[i]);
    memcpy(out_values + i * t->D, t->rows + (uint64_t)row * 2 * t->D, t->D * sizeof(float));
    if (out_versions) out_versions[i] = t->versions[row];
  }
}

void orc_peek(const orc_table* t, const uint64_t* ids, size_t n, float* out_w, float* out_acc,
              uint64_t* out_versions, uint8_t* out_present) {
  for (size_t i = 0; i < n; ++i) {
    int64_t r = index_find(t, ids[i]);
    if (out_present) out_present[i] = r >= 0;
    if (r < 0) continue;
    const float* w = t->rows + (uint64_t)r * 2 * t->D;
    if (out_w) memcpy(out_w + i * t->D, w, t->D * sizeof(float));
    if (out_acc) memcpy(out_acc + i * t->D, w + t->D, t->D * sizeof(float));
    if (out_versions) out_versions[i] = t->versions[r];
  }
}

static int all_finite(const float* g, uint32_t D) {
  for (uint32_t d = 0; d < D; ++d)
    if (!isfinite(g[d])) return 0;
  return 1;
}

/* PsShard::apply_gradients, embedding_ps.hpp:139-162: epoch fence, validate every
 * vector, then per entry in array order find_or_init -> count_delay -> bump -> apply. */
int orc_apply(orc_table* t, const uint64_t* ids, const float* grads, const uint64_t* read_versions,
              size_t n, float lr, uint32_t step_tag, uint32_t epoch, uint32_t* out_delays,
              int* accepted) {
  if (epoch != t->epoch) {
    t->stale_drops += n;
    if (accepted) *accepted = 0;
    return 0;
  }
  for (size_t i = 0; i < n; ++i)
    if (!all_finite(grads + i * t->D, t->D)) return 6;
  for (size_t i = 0; i < n; ++i) {
    uint32_t row = find_or_init(t, ids[i]);
    uint32_t dl = count_delay(t, row, read_versions ? read_versions[i] : 0, step_tag);
    if (out_delays) out_delays[i] = dl;
    bump_version(t, row, step_tag);
    apply_one(t, row, grads + i * t->D, lr);
  }
  if (accepted) *accepted = 1;
  return 0;
}

/* PsShard::apply_gradients_map, embedding_ps.hpp:165-189: untracked, one version
 * increment per write. */
int orc_apply_map(orc_table* t, const uint64_t* ids, const float* grads, size_t n, float lr) {
  for (size_t i = 0; i < n; ++i)
    if (!all_finite(grads + i * t->D, t->D)) return 6;
  for (size_t i = 0; i < n; ++i) {
    uint32_t row = find_or_init(t, ids[i]);
    t->versions[row]++;
    apply_one(t, row, grads + i * t->D, lr);
  }
  return 0;
}

/* EmbeddingWorker::serve_pull pooling, embedding_worker.hpp:541-557: per group,
 * fp64 sum of rows in listing order (duplicates counted), times 1/n (mean) or
 * 1 (sum), cast to float; empty groups are zeros. fetch_rows (:677-704) resolves
 * every distinct id before pooling, so reads see one consistent state. */
void orc_pull_batch(orc_table* t, uint32_t B, uint32_t F, const uint64_t* ids,
                    const uint64_t* offsets, int agg, float* out_pooled,
                    uint64_t* out_read_versions) {
  const uint32_t D = t->D;
  double* acc = (double*)malloc(D * sizeof(double));
  for (uint32_t b = 0; b < B; ++b) {
    uint64_t s0 = offsets[(uint64_t)b * F], s1 = offsets[(uint64_t)b * F + F];
    for (uint64_t i = s0; i < s1; ++i) (void)find_or_init(t, ids[i]);
    for (uint32_t g = 0; g < F; ++g) {
      uint64_t a = offsets[(uint64_t)b * F + g], e = offsets[(uint64_t)b * F + g + 1];
      float* out = out_pooled + ((uint64_t)b * F + g) * D;
      if (a == e) {
        memset(out, 0, D * sizeof(float));
        continue;
      }
      for (uint32_t d = 0; d < D; ++d) acc[d] = 0.0;
      for (uint64_t i = a; i < e; ++i) {
        int64_t r = index_find(t, ids[i]);
        const float* w = t->rows + (uint64_t)r * 2 * D;
        for (uint32_t d = 0; d < D; ++d) acc[d] = acc[d] + (double)w[d];
        if (out_read_versions) out_read_versions[i] = t->versions[r];
      }
      double scale = agg == 0 ? 1.0 / (double)(e - a) : 1.0;
      for (uint32_t d = 0; d < D; ++d) out[d] = (float)(acc[d] * scale);
    }
  }
  free(acc);
}

typedef struct {
  uint64_t id;
  uint64_t pos;
  uint32_t group;
} listing;

static int cmp_listing(const void* x, const void* y) {
  const listing* a = (const listing*)x;
  const listing* b = (const listing*)y;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return a->pos < b->pos ? -1 : (a->pos > b->pos);
}

typedef struct {
  uint64_t key;
  uint32_t b;
} sample_ord;

static int cmp_sample(const void* x, const void* y) {
  const sample_ord* a = (const sample_ord*)x;
  const sample_ord* b = (const sample_ord*)y;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->b < b->b ? -1 : (a->b > b->b);
}

/* EmbeddingWorker::push_to_shards (embedding_worker.hpp:726-775) for every sample
 * of the batch in ascending SampleId order (flush_step :788-800): per sample,
 * contribution c_id[d] = float(sum over groups g, over listings of id in g, in
 * listing order, of (double)grad[g*D+d] * scale_g) -- one apply per (sample,
 * unique id) -- then PsShard::apply_gradients (tracked) or apply_gradients_map. */
int orc_push_batch(orc_table* t, uint32_t B, uint32_t F, const uint64_t* ids,
                   const uint64_t* offsets, int agg, const float* grads,
                   const uint64_t* read_versions, const uint64_t* sample_keys, float lr,
                   uint32_t step_tag, uint32_t epoch, uint32_t* out_delays, uint64_t* out_n_delays,
                   int* accepted) {
  const uint32_t D = t->D;
  uint64_t N = offsets[(uint64_t)B * F];
  sample_ord* order = (sample_ord*)malloc((B ? B : 1) * sizeof(sample_ord));
  for (uint32_t b = 0; b < B; ++b) {
    order[b].key = sample_keys ? sample_keys[b] : b;
    order[b].b = b;
  }
  qsort(order, B, sizeof(sample_ord), cmp_sample);

  /* Build every (sample, unique id) contribution first (validation before mutation). */
  listing* ls = (listing*)malloc((N ? N : 1) * sizeof(listing));
  float* contrib = (float*)malloc((N ? N : 1) * D * sizeof(float));
  uint64_t* pair_id = (uint64_t*)malloc((N ? N : 1) * sizeof(uint64_t));
  uint64_t* pair_rv = (uint64_t*)malloc((N ? N : 1) * sizeof(uint64_t));
  uint64_t* sample_pair_off = (uint64_t*)malloc(((uint64_t)B + 1) * sizeof(uint64_t));
  double* acc = (double*)malloc(D * sizeof(double));
  uint64_t P = 0;
  int bad = 0;
  for (uint32_t k = 0; k < B; ++k) {
    uint32_t b = order[k].b;
    sample_pair_off[k] = P;
    uint64_t m = 0;
    for (uint32_t g = 0; g < F; ++g) {
      uint64_t a = offsets[(uint64_t)b * F + g], e = offsets[(uint64_t)b * F + g + 1];
      for (uint64_t i = a; i < e; ++i) {
        ls[m].id = ids[i];
        ls[m].pos = i;
        ls[m].group = g;
        ++m;
      }
    }
    qsort(ls, m, sizeof(listing), cmp_listing); /* std::map per_id: ascending id */
    for (uint64_t r = 0; r < m;) {
      uint64_t q = r;
      for (uint32_t d = 0; d < D; ++d) acc[d] = 0.0;
      while (q < m && ls[q].id == ls[r].id) {
        uint32_t g = ls[q].group;
        uint64_t cnt = offsets[(uint64_t)b * F + g + 1] - offsets[(uint64_t)b * F + g];
        double scale = agg == 0 ? 1.0 / (double)cnt : 1.0;
        const float* gr = grads + ((uint64_t)b * F + g) * D;
        for (uint32_t d = 0; d < D; ++d) {
          double prod = (double)gr[d] * scale;
          acc[d] = acc[d] + prod;
        }
        ++q;
      }
      float* c = contrib + P * D;
      for (uint32_t d = 0; d < D; ++d) c[d] = (float)acc[d];
      if (!all_finite(c, D)) bad = 1;
      pair_id[P] = ls[r].id;
      /* version_of.emplace keeps the first listing's read version (:746-749). */
      pair_rv[P] = read_versions ? read_versions[ls[r].pos] : 0;
      ++P;
      r = q;
    }
  }
  sample_pair_off[B] = P;
  int rc = 0;
  if (epoch != t->epoch) {
    t->stale_drops += P;
    if (accepted) *accepted = 0;
  } else if (bad) {
    rc = 6;
  } else {
    for (uint64_t p = 0; p < P; ++p) {
      uint32_t row = find_or_init(t, pair_id[p]);
      if (read_versions) {
        uint32_t dl = count_delay(t, row, pair_rv[p], step_tag);
        if (out_delays) out_delays[p] = dl;
        bump_version(t, row, step_tag);
      } else {
        t->versions[row]++;
      }
      apply_one(t, row, contrib + p * D, lr);
    }
    if (accepted) *accepted = 1;
  }
  if (out_n_delays) *out_n_delays = P;
  free(order);
  free(ls);
  free(contrib);
  free(pair_id);
  free(pair_rv);
  free(sample_pair_off);
  free(acc);
  return rc;
}

typedef struct {
  uint64_t id;
  uint32_t sample;
} posting;

static int cmp_posting(const void* x, const void* y) {
  const posting* a = (const posting*)x;
  const posting* b = (const posting*)y;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return a->sample < b->sample ? -1 : (a->sample > b->sample);
}

/* compress_indices, codec.hpp:123-156: per group, unique ids ascending, each with
 * the ascending list of samples listing it, within-sample duplicates collapsed. */
int orc_compress_indices(uint32_t B, uint32_t G, const uint64_t* ids, const uint64_t* offsets,
                         uint64_t* group_u_off, uint64_t* unique, uint64_t* post_off,
                         uint16_t* postings) {
  if (B > 65535) return 1;
  uint64_t N = offsets[(uint64_t)B * G];
  posting* ps = (posting*)malloc((N ? N : 1) * sizeof(posting));
  uint64_t u = 0, p = 0;
  group_u_off[0] = 0;
  post_off[0] = 0;
  for (uint32_t g = 0; g < G; ++g) {
    uint64_t m = 0;
    for (uint32_t b = 0; b < B; ++b)
      for (uint64_t i = offsets[(uint64_t)b * G + g]; i < offsets[(uint64_t)b * G + g + 1]; ++i) {
        ps[m].id = ids[i];
        ps[m].sample = b;
        ++m;
      }
    qsort(ps, m, sizeof(posting), cmp_posting);
    for (uint64_t i = 0; i < m; ++i) {
      int new_id = (i == 0 || ps[i].id != ps[i - 1].id);
      if (new_id) {
        if (u > 0 || i > 0) post_off[u] = p;
        unique[u++] = ps[i].id;
      }
      if (new_id || ps[i].sample != ps[i - 1].sample) postings[p++] = (uint16_t)ps[i].sample;
      post_off[u] = p;
    }
    group_u_off[g + 1] = u;
  }
  free(ps);
  return 0;
}
